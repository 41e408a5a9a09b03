set -x
mkdir -p gpurun_out/r01d
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r01d/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r01d/pytest_gpu.txt 2>&1
for wl in cfg2 cfg1 cfg3 cfg4-so2 cfg4-so4 cfg4-so8 cfg4-so12 cfg4-so16; do
  timeout 1200 python bench.py --workload $wl > gpurun_out/r01d/bench_$wl.json 2> gpurun_out/r01d/bench_$wl.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01d/bench_reference_cfg2.json 2> gpurun_out/r01d/bench_reference_cfg2.err
# launch list of a short cfg2 run (same command first without ncu)
timeout 600 python bench.py --workload cfg2 --time-steps 30 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r01d/short_cfg2.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01d/launches_cfg2.csv python bench.py --workload cfg2 --time-steps 30 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r01d/ncu_launch.log 2>&1
# full capture of the autotuned cfg2 sweep (tile fixed to the autotune pick so no tuning launches precede it)
TILE=$(python -c "
import json; d=json.loads(open('gpurun_out/r01d/bench_cfg2.json').read().strip().splitlines()[-1]); c=d['config']['sweep']
pair=1 if c['mapping'].startswith('column') else 0; rot=0 if 'shifted' in c['mapping'] else 1
by=c['warps']-1; ny=c['rows_per_thread']//2; print(f\"{by},{ny},{c['stages']},{rot},{pair} {c['zchunks']}\")")
set -- $TILE
SFDB200_TILE=$1 SFDB200_ZCHUNKS=$2 timeout 600 python tools/sweep_time.py --workload cfg2 --time-steps 4 > gpurun_out/r01d/ncu_full_pre.log 2>&1 && \
SFDB200_TILE=$1 SFDB200_ZCHUNKS=$2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep3d --launch-skip 6 --launch-count 1 -o gpurun_out/r01d/cfg2_full python tools/sweep_time.py --workload cfg2 --time-steps 4 > gpurun_out/r01d/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/r01d/cfg2_full.ncu-rep > gpurun_out/r01d/ncu_cfg2_full.json
echo done
