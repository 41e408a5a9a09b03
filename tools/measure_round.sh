# One-GPU measurement pass for profiles/: GPU tests, every bench workload,
# the reference arm, a launch list and one ncu --set full capture of the cfg2
# sweep.  Usage (on the GPU box): bash tools/measure_round.sh <outdir>
set -x
OUT=${1:-gpurun_out/round}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1
for wl in cfg2 cfg1 cfg3 cfg4-so2 cfg4-so4 cfg4-so8 cfg4-so12 cfg4-so16; do
  timeout 1200 python bench.py --workload $wl > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
timeout 1500 python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu --no-e2e > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference_cfg2.json 2> $OUT/bench_reference_cfg2.err
# the autotuned cfg2 tiling, fixed below so no tuning launches precede the profiled ones
set -- $(python -c "
import json; d=json.loads(open('$OUT/bench_cfg2.json').read().strip().splitlines()[-1]); c=d['config']['sweep']
print(c['variant'], c['zchunks'])")
# launch list of a short cfg2 bench run (same command first without ncu)
SFDB200_TILE=$1 SFDB200_ZCHUNKS=$2 timeout 600 python bench.py --workload cfg2 --time-steps 30 --steps 1 --warmup 3 --no-cpu --no-e2e > $OUT/short_cfg2.json 2>&1 && \
SFDB200_TILE=$1 SFDB200_ZCHUNKS=$2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_cfg2.csv python bench.py --workload cfg2 --time-steps 30 --steps 1 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_launch.log 2>&1
# full capture of one sweep
SFDB200_TILE=$1 SFDB200_ZCHUNKS=$2 timeout 600 python tools/sweep_time.py --workload cfg2 --time-steps 4 > $OUT/ncu_full_pre.log 2>&1 && \
SFDB200_TILE=$1 SFDB200_ZCHUNKS=$2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep3d --launch-skip 6 --launch-count 1 -o $OUT/cfg2_full python tools/sweep_time.py --workload cfg2 --time-steps 4 > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py $OUT/cfg2_full.ncu-rep > $OUT/ncu_cfg2_full.json
# the cfg4 so 8 sweep and the cfg3 gradient sweep, autotuned tilings
set -- $(python -c "
import json; d=json.loads(open('$OUT/bench_cfg4-so8.json').read().strip().splitlines()[-1]); c=d['config']['sweep']
print(c['variant'], c['zchunks'])")
SFDB200_TILE=$1 SFDB200_ZCHUNKS=$2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep3d --launch-skip 6 --launch-count 1 -o $OUT/cfg4so8_full python tools/sweep_time.py --workload cfg4-so8 --time-steps 4 > $OUT/ncu_cfg4.log 2>&1
python tools/ncu_summary.py $OUT/cfg4so8_full.ncu-rep > $OUT/ncu_cfg4so8_full.json
set -- $(python -c "
import json; d=json.loads(open('$OUT/bench_cfg3.json').read().strip().splitlines()[-1]); c=d['config']['sweep']
print(c['variant'], c['zchunks'])")
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep3d --launch-skip 4 --launch-count 1 -o $OUT/cfg3_full python tools/tune.py --workload cfg3 --gradient --time-steps 8 --tiles $1 --zchunks $2 --reps 1 > $OUT/ncu_cfg3.log 2>&1
python tools/ncu_summary.py $OUT/cfg3_full.ncu-rep > $OUT/ncu_cfg3_full.json
python tools/power_probe.py 4 > $OUT/power.jsonl 2>&1
echo done
