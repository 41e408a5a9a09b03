# One-GPU measurement pass for profiles/: GPU tests, every bench workload,
# the reference arm, a launch list and ncu --set full captures of the benched
# sweep instantiations (their DRAM traffic recorded in profiles/ncu_summary.json
# under the key bench.py looks up).  Usage (on the GPU box):
#   bash tools/measure_round.sh <outdir> [workloads...]
set -x
OUT=${1:-gpurun_out/round}
shift
WLS=${@:-cfg2 cfg1 cfg3 cfg4-so2 cfg4-so4 cfg4-so8 cfg4-so12 cfg4-so16 cfg5}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt
for wl in $WLS; do
  case $wl in
    cfg5) timeout 1500 python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu --no-e2e > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err ;;
    *) timeout 1200 python bench.py --workload $wl > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err ;;
  esac
done
# ncu: the instantiation each bench line autotuned to, forced, one launch captured
capture() {  # workload, bench line, extra tool args
  local wl=$1 line=$2
  [ -s $line ] || return
  set -- $(python -c "
import json; d=json.loads(open('$line').read().strip().splitlines()[-1]); c=d['config']['sweep']
print(c['variant'], c['zchunks'], c.get('ctas', 0))")
  local tile=$1 zc=$2
  export SFDB200_CTAS=$3
  if [ $wl = cfg3 ]; then
    SFDB200_TILE=$tile SFDB200_ZCHUNKS=$zc timeout 600 python tools/tune.py --workload cfg3 --gradient --time-steps 8 --tiles $tile --zchunks $zc --reps 1 > $OUT/ncu_pre_$wl.log 2>&1 && \
    SFDB200_TILE=$tile SFDB200_ZCHUNKS=$zc timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep3d --launch-skip 4 --launch-count 1 -o $OUT/${wl}_full python tools/tune.py --workload cfg3 --gradient --time-steps 8 --tiles $tile --zchunks $zc --reps 1 > $OUT/ncu_$wl.log 2>&1
  else
    SFDB200_TILE=$tile SFDB200_ZCHUNKS=$zc timeout 600 python tools/sweep_time.py --workload $wl --time-steps 4 > $OUT/ncu_pre_$wl.log 2>&1 && \
    SFDB200_TILE=$tile SFDB200_ZCHUNKS=$zc timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep3d --launch-skip 6 --launch-count 1 -o $OUT/${wl}_full python tools/sweep_time.py --workload $wl --time-steps 4 > $OUT/ncu_$wl.log 2>&1
  fi
  python tools/ncu_summary.py $OUT/${wl}_full.ncu-rep > $OUT/ncu_${wl}_full.json
  python tools/ncu_traffic.py $OUT/${wl}_full.ncu-rep $line profiles/${OUT#gpurun_out/}/ncu_${wl}_full.json > $OUT/ncu_traffic_$wl.json
  unset SFDB200_CTAS
}
for wl in $WLS; do
  case $wl in cfg1) ;; *) capture $wl $OUT/bench_$wl.json ;; esac
done
# launch list of a short cfg2 bench run (same command first without ncu)
if [ -s $OUT/bench_cfg2.json ]; then
  set -- $(python -c "
import json; d=json.loads(open('$OUT/bench_cfg2.json').read().strip().splitlines()[-1]); c=d['config']['sweep']
print(c['variant'], c['zchunks'])")
  SFDB200_TILE=$1 SFDB200_ZCHUNKS=$2 timeout 600 python bench.py --workload cfg2 --time-steps 30 --steps 1 --warmup 3 --no-cpu --no-e2e > $OUT/short_cfg2.json 2>&1 && \
  SFDB200_TILE=$1 SFDB200_ZCHUNKS=$2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_cfg2.csv python bench.py --workload cfg2 --time-steps 30 --steps 1 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_launch.log 2>&1
fi
[ -s $OUT/launches_cfg2.csv ] && python tools/launch_list.py $OUT/launches_cfg2.csv "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 of: SFDB200_TILE/ZCHUNKS=<autotuned cfg2 pick> python bench.py --workload cfg2 --time-steps 30 --steps 1 --warmup 3 --no-cpu --no-e2e (cold-cache, serialised)" > $OUT/launches_cfg2.json
cp profiles/ncu_summary.json $OUT/ncu_summary.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference_cfg2.json 2> $OUT/bench_reference_cfg2.err
python tools/power_probe.py 4 > $OUT/power.jsonl 2>&1
# gpurun merges at most 64 MiB back: keep the summaries, and only the cfg2 and
# so-16 reports themselves
for f in $OUT/*_full.ncu-rep; do
  case $f in *cfg2_full*|*cfg4-so16_full*) ;; *) rm -f $f ;; esac
done
echo done
