# Quick one-GPU check of a kernel change: a pytest subset, then device-resident
# bench lines (no CPU arm, no e2e) for the listed workloads, one summary row each.
#   bash tools/quick_bench.sh <outdir> "<pytest args or empty>" [workloads...]
O=${1:-gpurun_out/quick}; T=$2; shift 2
WLS=${@:-cfg4-so16 cfg4-so12 cfg4-so8 cfg2 cfg3}
mkdir -p $O
if [ -n "$T" ]; then timeout 1500 python -m pytest $T -x -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt; fi
for wl in $WLS; do
  timeout 900 python bench.py --workload $wl --no-cpu --no-e2e > $O/bench_$wl.json 2>> $O/err.txt
done
python - $O <<'P'
import json, glob, sys
for f in sorted(glob.glob(sys.argv[1] + '/bench_*.json')):
    for l in open(f):
        try: d = json.loads(l)
        except Exception: continue
        s = d['config']['sweep']
        print(f.split('/')[-1], round(d['value'], 1), 'Gpts/s; sweep', round(d['roofline']['mean_launch_ms'] * 1e3, 1), 'us; frac',
              round(d['roofline']['frac'], 3), s['variant'], 'z', s['zchunks'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
P
