# A/B of the sweep kernels' shared-memory carveout (SFDB200_CARVEOUT: unset =
# smallest carveout holding the register-limited CTAs, -1 = driver's choice,
# 100 = all shared).  Usage on the GPU box: bash tools/ab_carveout.sh OUTDIR
OUT=${1:-gpurun_out/carveout}; mkdir -p $OUT
for wl in cfg3 cfg2 cfg4-so8; do
 for cv in "" -1 100; do
  SFDB200_CARVEOUT=$cv timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/ab_${wl}_cv$cv.json 2> $OUT/ab_${wl}_cv$cv.err
 done
done
