import sys, os, time
sys.path.insert(0, '.')
os.environ['SFDB200_PROFILE'] = '1'
import numpy as np, torch, bench
from paper_1608_08658_b200 import _lib as L
w = bench.make_workload('cfg2')
model, src, rec = bench.problem(w)
plan = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints, rec.npoints, False, 0)
def pinned(shape): return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
u = pinned((3, *model.padded)); m = pinned(model.m.shape); m[:] = model.m; damp = pinned(model.damp.shape); damp[:] = model.damp
rd = pinned((w.nt, rec.npoints)); tr = pinned(w.wavelet.shape); tr[:] = w.wavelet
argv = [u, m, damp, L.i64(src.idx), L.f64(src.w), tr, L.i64(rec.idx), L.f64(rec.w), rd]
for i in range(3):
    t = time.perf_counter(); plan.run(argv); print('run', time.perf_counter() - t, flush=True)
