#!/usr/bin/env python
"""End-to-end cfg2 forward through sfdb200_run with plain (pageable) numpy
host arrays, as the reference's std::vector buffers would be, vs pinned
(pinned first, as bench.py does)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SFDB200_PROFILE", "1")
import numpy as np  # noqa: E402


def main():
    import torch
    import bench
    from paper_1608_08658_b200 import _lib as L
    w = bench.make_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
    model, src, rec = bench.problem(w)
    plan = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                  rec.npoints, False, 0)
    def pinned(shape):
        return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    u = pinned((3, *model.padded)); m = pinned(model.m.shape); m[:] = model.m
    d = pinned(model.damp.shape); d[:] = model.damp; rd = pinned((w.nt, rec.npoints))
    tr = pinned(w.wavelet.shape); tr[:] = w.wavelet
    for kind in ("pinned", "pageable", "pageable-touched"):
        if kind == "pinned":
            argv = [u, m, d, L.i64(src.idx), L.f64(src.w), tr, L.i64(rec.idx), L.f64(rec.w), rd]
        else:
            pu = np.empty_like(u); prd = np.empty_like(rd)
            if kind == "pageable-touched":
                pu[:] = 0; prd[:] = 0
            argv = [pu, np.array(m), np.array(d), L.i64(src.idx), L.f64(src.w), np.array(tr),
                    L.i64(rec.idx), L.f64(rec.w), prd]
        plan.run(argv)
        t0 = time.perf_counter()
        plan.run(argv)
        print(kind, "run ms", round((time.perf_counter() - t0) * 1e3, 1), flush=True)


if __name__ == "__main__":
    main()
