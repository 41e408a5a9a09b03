#!/usr/bin/env python
"""Mean sweep-launch time of one autotuned forward run (device-resident)."""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--time-steps", type=int, default=200)
    ap.add_argument("--no-rec", action="store_true")
    args = ap.parse_args()
    import torch
    import bench
    from paper_1608_08658_b200 import _lib as L
    w = bench.make_workload(args.workload, args.time_steps)
    if args.no_rec:
        w.rec_coords = w.rec_coords[:0]
    model, src, rec = bench.problem(w)
    argv = [None, model.m, model.damp, src.idx, src.w, w.wavelet, rec.idx, rec.w,
            np.zeros((w.nt, rec.npoints))]
    plan = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                  rec.npoints, False, 0)
    plan.upload(argv)
    plan.execute()
    plan.set_timing(True)
    best = 1e9
    for _ in range(3):
        plan.execute()
        ms, n = plan.stencil_time()
        best = min(best, ms / n)
    print(json.dumps({"workload": w.name, "no_rec": args.no_rec, "sweep_ms": best,
                      "gpts": plan.points_per_step / best / 1e6,
                      "frac": 20 * plan.points_per_step / (best / 1e3) / 6468.6e9,
                      "cfg": plan.info()}))


if __name__ == "__main__":
    main()
