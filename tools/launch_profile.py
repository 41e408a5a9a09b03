#!/usr/bin/env python
"""Per-launch sweep times across one run (CUDA events around every launch)."""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--time-steps", type=int, default=1000)
    ap.add_argument("--no-rec", action="store_true")
    ap.add_argument("--runs", type=int, default=3)
    args = ap.parse_args()
    import ctypes as C
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
    import torch
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    plan.set_stream(stream.cuda_stream)
    plan.upload(argv)
    plan.execute()
    for r in range(args.runs):
        plan.set_timing(True)
        plan.execute()
        ms, n = plan.stencil_time()
        plan.set_timing(False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        plan.execute()
        e1.record()
        torch.cuda.synchronize()
        whole = e0.elapsed_time(e1)
        print(json.dumps({"run": r, "mean_us": ms / n * 1e3, "launches": n,
                          "gpts_kernel": plan.points_per_step / (ms / n) / 1e6,
                          "gpts_whole": plan.points_per_step * plan.steps / whole / 1e6}),
              flush=True)


if __name__ == "__main__":
    main()
