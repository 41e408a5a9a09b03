#!/usr/bin/env python
"""Whole-run step time vs per-launch sweep time of one forward plan (device
resident), for the autotuned tiling or SFDB200_TILE / SFDB200_ZCHUNKS /
SFDB200_PDL from the environment.  Prints one JSON line."""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--time-steps", type=int, default=300)
    ap.add_argument("--no-rec", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import bench
    from paper_1608_08658_b200 import _lib as L
    w = bench.make_workload(args.workload, args.time_steps)
    if args.no_rec:
        w.rec_coords = w.rec_coords[:0]
    model, src, rec = bench.problem(w)
    argv = [None, L.f64(model.m), L.f64(model.damp), L.i64(src.idx), L.f64(src.w),
            L.f64(w.wavelet), L.i64(rec.idx), L.f64(rec.w), np.empty((w.nt, rec.npoints))]
    plan = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                  rec.npoints, False, 0)
    stream = torch.cuda.Stream()
    plan.set_stream(stream.cuda_stream)
    plan.upload(argv)
    plan.execute()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step = []
    for _ in range(args.reps):
        e0.record(stream)
        plan.execute()
        e1.record(stream)
        torch.cuda.synchronize()
        step.append(e0.elapsed_time(e1) / plan.steps)
    plan.set_timing(True)
    plan.execute()
    torch.cuda.synchronize()
    ms, n = plan.stencil_time()
    print(json.dumps({"workload": w.name, "no_rec": args.no_rec, "env": {k: v for k, v in os.environ.items() if k.startswith("SFDB200_")},
                      "step_ms": min(step), "steps_ms_all": step, "sweep_ms": ms / n,
                      "gpts_step": plan.points_per_step / min(step) / 1e6,
                      "cfg": plan.info()}), flush=True)


if __name__ == "__main__":
    main()
