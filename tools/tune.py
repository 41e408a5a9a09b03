#!/usr/bin/env python
"""Sweep-kernel tiling sweep on one GPU: for each SFDB200_TILE / SFDB200_ZCHUNKS
setting, create a forward plan for the workload and time execute() with CUDA
events (device-resident inputs).  Prints one JSON line per setting."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--time-steps", type=int, default=100)
    ap.add_argument("--tiles", default="4,2,4,1;4,2,4,0;4,1,4,1;8,1,3,1")
    ap.add_argument("--zchunks", default="0")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-rec", action="store_true")
    ap.add_argument("--gradient", action="store_true",
                    help="time the fused gradient (GRAD) kernel with a zero history")
    args = ap.parse_args()

    import torch
    import bench
    from paper_1608_08658_b200 import _lib as L

    w = bench.make_workload(args.workload, args.time_steps)
    if args.no_rec:
        w.rec_coords = w.rec_coords[:0]
    model, src, rec = bench.problem(w)
    argv = [np.empty((3, *model.padded)), L.f64(model.m), L.f64(model.damp), L.i64(src.idx),
            L.f64(src.w), L.f64(w.wavelet), L.i64(rec.idx), L.f64(rec.w),
            np.empty((w.nt, rec.npoints))]
    kind, nsrc = L.FORWARD, src.npoints
    if args.gradient:  # residual injected at the receivers, u history all zero
        kind, nsrc = L.GRADIENT, 0
        hist = np.zeros((w.nt + 1, *model.padded))
        resid = np.random.default_rng(0).standard_normal((w.nt, rec.npoints))
        argv = [None, hist, L.f64(model.m), L.f64(model.damp), np.empty(model.padded),
                L.i64(rec.idx), L.f64(rec.w), resid]
    for tile in args.tiles.split(";"):
        for zc in args.zchunks.split(","):
            os.environ["SFDB200_TILE"] = tile
            if zc != "0":
                os.environ["SFDB200_ZCHUNKS"] = zc
            else:
                os.environ.pop("SFDB200_ZCHUNKS", None)
            plan = L.Plan(kind, 3, model.padded, w.space_order, w.nt, w.dt, w.h,
                          nsrc, rec.npoints, False, 0)
            plan.upload(argv)
            plan.execute()
            torch.cuda.synchronize()
            plan.set_timing(True)
            best = None
            for _ in range(args.reps):
                plan.execute()
                ms, n = plan.stencil_time()
                best = ms / n if best is None else min(best, ms / n)
            plan.set_timing(False)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.execute()
            e1.record()
            torch.cuda.synchronize()
            step_ms = e0.elapsed_time(e1) / plan.steps
            gbs = plan.info()["bytes_per_point"] * plan.points_per_step / (best / 1e3) / 1e9
            print(json.dumps({"workload": w.name, "tile": tile, "zchunks": zc,
                              "sweep_ms": best, "step_ms": step_ms, "cfg": plan.info(), "gpts": plan.points_per_step / best / 1e6,
                              "alg_GBps": gbs}), flush=True)
            plan.close()


if __name__ == "__main__":
    main()
