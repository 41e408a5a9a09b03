#!/usr/bin/env python
"""Decomposition overhead of the z-slab split, measured on ONE GPU: the
workload as one plan, and as N emulated ranks (loopback communicators, the
fused P2P launch with its boundary tiles first, peer stores into each other's
rows) run in lockstep by sfdb200_execute_group on one stream.  The group runs
the ranks' launches one after another, so its device time is the sum of the
per-rank sweep times: the ratio one_plan / (group / N) is the parallel
efficiency the decomposition itself allows (boundary items, their queue
prologues, per-launch tails), before any NVLink transfer or synchronisation
cost.  One JSON line per N.

  python tools/emulated_scaling.py --workload cfg5 --time-steps 50 --ranks 2,4,8
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg5")
    ap.add_argument("--time-steps", type=int, default=50)
    ap.add_argument("--ranks", default="2,4,8")
    ap.add_argument("--no-p2p", action="store_true",
                    help="ghost planes by device copies between the plans (the planes the "
                         "NCCL exchange sends) instead of the fused P2P launch")
    args = ap.parse_args()
    import torch
    import bench
    from paper_1608_08658_b200 import _lib as L
    from paper_1608_08658_b200 import seismic as S
    w = bench.make_workload(args.workload, args.time_steps)
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    src, rec = S.locate_points(model, w.src_coords), S.locate_points(model, w.rec_coords)
    stream = torch.cuda.Stream()

    def argv():
        return [None, model.m, model.damp, src.idx, src.w, np.ascontiguousarray(w.wavelet),
                rec.idx, rec.w, np.zeros((w.nt, rec.npoints))]

    def timed(fn, reps=2):
        fn()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    p = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
               rec.npoints, False, 0)
    p.set_stream(stream.cuda_stream)
    p.upload(argv())
    one = timed(p.execute)
    info = p.info()
    pts = w.points_per_step * (w.nt - 2)
    print(json.dumps({"workload": w.name, "ranks": 1, "ms": one, "gpts": pts / one / 1e6,
                      "sweep": info["instantiation"]}), flush=True)
    for n in [int(x) for x in args.ranks.split(",")]:
        comms = [L.Comm.loopback(n, r, 0) for r in range(n)]
        plans = []
        for r in range(n):
            q = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h,
                       src.npoints, rec.npoints, False, 0, comm=comms[r])
            q.set_stream(stream.cuda_stream)
            plans.append(q)
        if not args.no_p2p:
            L.peer_group(plans)
        for q in plans:
            q.upload(argv())
        ms = timed(lambda: L.execute_group(plans))
        print(json.dumps({"workload": w.name, "ranks": n, "group_ms": ms,
                          "per_rank_ms": ms / n, "efficiency_bound": one / ms,
                          "sweep": plans[0].info()["instantiation"],
                          "zchunks": plans[0].info()["zchunks"]}), flush=True)
        for q in plans:
            q.close()
        for c in comms:
            c.close()
    # the single plan again after the groups: clock / power drift over the run
    # shows as a change of this figure
    again = timed(p.execute)
    p.close()
    print(json.dumps({"workload": w.name, "ranks": 1, "ms_after": again,
                      "gpts_after": pts / again / 1e6}), flush=True)


if __name__ == "__main__":
    main()
