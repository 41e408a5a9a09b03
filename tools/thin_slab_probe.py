#!/usr/bin/env python
"""Throughput of a standalone plan whose z extent is one z-slab rank's
(cfg5 at 8 ranks: 154 padded planes of 1120 x 1120), against taller grids: how
much a thin slab costs by itself, without any exchange."""
import json, sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
from paper_1608_08658_b200 import _lib as L, seismic as S
for nz in (58, 116, 1024):
    model = S.make_constant_model([nz, 1024, 1024], 10.0, 40, 16, 3000.0)
    dt = 0.8 * S.critical_dt(model)
    nt = 22
    src = S.locate_points(model, [[10.0, 5000.0, 5000.0]])
    rec = S.locate_points(model, [[20.0, 100.0, 100.0]])
    p = L.Plan(L.FORWARD, 3, model.padded, 16, nt, dt, 10.0, 1, 1, False, 0)
    st = torch.cuda.Stream(); p.set_stream(st.cuda_stream)
    p.upload([None, model.m, model.damp, src.idx, src.w, np.zeros((nt, 1)), rec.idx, rec.w, np.zeros((nt, 1))])
    p.execute(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); p.execute(); e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"nz": nz, "padded": model.padded, "gpts": p.points_per_step * p.steps / ms / 1e6, "cfg": {k: p.info()[k] for k in ("zchunks", "instantiation", "ctas")}}))
    p.close(); del model
