#!/usr/bin/env python
"""One seeded case of tests/test_gpu_fuzz.py with its errors printed (B200):
   python tools/fuzz_case.py 432 441"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import json
import numpy as np
import oracle_lib as O
import test_gpu_fuzz as F
from paper_1608_08658_b200 import seismic as S

for seed in map(int, sys.argv[1:]):
    model, src, rec, wav, nt, dt = F._case(seed)
    P, so, h = model.padded, model.space_order, model.h
    uo, ro = O.forward(P, so, h, dt, nt, model.m, model.damp, src.idx, src.w, wav, rec.idx, rec.w, save=True)
    f = S.forward(model, src, wav, rec, nt, dt, True)
    white = np.random.default_rng(seed).standard_normal((nt, rec.npoints))
    pulse = S.ricker(0.05 / dt / 4, 1.2 * 4 * dt / 0.05, nt, dt)
    smooth = np.stack([np.convolve(white[:, r], pulse)[:nt] for r in range(rec.npoints)], 1)
    resid = O._f64((smooth / np.abs(smooth).max()).astype(np.float32))
    rs = S.ShotRecord(nt, dt, rec.npoints, resid)
    a = S.adjoint(model, rec, rs, src, nt, dt)
    vo, so_ = O.adjoint(P, so, h, dt, nt, model.m, model.damp, src.idx, src.w, rec.idx, rec.w, resid)
    g = S.gradient(model, rec, rs, uo, nt, dt)
    go, _ = O.gradient(P, so, h, dt, nt, model.m, model.damp, uo, rec.idx, rec.w, resid)
    # the same gradient from the GPU's own fp32 history (what fwi_gradient uses)
    g2 = S.gradient(model, rec, rs, np.asarray(f.u), nt, dt)
    print(json.dumps({"seed": seed, "padded": list(map(int, P)), "so": so, "nt": nt, "nsrc": src.npoints,
                      "nrec": rec.npoints, "dt_over_crit": dt / S.critical_dt(model),
                      "fwd_rel_l2": O.rel_l2(f.u, uo), "adj_rel_l2": O.rel_l2(a.v, vo),
                      "grad_rel_l2": O.rel_l2(g.grad, go), "grad_rel_l2_gpu_history": O.rel_l2(g2.grad, go),
                      "grad_norm": float(np.linalg.norm(go)), "u_norm": float(np.linalg.norm(uo)),
                      "v_norm": float(np.linalg.norm(vo))}), flush=True)
