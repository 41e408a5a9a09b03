#!/usr/bin/env python
"""Bitwise comparison of forward runs under different tiling settings against a
base setting (all pair tilings do the same arithmetic per point).
   python tools/variant_diff.py <so> <n> <nt> '<base env json>' '<env json>' ..."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1608_08658_b200 import configs, seismic as S

so, n, nt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
envs = [json.loads(a) for a in sys.argv[4:]]
w = configs.cfg4(so, n=n, nt=nt)
model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
src = S.locate_points(model, w.src_coords)
rec = S.locate_points(model, w.rec_coords)
print(json.dumps({"padded": list(map(int, model.padded)), "src_idx": np.asarray(src.idx).tolist()}))
KEYS = ("SFDB200_GROUP", "SFDB200_AUTOTUNE", "SFDB200_TILE", "SFDB200_ZCHUNKS", "SFDB200_CTAS", "SFDB200_PDL",
        "SFDB200_UNFUSED", "SFDB200_CARVEOUT")
base = None
for env in envs:
    for k in KEYS:
        os.environ.pop(k, None)
    os.environ.update(env)
    f = S.forward(model, src, w.wavelet, rec, w.nt, w.dt, False)
    u = np.asarray(f.u).copy()
    if base is None:
        base = u
        print(json.dumps({"env": env, "base": True, "norm": float(np.linalg.norm(u))}), flush=True)
        continue
    d = u != base
    out = {"env": env, "differing_cells": int(d.sum())}
    if d.any():
        idx = np.argwhere(d)
        out["box"] = [idx.min(0).tolist(), idx.max(0).tolist()]
        out["rel_l2"] = float(np.linalg.norm(u - base) / np.linalg.norm(base))
    print(json.dumps(out), flush=True)
