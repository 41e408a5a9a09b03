#!/usr/bin/env python
"""Forward runs of one workload under several tiling settings, each compared
with the unmodified reference (oracle/_ref) once computed: finds which sweep
instantiation / item order a parity failure belongs to.
   python tools/variant_check.py cfg4-so4 [n] [nt]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle_lib as O
from paper_1608_08658_b200 import configs, seismic as S

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4-so4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
nt = int(sys.argv[3]) if len(sys.argv) > 3 else 202
so = int(name.split("so")[1])
w = configs.cfg4(so, n=n, nt=nt)
model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
src = S.locate_points(model, w.src_coords)
rec = S.locate_points(model, w.rec_coords)
uo, ro, _ = O.ref_forward(w.interior, w.h, w.nbpml, w.space_order, w.m_interior, w.src_coords,
                          w.wavelet, w.rec_coords, w.nt, w.dt)
SETTINGS = [{}, {"SFDB200_GROUP": "0"}, {"SFDB200_AUTOTUNE": "0"},
            {"SFDB200_TILE": "4,2,4,4,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,4,4,1", "SFDB200_ZCHUNKS": "4", "SFDB200_GROUP": "0"},
            {"SFDB200_TILE": "4,2,4,4,1", "SFDB200_ZCHUNKS": "5"},
            {"SFDB200_TILE": "4,2,4,1,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,3,0,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,4,0,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,4,2,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,4,3,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,3,3,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,3,4,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,5,5,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,5,0,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,3,1,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "8,2,3,1,1", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,4,1,0", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,1,4,1,0", "SFDB200_ZCHUNKS": "4"},
            {"SFDB200_TILE": "4,2,4,4,1", "SFDB200_ZCHUNKS": "4", "SFDB200_CTAS": "-2"},
            {"SFDB200_TILE": "4,2,4,4,1", "SFDB200_ZCHUNKS": "4", "SFDB200_PDL": "0"}]
for env in SETTINGS:
    for k in ("SFDB200_GROUP", "SFDB200_AUTOTUNE", "SFDB200_TILE", "SFDB200_ZCHUNKS", "SFDB200_CTAS",
              "SFDB200_PDL"):
        os.environ.pop(k, None)
    os.environ.update(env)
    try:
        f = S.forward(model, src, w.wavelet, rec, w.nt, w.dt, False)
        u = np.asarray(f.u)
        errs = [O.rel_l2(u[t % 3], uo[t % 3]) for t in (w.nt - 3, w.nt - 2, w.nt - 1)]
        bad = np.argwhere(np.abs(u[(w.nt - 1) % 3] - uo[(w.nt - 1) % 3]) >
                          1e-3 * np.abs(uo[(w.nt - 1) % 3]).max())
        box = [bad.min(0).tolist(), bad.max(0).tolist(), len(bad)] if len(bad) else None
        print(json.dumps({"env": env, "rel_l2": errs, "bad_box": box}), flush=True)
    except Exception as e:  # a refused tiling
        print(json.dumps({"env": env, "error": str(e)[:200]}), flush=True)
