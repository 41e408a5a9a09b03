#!/usr/bin/env python
"""Repeats one forward run under each tiling setting and counts the distinct
results (a race shows up as more than one).
   python tools/race_hunt.py <so> <n> <nt> <reps> '<env json>' ..."""
import hashlib, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1608_08658_b200 import configs, seismic as S

so, n, nt, reps = (int(a) for a in sys.argv[1:5])
envs = [json.loads(a) for a in sys.argv[5:]]
# so = 5: the cfg5 shape (so 16, 4 sources, receiver carpet) at n^3; so = -8: cfg2's
w = (configs.cfg5(n=n, nt=nt, nrec_side=max(8, n // 2)) if so == 5 else
     configs.cfg2(n=n, nt=nt, nrec_side=max(8, n // 2)) if so == -8 else configs.cfg4(so, n=n, nt=nt))
model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
src = S.locate_points(model, w.src_coords)
rec = S.locate_points(model, w.rec_coords)
KEYS = ("SFDB200_GROUP", "SFDB200_AUTOTUNE", "SFDB200_TILE", "SFDB200_ZCHUNKS", "SFDB200_CTAS", "SFDB200_PDL",
        "SFDB200_UNFUSED", "SFDB200_CARVEOUT")
for env in envs:
    for k in KEYS:
        os.environ.pop(k, None)
    os.environ.update(env)
    seen = {}
    for _ in range(reps):
        f = S.forward(model, src, w.wavelet, rec, w.nt, w.dt, False)
        u = np.ascontiguousarray(np.asarray(f.u)[(w.nt - 1) % 3])
        h = hashlib.md5(u.tobytes() + np.ascontiguousarray(f.record.data).tobytes()).hexdigest()[:8]
        seen.setdefault(h, [0, float(np.linalg.norm(u))])[0] += 1
    print(json.dumps({"env": env, "distinct": len(seen), "results": seen}), flush=True)
