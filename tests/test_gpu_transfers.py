"""Half-width host transfers (hostio.cpp copy_h2d_narrow / copy_d2h_widen):
pageable fp64 caller buffers -- the reference's std::vectors -- cross PCIe as
fp32 (narrowed on the host exactly as the device rounds, widened back
exactly), so results must equal the direct fp64 DMA of pinned buffers (and
SFDB200_NARROW=0) bit for bit; a model that is not fp32-representable falls
back to moving m as fp64, with the same bits again."""
import numpy as np
import pytest

import oracle_lib as O
from paper_1608_08658_b200 import _lib as L
from paper_1608_08658_b200 import configs, seismic as S

pytestmark = pytest.mark.gpu


def _pinned(a):
    import torch
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
    t[...] = a
    return t


def _forward_outputs(plan, model, src, rec, w, alloc):
    u = alloc(np.full((3, *model.padded), 3.0))
    r = alloc(np.full((w.nt, rec.npoints), 5.0))
    argv = [u, alloc(model.m), alloc(model.damp), src.idx, src.w, alloc(O._f64(w.wavelet)),
            rec.idx, rec.w, r]
    plan.run(argv)
    return u.copy(), r.copy(), plan.h2d_bytes, plan.d2h_bytes


@pytest.mark.parametrize("exact_model", [True, False])
def test_forward_pageable_pinned_and_fp64_paths_bitwise(monkeypatch, exact_model):
    w = configs.cfg2(n=48, nt=150, nbpml=8, nrec_side=64)  # record > one 32 MB chunk
    mi = w.m_interior.copy()
    if not exact_model:  # a few cells off the fp32 grid: m must travel as fp64
        mi[::97] *= 1.0 + 2.0 ** -40
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, mi)
    src, rec = S.locate_points(model, w.src_coords), S.locate_points(model, w.rec_coords)
    p = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
               rec.npoints, False, 0)
    _forward_outputs(p, model, src, rec, w, np.array)  # builds the sparse tables once
    pageable = _forward_outputs(p, model, src, rec, w, np.array)
    pinned = _forward_outputs(p, model, src, rec, w, _pinned)
    monkeypatch.setenv("SFDB200_NARROW", "0")
    fp64 = _forward_outputs(p, model, src, rec, w, np.array)
    p.close()
    for out in (pinned, fp64):
        assert np.array_equal(pageable[0], out[0]) and np.array_equal(pageable[1], out[1])
    cells = int(np.prod(model.padded))
    # m: 4 B per cell when exact, else 8; the source trace, the u slots and the
    # record: 4 B per value
    assert pinned[2] - pageable[2] == (cells * 4 if exact_model else 0) + w.nt * src.npoints * 4
    assert pinned[3] - pageable[3] == (3 * cells + w.nt * rec.npoints) * 4
    assert fp64[2] == pinned[2] and fp64[3] == pinned[3]
    uo, ro = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                       src.idx, src.w, w.wavelet, rec.idx, rec.w)
    assert O.rel_l2(pageable[0], uo) <= 1e-5 and O.rel_l2(pageable[1], ro) <= 1e-5


def test_adjoint_and_gradient_host_history_bitwise(monkeypatch):
    """The adjoint's residual in / source samples out, and the gradient's
    uploaded host u history (nt + 1 rows) and grad out, through both paths."""
    w = configs.cfg2(n=32, nt=110, nbpml=8, nrec_side=12)
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    src, rec = S.locate_points(model, w.src_coords), S.locate_points(model, w.rec_coords)
    uh, rr = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                       src.idx, src.w, w.wavelet, rec.idx, rec.w, save=True)
    resid = O._f64(np.random.default_rng(3).standard_normal(rr.shape).astype(np.float32))
    res = {}
    for name, alloc, narrow in (("pageable", np.array, "1"), ("pinned", _pinned, "1"),
                                ("fp64", np.array, "0")):
        monkeypatch.setenv("SFDB200_NARROW", narrow)
        pa = L.Plan(L.ADJOINT, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                    rec.npoints, False, 0)
        v, sm = alloc(np.zeros((3, *model.padded))), alloc(np.zeros((w.nt, src.npoints)))
        pa.run([v, alloc(model.m), alloc(model.damp), src.idx, src.w, sm, rec.idx, rec.w,
                alloc(resid)])
        pa.close()
        pg = L.Plan(L.GRADIENT, 3, model.padded, w.space_order, w.nt, w.dt, w.h, 0,
                    rec.npoints, False, 0)
        g = alloc(np.zeros(model.padded))
        pg.run([alloc(np.zeros((3, *model.padded))), alloc(uh), alloc(model.m),
                alloc(model.damp), g, rec.idx, rec.w, alloc(resid)])
        pg.close()
        res[name] = (v.copy(), sm.copy(), g.copy())
    for name in ("pinned", "fp64"):
        for a, b in zip(res["pageable"], res[name]):
            assert np.array_equal(a, b), name
    go, _ = O.gradient(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp, uh,
                       rec.idx, rec.w, resid)
    assert O.rel_l2(res["pageable"][2], go) <= 1e-5
