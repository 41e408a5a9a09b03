"""GPU parity: the B200 operators (through the C ABI) against the CPU oracle.

Gate (BASELINE.json north_star): wavefield slots and traces within
rel-L2 <= 1e-5 of the fp64 oracle after the FULL step count, on identical
fp32-rounded inputs; index computation bit-exact.
"""
import numpy as np
import pytest

import oracle_lib as O
from paper_1608_08658_b200 import configs, seismic as S

TOL = 1e-5
pytestmark = pytest.mark.gpu


def _setup(w):
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    src = S.locate_points(model, w.src_coords)
    rec = S.locate_points(model, w.rec_coords)
    return model, src, rec


def _oracle_forward(w, model, src, rec, save=False):
    return O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                     src.idx, src.w, w.wavelet, rec.idx, rec.w, save=save)


@pytest.mark.parametrize("case", [
    ("cfg1-full", lambda: configs.cfg1()),
    ("3d-so2", lambda: configs.cfg4(2, n=48, nt=202, nbpml=10)),
    ("3d-so8", lambda: configs.cfg2(n=48, nt=402, nbpml=20, nrec_side=16)),
    ("3d-so16", lambda: configs.cfg4(16, n=40, nt=202, nbpml=12)),
])
def test_forward_matches_oracle(case):
    name, make = case
    w = make()
    model, src, rec = _setup(w)
    f = S.forward(model, src, w.wavelet, rec, w.nt, w.dt, False)
    u, r = _oracle_forward(w, model, src, rec)
    assert O.rel_l2(f.u, u) <= TOL, name
    if rec.npoints:
        assert O.rel_l2(f.record.data, r) <= TOL, name
    # rows 0 and 1 of the record are never written (time loop starts at 2)
    assert np.all(f.record.data[:2] == 0)


def test_forward_save_history():
    w = configs.cfg2(n=32, nt=122, nbpml=10, nrec_side=8)
    model, src, rec = _setup(w)
    f = S.forward(model, src, w.wavelet, rec, w.nt, w.dt, True)
    u, r = _oracle_forward(w, model, src, rec, save=True)
    assert f.u.shape[0] == w.nt + 1
    assert O.rel_l2(f.u, u) <= TOL
    assert O.rel_l2(f.record.data, r) <= TOL
    assert np.all(f.u[0] == 0) and np.all(f.u[1] == 0) and np.all(f.u[w.nt] == 0)


def test_adjoint_matches_oracle():
    w = configs.cfg2(n=40, nt=302, nbpml=16, nrec_side=12)
    model, src, rec = _setup(w)
    rng = np.random.default_rng(3)
    resid = O._f64(rng.standard_normal((w.nt, rec.npoints)).astype(np.float32))
    a = S.adjoint(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), src, w.nt, w.dt)
    v, s = O.adjoint(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                     src.idx, src.w, rec.idx, rec.w, resid)
    assert O.rel_l2(a.v, v) <= TOL
    assert O.rel_l2(a.src_samples.data, s) <= TOL


def test_gradient_matches_oracle():
    w = configs.cfg2(n=36, nt=252, nbpml=12, nrec_side=10)
    model, src, rec = _setup(w)
    u, r = _oracle_forward(w, model, src, rec, save=True)
    rng = np.random.default_rng(5)
    resid = O._f64((0.5 * r + 0.01 * np.abs(r).max() * rng.standard_normal(r.shape))
                   .astype(np.float32))
    g = S.gradient(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), u, w.nt, w.dt)
    go, _ = O.gradient(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp, u,
                       rec.idx, rec.w, resid)
    assert O.rel_l2(g.grad, go) <= TOL


def test_scattered_points_forward_and_adjoint():
    """Receivers/sources scattered through the volume: exercises fused
    sampling across tile / z-chunk boundaries, its fallback, and fused
    injection with colliding corners."""
    w = configs.cfg2(n=56, nt=162, nbpml=12, nrec_side=4)
    rng = np.random.default_rng(11)
    span = (w.interior[0] - 1) * w.h
    rec_c = rng.uniform(0.0, span, size=(700, 3))
    rec_c[:50] = np.round(rec_c[:50] / w.h) * w.h        # on-node points
    rec_c[50:60] = rec_c[60:70]                           # exact duplicates collide
    src_c = rng.uniform(0.0, span, size=(5, 3))
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    src = S.locate_points(model, src_c)
    rec = S.locate_points(model, rec_c)
    wav = O._f64(np.repeat(w.wavelet[:, :1], 5, axis=1))
    f = S.forward(model, src, wav, rec, w.nt, w.dt, False)
    u, r = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                     src.idx, src.w, wav, rec.idx, rec.w)
    assert O.rel_l2(f.u, u) <= TOL
    assert O.rel_l2(f.record.data, r) <= TOL
    resid = O._f64(rng.standard_normal((w.nt, rec.npoints)).astype(np.float32))
    a = S.adjoint(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), src, w.nt, w.dt)
    v, s = O.adjoint(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                     src.idx, src.w, rec.idx, rec.w, resid)
    assert O.rel_l2(a.v, v) <= TOL
    assert O.rel_l2(a.src_samples.data, s) <= TOL
