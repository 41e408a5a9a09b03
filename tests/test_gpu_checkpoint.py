"""Uniform checkpointing of the forward history for the FWI gradient
(include/sfdb200.h sfdb200_set_checkpointing).

The gradient recomputed from checkpoints must equal the gradient over the
full saved history (same kernels, same order: bitwise except for atomics on
colliding injection corners) and the CPU oracle's gradient within the fp32
gate."""
import numpy as np
import pytest

import oracle_lib as O
from paper_1608_08658_b200 import _lib as L
from paper_1608_08658_b200 import configs, seismic as S

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _problem(n=30, nt=152, nbpml=8, nrec_side=8):
    w = configs.cfg3(n=n, nt=nt, nbpml=nbpml, nrec_side=nrec_side)
    true = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    bg = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.extra["m_background"])
    src = S.locate_points(bg, w.src_coords)
    rec = S.locate_points(bg, w.rec_coords)
    obs = S.forward(true, src, w.wavelet, rec, w.nt, w.dt, False).record
    return w, bg, src, rec, obs


@pytest.fixture(scope="module")
def problem():
    return _problem()


@pytest.fixture(scope="module")
def full(problem):
    w, bg, src, rec, obs = problem
    return S.fwi_gradient(bg, src, w.wavelet, rec, obs, w.nt, w.dt, checkpoint_interval=0)


@pytest.mark.parametrize("k", [1, 7, 16, 150, 400])
def test_checkpointed_gradient_equals_full_history(problem, full, k):
    w, bg, src, rec, obs = problem
    r = S.fwi_gradient(bg, src, w.wavelet, rec, obs, w.nt, w.dt, checkpoint_interval=k)
    assert r.phi == full.phi
    assert np.array_equal(r.record.data, full.record.data)
    assert O.rel_l2(r.grad, full.grad) <= 1e-6, k
    steps = w.nt - 2
    segs = -(-steps // k)
    cells = 1
    for e in bg.padded[:-1]:
        cells *= e
    cells *= (bg.padded[-1] + 31) // 32 * 32
    assert r.history_bytes == (2 * (segs - 1) + k + 2) * cells * 4


def test_full_history_gradient_matches_oracle(problem, full):
    w, bg, src, rec, obs = problem
    u, syn = O.forward(bg.padded, w.space_order, w.h, w.dt, w.nt, bg.m, bg.damp, src.idx,
                       src.w, w.wavelet, rec.idx, rec.w, save=True)
    resid = syn - L.f64(obs.data).reshape(syn.shape)
    go, _ = O.gradient(bg.padded, w.space_order, w.h, w.dt, w.nt, bg.m, bg.damp, u, rec.idx,
                       rec.w, resid)
    assert O.rel_l2(full.grad, go) <= TOL
    assert O.rel_l2(full.record.data, syn) <= TOL


def test_checkpoint_api_errors(problem):
    w, bg, src, rec, obs = problem
    f_saved = L.Plan(L.FORWARD, 3, bg.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                     rec.npoints, True, 0)
    with pytest.raises(ValueError):
        f_saved.set_checkpointing(8)  # a saved history needs no checkpoints
    f_saved.close()
    fwd = L.Plan(L.FORWARD, 3, bg.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                 rec.npoints, False, 0)
    g = L.Plan(L.GRADIENT, 3, bg.padded, w.space_order, w.nt, w.dt, w.h, 0, rec.npoints,
               False, 0)
    with pytest.raises(ValueError):
        g.bind_checkpoints(fwd)  # checkpointing not enabled
    fwd.set_checkpointing(10)
    g.bind_checkpoints(fwd)
    grad = np.empty(bg.padded)
    resid = np.zeros((w.nt, rec.npoints))
    with pytest.raises(ValueError):  # the forward plan has not run
        g.run([None, None, bg.m, bg.damp, grad, rec.idx, rec.w, resid])
    g.close()
    fwd.close()
    with pytest.raises(ValueError):
        S.fwi_gradient(S.make_constant_model([20, 20], 10.0, 4, 4, 1500.0), src, w.wavelet,
                       rec, obs, w.nt, w.dt, checkpoint_interval=4)
