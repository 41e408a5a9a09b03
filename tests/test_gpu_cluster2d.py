"""The 2-D single-cluster time loop (cluster2d.cu) against the cooperative
grid loop (loop2d_kernel) and the oracle: forward (rolling and saved),
adjoint and gradient, with injections / receivers on band boundaries."""
import os

import numpy as np
import pytest

import oracle_lib as O
from paper_1608_08658_b200 import _lib as L
from paper_1608_08658_b200 import configs, seismic as S

pytestmark = pytest.mark.gpu


def _run(kind, cluster, model, w, src, rec, save=False, resid=None, hist=None):
    os.environ["SFDB200_CLUSTER2D"] = "1" if cluster else "0"
    try:
        nt = w.nt
        if kind == L.FORWARD:
            u = np.zeros(((nt + 1) if save else 3, *model.padded))
            r = np.zeros((nt, rec.npoints))
            p = L.Plan(L.FORWARD, 2, model.padded, w.space_order, nt, w.dt, w.h, src.npoints,
                       rec.npoints, save, 0)
            p.run([u, model.m, model.damp, src.idx, src.w, O._f64(w.wavelet), rec.idx, rec.w, r])
            info = p.info()
            p.close()
            return info, u, r
        if kind == L.ADJOINT:
            v = np.zeros((3, *model.padded))
            s = np.zeros((nt, src.npoints))
            p = L.Plan(L.ADJOINT, 2, model.padded, w.space_order, nt, w.dt, w.h, src.npoints,
                       rec.npoints, False, 0)
            p.run([v, model.m, model.damp, src.idx, src.w, s, rec.idx, rec.w, resid])
            info = p.info()
            p.close()
            return info, v, s
        v = np.zeros((3, *model.padded))
        g = np.zeros(model.padded)
        p = L.Plan(L.GRADIENT, 2, model.padded, w.space_order, nt, w.dt, w.h, 0, rec.npoints,
                   False, 0)
        p.run([v, hist, model.m, model.damp, g, rec.idx, rec.w, resid])
        info = p.info()
        p.close()
        return info, v, g
    finally:
        os.environ.pop("SFDB200_CLUSTER2D", None)


@pytest.fixture(scope="module")
def setup():
    w = configs.cfg1(n=121, nt=302, nbpml=20)
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    rng = np.random.default_rng(4)
    span = (w.interior[0] - 1) * w.h
    src_c = np.array([[300.0, 600.0], [span - 5.0, 10.0]])
    rec_c = rng.uniform(0.0, span, size=(60, 2))
    rec_c[:20, 0] = np.round(rec_c[:20, 0] / w.h) * w.h  # base rows on node rows
    src = S.locate_points(model, src_c)
    rec = S.locate_points(model, rec_c)
    w.wavelet = O._f64(np.repeat(w.wavelet[:, :1], 2, axis=1))
    return w, model, src, rec


def test_forward_cluster_equals_grid_loop_and_oracle(setup):
    w, model, src, rec = setup
    ic, uc, rc = _run(L.FORWARD, True, model, w, src, rec)
    ig, ug, rg = _run(L.FORWARD, False, model, w, src, rec)
    assert ic["cluster2d_ctas"] >= 2 and ig["cluster2d_ctas"] == 0
    assert np.array_equal(uc, ug) and np.array_equal(rc, rg)  # same arithmetic, same order
    uo, ro = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                       src.idx, src.w, w.wavelet, rec.idx, rec.w)
    assert O.rel_l2(uc, uo) <= 1e-5 and O.rel_l2(rc, ro) <= 1e-5
    _, hs, rs = _run(L.FORWARD, True, model, w, src, rec, save=True)
    assert np.array_equal(rs, rc)
    for t in range(w.nt - 3, w.nt):
        assert np.array_equal(hs[t], uc[t % 3])


def test_adjoint_and_gradient_cluster(setup):
    w, model, src, rec = setup
    rng = np.random.default_rng(8)
    resid = O._f64(rng.standard_normal((w.nt, rec.npoints)).astype(np.float32))
    _, vc, sc = _run(L.ADJOINT, True, model, w, src, rec, resid=resid)
    _, vg, sg = _run(L.ADJOINT, False, model, w, src, rec, resid=resid)
    assert np.array_equal(vc, vg) and np.array_equal(sc, sg)
    _, hist, _ = _run(L.FORWARD, True, model, w, src, rec, save=True)
    _, _, gc = _run(L.GRADIENT, True, model, w, src, rec, resid=resid, hist=hist)
    _, _, gg = _run(L.GRADIENT, False, model, w, src, rec, resid=resid, hist=hist)
    assert O.rel_l2(gc, gg) <= 1e-6
    go, _ = O.gradient(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp, hist,
                       rec.idx, rec.w, resid)
    assert O.rel_l2(gc, go) <= 1e-5
