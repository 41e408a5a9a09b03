"""One plan reused across shots, as sfdb200_call's per-descriptor plan cache
reuses it under the reference's operators (an FWI loop calls forward / gradient
once per shot with the same grid and set sizes but new source positions,
receivers, traces and model).  The fused sparse tables are cached by a hash of
their inputs (sparse.cpp upload_sparse): every change must rebuild them, and a
repeated shot must reproduce its first result bit for bit."""
import numpy as np
import pytest

import oracle_lib as O
from paper_1608_08658_b200 import _lib as L
from paper_1608_08658_b200 import configs, seismic as S

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _shot(model, w, rng, nsrc, nrec):
    span = np.array([(n - 1) * w.h for n in w.interior])
    src = S.locate_points(model, 0.2 * span + rng.random((nsrc, len(span))) * 0.6 * span)
    rec = S.locate_points(model, rng.random((nrec, len(span))) * span)
    wav = O._f64((np.asarray(w.wavelet).reshape(w.nt, -1)[:, :1] *
                  (0.5 + rng.random(nsrc))).astype(np.float32))
    return src, rec, wav


def _argv(model, src, rec, wav, nt):
    return [np.zeros((3, *model.padded)), L.f64(model.m), L.f64(model.damp), L.i64(src.idx),
            L.f64(src.w), wav, L.i64(rec.idx), L.f64(rec.w), np.zeros((nt, rec.npoints))]


@pytest.mark.parametrize("so,nd", [(8, 3), (16, 3), (4, 2)])
def test_forward_plan_reused_across_shots(so, nd, monkeypatch):
    # one tiling for every plan: each plan autotunes on its own, and at so >= 10
    # the pair and half-tile mappings round the Laplacian differently (two
    # partial sums vs one), so bitwise comparisons need the same kernel
    monkeypatch.setenv("SFDB200_TILE", "4,2,4,2,1" if so == 16 else "4,2,4,4,1")
    rng = np.random.default_rng(so + nd)
    if nd == 3:
        w = configs.cfg2(n=36, nt=72, nbpml=8, nrec_side=4) if so == 8 else \
            configs.cfg4(so, n=36, nt=72, nbpml=8)
    else:
        w = configs.cfg1(n=90, nt=122, nbpml=12)
    m1 = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    m2 = S.make_model(w.interior, w.h, w.nbpml, w.space_order,
                      configs._round32(np.asarray(w.m_interior) * (1.0 + 0.1 * rng.random(
                          np.asarray(w.m_interior).shape))))
    nsrc, nrec = 2, 9
    shots = [(m1,) + _shot(m1, w, rng, nsrc, nrec), (m2,) + _shot(m2, w, rng, nsrc, nrec),
             (m1,) + _shot(m1, w, rng, nsrc, nrec)]
    # same positions as shot 0 with other weights only / another trace only
    s0 = shots[0]
    shots.append((m1, S.SparsePoints(s0[1].npoints, s0[1].ndim, s0[1].idx, s0[1].w[:, ::-1].copy()),
                  s0[2], s0[3]))
    shots.append((m1, s0[1], s0[2], O._f64((s0[3] * 1.5).astype(np.float32))))

    def fresh(sh):
        model, src, rec, wav = sh
        p = L.Plan(L.FORWARD, nd, model.padded, so, w.nt, w.dt, w.h, nsrc, nrec, False, 0)
        try:
            a = _argv(model, src, rec, wav, w.nt)
            p.run(a)
            return a[0].copy(), a[8].copy()
        finally:
            p.close()

    want = [fresh(sh) for sh in shots]
    p = L.Plan(L.FORWARD, nd, shots[0][0].padded, so, w.nt, w.dt, w.h, nsrc, nrec, False, 0)
    try:
        for k in (0, 1, 2, 3, 4, 0, 1):
            model, src, rec, wav = shots[k]
            a = _argv(model, src, rec, wav, w.nt)
            p.run(a)
            assert np.array_equal(a[0], want[k][0]) and np.array_equal(a[8], want[k][1]), k
    finally:
        p.close()
    model, src, rec, wav = shots[1]
    P = model.padded
    uo, ro = O.forward(P, so, w.h, w.dt, w.nt, model.m, model.damp, src.idx, src.w, wav, rec.idx,
                       rec.w)
    assert O.rel_l2(want[1][0], uo) <= TOL and O.rel_l2(want[1][1], ro) <= TOL


def test_gradient_plan_reused_across_shots(monkeypatch):
    monkeypatch.setenv("SFDB200_TILE", "4,1,4,0,1")
    rng = np.random.default_rng(5)
    w = configs.cfg2(n=30, nt=62, nbpml=8, nrec_side=4)
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    nrec = 12
    shots = []
    for _ in range(3):
        src, rec, wav = _shot(model, w, rng, 1, nrec)
        us, rs = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                           src.idx, src.w, wav, rec.idx, rec.w, save=True)
        resid = O._f64(rng.standard_normal(rs.shape).astype(np.float32))
        shots.append((rec, us, resid))

    def argv(sh):
        rec, us, resid = sh
        return [None, L.f64(us), L.f64(model.m), L.f64(model.damp), np.zeros(model.padded),
                L.i64(rec.idx), L.f64(rec.w), resid]

    def fresh(sh):
        p = L.Plan(L.GRADIENT, 3, model.padded, w.space_order, w.nt, w.dt, w.h, 0, nrec, False, 0)
        try:
            a = argv(sh)
            p.run(a)
            return a[4].copy()
        finally:
            p.close()

    want = [fresh(sh) for sh in shots]
    p = L.Plan(L.GRADIENT, 3, model.padded, w.space_order, w.nt, w.dt, w.h, 0, nrec, False, 0)
    try:
        for k in (0, 1, 2, 0):
            a = argv(shots[k])
            p.run(a)
            assert np.array_equal(a[4], want[k]), k
    finally:
        p.close()
    rec, us, resid = shots[2]
    go, _ = O.gradient(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp, us,
                       rec.idx, rec.w, resid)
    assert O.rel_l2(want[2], go) <= 5e-5


def test_colliding_injection_corners_are_deterministic(monkeypatch):
    """A receiver carpet at the grid spacing shares corners between neighbours
    (cfg3's 200 x 200 carpet): the fused injection sums each cell's entries in
    the reference's (p, c) order and adds the sum once, so the adjoint and the
    gradient are bit-identical from run to run and across z-chunk counts
    (which change the CTA that owns a cell, not the order within the cell)."""
    monkeypatch.setenv("SFDB200_TILE", "4,1,4,0,1")
    rng = np.random.default_rng(9)
    w = configs.cfg2(n=30, nt=62, nbpml=8, nrec_side=4)
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    span = (w.interior[0] - 1) * w.h
    c = 3.3 + np.arange(24) * w.h                      # 24 x 24 carpet, spacing = h
    yy, xx = np.meshgrid(c, c, indexing="ij")
    rec = S.locate_points(model, np.stack([np.full(yy.size, 27.1), yy.ravel(), xx.ravel()], 1))
    src = S.locate_points(model, np.array([[0.5 * span, 0.45 * span, 0.55 * span]]))
    cells = [tuple(i + np.array([(k >> 2) & 1, (k >> 1) & 1, k & 1])) for i in rec.idx for k in range(8)]
    assert len(set(cells)) < len(cells) // 3          # most corners are shared
    wav = O._f64(np.asarray(w.wavelet).reshape(w.nt, -1)[:, :1])
    us, rs = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp, src.idx,
                       src.w, wav, rec.idx, rec.w, save=True)
    resid = O._f64(rng.standard_normal(rs.shape).astype(np.float32))
    rsr = S.ShotRecord(w.nt, w.dt, rec.npoints, resid)
    outs = []
    for zc in ("2", "2", "3", "2"):
        monkeypatch.setenv("SFDB200_ZCHUNKS", zc)
        a = S.adjoint(model, rec, rsr, src, w.nt, w.dt)
        g = S.gradient(model, rec, rsr, us, w.nt, w.dt)
        outs.append((np.asarray(a.v).copy(), np.asarray(a.src_samples.data).copy(),
                     np.asarray(g.grad).copy()))
    for o in outs[1:]:
        for x, y in zip(o, outs[0]):
            assert np.array_equal(x, y)
    vo, so_ = O.adjoint(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp, src.idx,
                        src.w, rec.idx, rec.w, resid)
    go, _ = O.gradient(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp, us,
                       rec.idx, rec.w, resid)
    assert O.rel_l2(outs[0][0], vo) <= TOL and O.rel_l2(outs[0][1], so_) <= TOL
    assert O.rel_l2(outs[0][2], go) <= 5e-5
