"""Every tiling variant the autotuner may pick (plan.cu sweep_variants), forced
through SFDB200_TILE, against the oracle: forward at so 8 / 12 / 16 and the
gradient kernel at so 8 (GRAD instantiations)."""
import os

import numpy as np
import pytest

import oracle_lib as O
from paper_1608_08658_b200 import configs, seismic as S

pytestmark = pytest.mark.gpu
TOL = 1e-5

# "by,ny,stages,rot,pair" (sweep3d.cuh launch3d_r)
LOW = ["4,2,3,0,1", "4,2,4,1,1", "4,2,3,1,1", "4,2,4,0,1", "4,2,3,1,0", "4,1,4,1,0", "8,2,3,1,1",
       "4,2,4,4,1", "4,2,4,3,1", "4,2,4,2,1", "4,2,5,0,1", "4,2,5,5,1"]
HIGH = ["4,2,4,4,1", "4,2,4,2,1", "4,2,4,8,1", "4,2,4,0,1", "4,2,3,0,1", "8,2,3,1,1",
        "4,1,4,0,1", "4,1,4,1,0", "4,1,3,1,0", "4,2,5,0,1", "4,2,5,5,1"]


def _forced(tile):
    os.environ["SFDB200_TILE"] = tile


@pytest.fixture(autouse=True)
def _clean_env():
    yield
    os.environ.pop("SFDB200_TILE", None)


@pytest.mark.parametrize("so,tile", [(8, t) for t in LOW] + [(12, t) for t in HIGH] +
                         [(16, t) for t in HIGH])
def test_forward_variant(so, tile):
    w = configs.cfg4(so, n=36, nt=82, nbpml=8) if so != 8 else \
        configs.cfg2(n=36, nt=82, nbpml=8, nrec_side=8)
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    src = S.locate_points(model, w.src_coords)
    rec = S.locate_points(model, w.rec_coords)
    _forced(tile)
    f = S.forward(model, src, w.wavelet, rec, w.nt, w.dt, False)
    u, r = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                     src.idx, src.w, w.wavelet, rec.idx, rec.w)
    assert O.rel_l2(f.u, u) <= TOL, tile
    if rec.npoints:
        assert O.rel_l2(f.record.data, r) <= TOL, tile


@pytest.mark.parametrize("tile", LOW)
def test_gradient_variant(tile):
    w = configs.cfg2(n=30, nt=102, nbpml=8, nrec_side=8)
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    src = S.locate_points(model, w.src_coords)
    rec = S.locate_points(model, w.rec_coords)
    u, r = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                     src.idx, src.w, w.wavelet, rec.idx, rec.w, save=True)
    resid = O._f64(np.random.default_rng(2).standard_normal(r.shape).astype(np.float32))
    _forced(tile)
    g = S.gradient(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), u, w.nt, w.dt)
    go, _ = O.gradient(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp, u,
                       rec.idx, rec.w, resid)
    assert O.rel_l2(g.grad, go) <= TOL, tile


@pytest.mark.parametrize("tile,ctas,zc", [("4,2,4,4,1", 3, 3), ("4,2,4,1,1", 5, 3), ("4,2,4,0,1", 7, 2),
                                          ("4,2,3,3,1", 2, 3), ("4,2,5,5,1", 4, 2), ("4,2,4,4,1", 1, 1)])
def test_persistent_multi_item(tile, ctas, zc):
    """Few persistent CTAs, each walking many (tile, z chunk) items with the
    TMA ring running across items (skip stages, ring-staged queue prologue,
    per-item injection): forward and gradient against the oracle."""
    os.environ["SFDB200_CTAS"] = str(ctas)
    os.environ["SFDB200_ZCHUNKS"] = str(zc)
    try:
        w = configs.cfg2(n=30, nt=62, nbpml=8, nrec_side=7)
        model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
        src = S.locate_points(model, w.src_coords)
        rec = S.locate_points(model, w.rec_coords)
        _forced(tile)
        f = S.forward(model, src, w.wavelet, rec, w.nt, w.dt, False)
        u, r = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                         src.idx, src.w, w.wavelet, rec.idx, rec.w)
        assert O.rel_l2(f.u, u) <= TOL and O.rel_l2(f.record.data, r) <= TOL
        us, rs = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                           src.idx, src.w, w.wavelet, rec.idx, rec.w, save=True)
        resid = O._f64(np.random.default_rng(3).standard_normal(rs.shape).astype(np.float32))
        g = S.gradient(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), us, w.nt, w.dt)
        go, _ = O.gradient(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp, us,
                           rec.idx, rec.w, resid)
        assert O.rel_l2(g.grad, go) <= TOL
    finally:
        os.environ.pop("SFDB200_CTAS", None)
        os.environ.pop("SFDB200_ZCHUNKS", None)


@pytest.mark.parametrize("group,zc,so", [(3, 3, 8), (5, 4, 8), (7, 2, 16), (2, 2, 16)])
def test_grouped_item_order(group, zc, so):
    """The grouped item order (SweepArgs::group: tiles in groups of the
    resident slots, every z chunk of a group in turn, all streaming up), forced
    on a small grid with a small group size: forward (bitwise equal to the
    tile-major order, the same arithmetic per point) and gradient."""
    from paper_1608_08658_b200 import _lib as L
    w = configs.cfg2(n=40, nt=62, nbpml=8, nrec_side=7) if so == 8 else \
        configs.cfg4(so, n=40, nt=62, nbpml=8)
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    src = S.locate_points(model, w.src_coords)
    rec = S.locate_points(model, w.rec_coords)
    os.environ["SFDB200_ZCHUNKS"] = str(zc)
    outs = []
    try:
        for g in (str(group), "0"):
            os.environ["SFDB200_GROUP"] = g
            _forced("4,2,4,4,1" if so == 8 else "4,2,4,2,1")
            f = S.forward(model, src, w.wavelet, rec, w.nt, w.dt, False)
            outs.append((f.u, f.record.data))
        assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
        u, r = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                         src.idx, src.w, w.wavelet, rec.idx, rec.w)
        assert O.rel_l2(outs[0][0], u) <= TOL and O.rel_l2(outs[0][1], r) <= TOL
        if so == 8:
            os.environ["SFDB200_GROUP"] = str(group)
            us, rs = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m,
                               model.damp, src.idx, src.w, w.wavelet, rec.idx, rec.w, save=True)
            resid = O._f64(np.random.default_rng(3).standard_normal(rs.shape).astype(np.float32))
            gr = S.gradient(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), us, w.nt,
                            w.dt)
            go, _ = O.gradient(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                               us, rec.idx, rec.w, resid)
            assert O.rel_l2(gr.grad, go) <= TOL
    finally:
        os.environ.pop("SFDB200_ZCHUNKS", None)
        os.environ.pop("SFDB200_GROUP", None)


@pytest.mark.parametrize("so,zc", [(8, 3), (16, 2), (4, 4)])
def test_dynamic_persistent_items(so, zc):
    """Dynamic persistent sweeps (SweepConfig::ctas = -2: one CTA per resident
    slot taking (tile, z chunk) items from a counter, the item index staged
    with the item's first plane, an end-of-work stage): forward bitwise equal to
    one CTA per item, gradient against the oracle."""
    w = configs.cfg2(n=40, nt=62, nbpml=8, nrec_side=7) if so == 8 else \
        configs.cfg4(so, n=40, nt=62, nbpml=8)
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    src = S.locate_points(model, w.src_coords)
    rec = S.locate_points(model, w.rec_coords)
    os.environ["SFDB200_ZCHUNKS"] = str(zc)
    outs = []
    try:
        for ctas in ("-2", "0"):
            os.environ["SFDB200_CTAS"] = ctas
            _forced("4,2,4,4,1" if so != 16 else "4,2,4,2,1")
            f = S.forward(model, src, w.wavelet, rec, w.nt, w.dt, False)
            outs.append((f.u, f.record.data))
        assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
        u, r = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                         src.idx, src.w, w.wavelet, rec.idx, rec.w)
        assert O.rel_l2(outs[0][0], u) <= TOL and O.rel_l2(outs[0][1], r) <= TOL
        if so == 8:
            os.environ["SFDB200_CTAS"] = "-2"
            us, rs = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m,
                               model.damp, src.idx, src.w, w.wavelet, rec.idx, rec.w, save=True)
            resid = O._f64(np.random.default_rng(3).standard_normal(rs.shape).astype(np.float32))
            g = S.gradient(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), us, w.nt, w.dt)
            go, _ = O.gradient(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                               us, rec.idx, rec.w, resid)
            assert O.rel_l2(g.grad, go) <= TOL
    finally:
        os.environ.pop("SFDB200_ZCHUNKS", None)
        os.environ.pop("SFDB200_CTAS", None)
