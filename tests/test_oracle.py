"""CPU tests: pin the oracle (C restatement, oracle/sfd_oracle.c) against the
reference's own outputs (golden fixtures made by tests/golden/make_golden.py
from the unmodified reference build) and its frozen known answers."""
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle_lib as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


def test_fd2_frozen_reference_weights():
    """Known answers of proj/tests/test_fd.cpp:22-65 (second derivative)."""
    assert list(O.fd2(2)) == [1.0, -2.0, 1.0]
    w4 = O.fd2(4)
    assert list(w4) == [float(Fraction(-1, 12)), float(Fraction(4, 3)), -2.5,
                        float(Fraction(4, 3)), float(Fraction(-1, 12))]
    w14 = O.fd2(14)
    assert w14[7] == float(Fraction(-266681, 88200))
    assert w14[8] == float(Fraction(7, 4))
    assert w14[9] == float(Fraction(-7, 24))
    assert w14[10] == float(Fraction(7, 108))
    assert w14[11] == float(Fraction(-7, 528))


def test_fd2_matches_reference_and_moments():
    g = load("ref_helpers.npz")
    for so in range(2, 17, 2):
        w = O.fd2(so)
        assert np.array_equal(w, g[f"fd2_so{so}"]), so
        k = np.arange(-so // 2, so // 2 + 1, dtype=np.float64)
        # exact second-derivative moments: sum w = 0, sum w k^2 = 2, odd moments 0
        assert abs(w.sum()) < 1e-12 and abs((w * k * k).sum() - 2.0) < 1e-12
        for p in range(4, so + 1, 2):
            assert abs((w * k ** p).sum()) < 1e-6 * float(np.abs(w * k ** p).sum())


def test_model_damping_locate_ricker_critical_dt_bit_exact():
    g = load("ref_helpers.npz")
    padded, m, damp = O.make_model([9, 7], 10.0, 5, 4, 1e-6 * np.arange(1, 64))
    assert list(padded) == list(g["model_padded"])
    assert np.array_equal(m, g["model_m"]) and np.array_equal(damp, g["model_damp"])
    _, _, d1 = O.make_model([8], 12.5, 8, 4, np.full(8, 1e-7))
    assert np.array_equal(d1, g["damp1d"])
    idx, w = O.locate([33, 33], 15.0, 10, 4, g["locate_pts"])
    assert np.array_equal(idx, g["locate_idx"]) and np.array_equal(w, g["locate_w"])
    assert np.array_equal(O.ricker(10.0, 0.1, 2001, 1e-4), g["ricker"])
    crit = [O.critical_dt(2, 10.0, so, 1 / v ** 2) for so in (2, 4, 8, 12, 16)
            for v in (1500.0, 4500.0)]
    assert np.array_equal(np.array(crit), g["crit"])


def test_damping_profile_properties():
    """proj/tests/test_seismic.cpp:50-75: taper shape, halo replication."""
    nbpml, halo, h = 8, 2, 12.5
    _, _, damp = O.make_model([8], h, nbpml, 4, np.full(8, 1e-7))
    c = 1.5 * np.log(1000.0) / (nbpml * h)
    assert damp[halo] == pytest.approx(c, rel=1e-12)
    assert damp[0] == damp[halo]
    assert np.all(damp[halo + nbpml: len(damp) - halo - nbpml] == 0.0)
    assert np.all(np.diff(damp[halo: halo + nbpml + 1]) < 0)


@pytest.mark.parametrize("name", ["ref_2d_so4.npz", "ref_3d_so8.npz"])
def test_oracle_operators_match_reference(name):
    g = load(name)
    interior, h, nbpml, so = list(g["interior"]), float(g["h"]), int(g["nbpml"]), int(g["so"])
    nt, dt = int(g["nt"]), float(g["dt"])
    padded, m, damp = O.make_model(interior, h, nbpml, so, g["m_interior"])
    assert np.array_equal(m, g["m"]) and np.array_equal(damp, g["damp"])
    si, sw = O.locate(interior, h, nbpml, so, g["src_coords"])
    ri, rw = O.locate(interior, h, nbpml, so, g["rec_coords"])
    assert np.array_equal(si, g["src_idx"]) and np.array_equal(ri, g["rec_idx"])
    assert np.array_equal(sw, g["src_w"]) and np.array_equal(rw, g["rec_w"])
    assert O.critical_dt(len(interior), h, so, m.min()) == float(g["critical_dt"])
    u, r = O.forward(padded, so, h, dt, nt, m, damp, si, sw, g["wavelet"], ri, rw)
    assert O.rel_l2(r, g["rec"]) < 1e-12
    if "u" in g:
        assert O.rel_l2(u, g["u"]) < 1e-12
    else:
        assert O.rel_l2(u[(nt - 1) % 3], g["u_last"]) < 1e-12
    v, s = O.adjoint(padded, so, h, dt, nt, m, damp, si, sw, ri, rw, g["residual"])
    assert O.rel_l2(s, g["src_samples"]) < 1e-12
    if "v" in g:
        assert O.rel_l2(v, g["v"]) < 1e-12
    else:
        assert O.rel_l2(v[2 % 3], g["v_last"]) < 1e-12
    uh, rh = O.forward(padded, so, h, dt, nt, m, damp, si, sw, g["wavelet"], ri, rw, save=True)
    if "rec_saved" in g:
        assert O.rel_l2(rh, g["rec_saved"]) < 1e-12
        assert O.rel_l2(uh[nt - 3:], g["u_hist_tail"]) < 1e-12
    gr, _ = O.gradient(padded, so, h, dt, nt, m, damp, uh, ri, rw, g["residual"])
    assert O.rel_l2(gr, g["grad"]) < 1e-11


def test_saved_and_rolling_agree_and_zero_source_is_silent():
    """test_seismic.cpp:173-188 and :220-241 on the oracle."""
    g = load("ref_2d_so4.npz")
    interior, h, nbpml, so = list(g["interior"]), float(g["h"]), int(g["nbpml"]), int(g["so"])
    nt, dt = int(g["nt"]), float(g["dt"])
    padded, m, damp = O.make_model(interior, h, nbpml, so, g["m_interior"])
    si, sw = O.locate(interior, h, nbpml, so, g["src_coords"])
    ri, rw = O.locate(interior, h, nbpml, so, g["rec_coords"])
    u, r = O.forward(padded, so, h, dt, nt, m, damp, si, sw, g["wavelet"], ri, rw)
    uh, rh = O.forward(padded, so, h, dt, nt, m, damp, si, sw, g["wavelet"], ri, rw, save=True)
    assert np.array_equal(r, rh)
    for t in range(nt - 3, nt):
        assert np.array_equal(uh[t], u[t % 3])
    z, rz = O.forward(padded, so, h, dt, nt, m, damp, si, sw, np.zeros(nt), ri, rw)
    assert not z.any() and not rz.any()


def test_oracle_adjoint_dot_product():
    """verify.cpp:123-177: <F x, y> = <x, F^T y> to 1e-10 in fp64."""
    g = load("ref_2d_so4.npz")
    interior, h, nbpml, so = list(g["interior"]), float(g["h"]), int(g["nbpml"]), int(g["so"])
    nt, dt = int(g["nt"]), float(g["dt"])
    padded, m, damp = O.make_model(interior, h, nbpml, so, g["m_interior"])
    si, sw = O.locate(interior, h, nbpml, so, g["src_coords"])
    ri, rw = O.locate(interior, h, nbpml, so, g["rec_coords"])
    rng = np.random.default_rng(1)
    x = rng.standard_normal(nt)
    y = rng.standard_normal((nt, len(ri)))
    _, r = O.forward(padded, so, h, dt, nt, m, damp, si, sw, x, ri, rw)
    _, s = O.adjoint(padded, so, h, dt, nt, m, damp, si, sw, ri, rw, y)
    a, b = float((r * y).sum()), float((x[:, None] * s).sum())
    assert abs(a - b) / abs(a) < 1e-10
