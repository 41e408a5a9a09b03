"""CPU tests of the B200 backend's host side: the C ABI library loads and
exports every symbol include/sfdb200.h declares; the host helpers mirroring
sfd::seismic are bit-exact with the reference (golden fixtures); the operator
API validates like the reference (std::invalid_argument -> ValueError) before
any device work."""
import os
import re

import numpy as np
import pytest

from paper_1608_08658_b200 import _lib as L
from paper_1608_08658_b200 import configs
from paper_1608_08658_b200 import seismic as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "sfdb200.h")).read()
    return sorted(set(re.findall(r"SFDB200_API\s+[\w\s\*]+?\b(sfdb200_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    names = header_symbols()
    assert len(names) >= 20
    lib = L.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(L.EXPORTS)
    assert b"sm_100a" in lib.sfdb200_version()


def test_host_helpers_bit_exact_with_reference():
    g = np.load(os.path.join(GOLD, "ref_helpers.npz"))
    for so in range(2, 17, 2):
        assert np.array_equal(S.fd_coefficients2(so), g[f"fd2_so{so}"]), so
    mdl = S.make_model([9, 7], 10.0, 5, 4, 1e-6 * np.arange(1, 64))
    assert mdl.padded == list(g["model_padded"])
    assert np.array_equal(mdl.m, g["model_m"]) and np.array_equal(mdl.damp, g["model_damp"])
    assert np.array_equal(S.build_damping(list(g["damp1d_padded"]), 8, 2, 12.5), g["damp1d"])
    m33 = S.make_constant_model([33, 33], 15.0, 10, 4, 1500.0)
    pts = S.locate_points(m33, g["locate_pts"])
    assert np.array_equal(pts.idx, g["locate_idx"]) and np.array_equal(pts.w, g["locate_w"])
    assert np.array_equal(S.ricker(10.0, 0.1, 2001, 1e-4), g["ricker"])
    crit = [S.critical_dt(S.make_constant_model([17, 13], 10.0, 6, so, v))
            for so in (2, 4, 8, 12, 16) for v in (1500.0, 4500.0)]
    assert np.array_equal(np.array(crit), g["crit"])


@pytest.mark.parametrize("name", ["ref_2d_so4.npz", "ref_3d_so8.npz"])
def test_model_and_points_match_reference_fixture(name):
    g = np.load(os.path.join(GOLD, name))
    mdl = S.make_model(list(g["interior"]), float(g["h"]), int(g["nbpml"]), int(g["so"]),
                       g["m_interior"])
    assert np.array_equal(mdl.m, g["m"]) and np.array_equal(mdl.damp, g["damp"])
    assert S.critical_dt(mdl) == float(g["critical_dt"])
    for kind in ("src", "rec"):
        p = S.locate_points(mdl, g[f"{kind}_coords"])
        assert np.array_equal(p.idx, g[f"{kind}_idx"]) and np.array_equal(p.w, g[f"{kind}_w"])


def test_model_validation_mirrors_reference():
    """proj/tests/test_seismic.cpp:28-48."""
    mdl = S.make_model([9, 7], 10.0, 5, 4, 1e-6 * np.arange(1, 64))
    assert mdl.pad() == 7 and mdl.padded == [23, 21] and mdl.cells() == 23 * 21
    at = lambda i, j: mdl.m[i * 21 + j]  # noqa: E731
    mi = 1e-6 * np.arange(1, 64)
    assert at(7, 7) == mi[0] and at(0, 0) == mi[0] and at(0, 10) == mi[3]
    assert at(15, 20) == mi[8 * 7 + 6]
    assert np.array_equal(S.restrict_interior(mdl, mdl.m), mi)
    with pytest.raises(ValueError):
        S.make_model([4], 10.0, 2, 4, np.ones(3))
    with pytest.raises(ValueError):
        S.make_model([4], 10.0, 2, 4, -np.ones(4))
    with pytest.raises(ValueError):
        S.make_constant_model([9, 9], 10.0, 2, 3, 1500.0)


def test_point_location_and_errors():
    """test_seismic.cpp:108-134."""
    m = S.make_constant_model([33, 33], 15.0, 10, 4, 1500.0)
    on = S.locate_points(m, [[60.0, 135.0]])
    assert list(on.idx[0]) == [4 + m.pad(), 9 + m.pad()] and list(on.w[0]) == [1, 0, 0, 0]
    mid = S.locate_points(m, [[67.5, 142.5]])
    assert np.allclose(mid.w, 0.25, rtol=1e-14)
    rng = np.random.default_rng(11)
    p = S.locate_points(m, rng.uniform(0.0, 480.0, size=(500, 2)))
    assert np.all(p.w >= 0) and np.all(p.w <= 1)
    assert np.all(np.abs(p.w.sum(axis=1) - 1.0) <= 1e-15)
    for bad in ([[-1.0, 10.0]], [[10.0, 480.1]], [[10.0]]):
        with pytest.raises(ValueError):
            S.locate_points(m, bad)


def test_operators_refuse_unstable_or_malformed_input_before_device_work():
    """test_seismic.cpp:399-412 (raised on the host, no GPU needed)."""
    m = S.make_constant_model([33, 33], 15.0, 10, 4, 1500.0)
    dt = 1.01 * S.critical_dt(m)
    src = S.locate_points(m, [[240.0, 240.0]])
    rec = S.locate_points(m, [[100.0, 380.0]])
    with pytest.raises(ValueError, match="CFL"):
        S.forward(m, src, np.zeros(40), rec, 40, dt, False)
    with pytest.raises(ValueError):
        S.adjoint(m, rec, S.zero_record(40, dt, 1), src, 40, dt)
    ok = 0.9 * S.critical_dt(m)
    with pytest.raises(ValueError):
        S.forward(m, src, np.zeros(10), rec, 40, ok, False)
    with pytest.raises(ValueError):
        S.adjoint(m, rec, S.zero_record(40, ok, 2), src, 40, ok)
    with pytest.raises(ValueError):
        S.gradient(m, rec, S.zero_record(40, ok, 1), np.zeros(10), 40, ok)


def test_objective_and_interior_helpers():
    """test_seismic.cpp:362-380."""
    a = S.zero_record(4, 0.001, 2)
    b = S.zero_record(4, 0.001, 2)
    a.data = (np.arange(8) * 0.5).reshape(4, 2)
    assert S.objective(a, a) == 0.0
    sq = float((a.data ** 2).sum())
    assert S.objective(a, b) == pytest.approx(0.5 * sq, rel=1e-15)
    phi, resid = S.objective(a, b, want_residual=True)
    assert np.array_equal(resid.data, a.data)
    with pytest.raises(ValueError):
        S.objective(a, S.zero_record(3, 0.001, 2))
    m = S.make_model([9, 7], 10.0, 5, 4, 1e-6 * np.arange(1, 64))
    f = np.zeros(m.cells())
    S.add_interior(m, np.ones(63), 2.0, f)
    assert f.sum() == 126.0 and np.array_equal(S.restrict_interior(m, f), np.full(63, 2.0))


def test_model_and_record_files_round_trip(tmp_path):
    mi = 1e-6 * (1 + np.arange(11 * 9))
    m = S.make_model([11, 9], 12.0, 4, 4, mi)
    S.save_model(m, str(tmp_path / "model"))
    m2 = S.load_model(str(tmp_path / "model"), 4)
    assert np.array_equal(m2.m, m.m) and m2.interior == m.interior and m2.h == m.h
    r = S.zero_record(5, 0.002, 3)
    r.data = np.arange(15.0).reshape(5, 3)
    coords = [[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]]
    S.save_record(r, coords, str(tmp_path / "rec"))
    r2, c2 = S.load_record(str(tmp_path / "rec"))
    assert np.array_equal(r2.data, r.data) and c2 == coords and r2.dt == r.dt


def test_synthetic_configs_have_the_baseline_shapes():
    w1 = configs.cfg1(n=41, nt=12)
    assert w1.ndim == 2 and w1.space_order == 4 and len(w1.rec_coords) == 101
    w2 = configs.cfg2(n=24, nt=12, nrec_side=8)
    assert w2.padded == [24 + 88] * 3 and len(w2.rec_coords) == 64
    assert w2.m_interior.min() == pytest.approx(1 / 4500.0 ** 2, rel=1e-6)
    assert np.array_equal(w2.m_interior, w2.m_interior.astype(np.float32).astype(np.float64))
    w5 = configs.cfg4(16, n=16, nt=12, nbpml=4)
    m = S.make_model(w5.interior, w5.h, w5.nbpml, 16, w5.m_interior)
    assert w5.dt <= S.critical_dt(m)


def test_cli_config_patch_and_refusal(tmp_path):
    """sfd.cpp:58-78 (--set) and :555-565 (refusal -> exit 2 with a summary)."""
    from paper_1608_08658_b200 import cli
    p = cli.build_patch("", ["interior=[9,9]", "h=12.5", "source.0=3", "kernel=adjoint"])
    assert p == {"interior": [9, 9], "h": 12.5, "source": {"0": 3}, "kernel": "adjoint"}
    ex = cli.build_experiment({"interior": [20, 24], "nbpml": 4, "space_order": 4,
                               "receivers": 3, "time": 0.05})
    assert ex["rec"].npoints == 3 and ex["nt"] >= 4
    assert ex["dt"] == 0.9 * S.critical_dt(ex["model"])
    rc = cli.main(["--out", str(tmp_path), "--set", "dt=1.0", "--set", "interior=[9,9]",
                   "run"])
    assert rc == 2
    import json as _json
    summ = _json.load(open(tmp_path / "summary.json"))
    assert summ["command"] == "error" and "CFL" in summ["error"]


def test_operators_fail_loudly_without_the_cuda_library(monkeypatch, tmp_path):
    """No CPU fallback: with libsfdb200.so absent the operators raise instead of
    computing anything, and on a host without a GPU the device plan refuses."""
    m = S.make_constant_model([17, 17], 15.0, 4, 4, 1500.0)
    dt = 0.5 * S.critical_dt(m)
    src = S.locate_points(m, [[120.0, 120.0]])
    rec = S.locate_points(m, [[60.0, 200.0]])
    wav = S.ricker(20.0, 0.05, 12, dt)
    monkeypatch.setattr(L, "LIB_PATH", str(tmp_path / "libsfdb200.so"))
    monkeypatch.setattr(L, "_lib", None)
    with pytest.raises(ImportError, match="missing"):
        S.forward(m, src, wav, rec, 12, dt, False)
    monkeypatch.undo()
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(L.SfdError):
            S.forward(m, src, wav, rec, 12, dt, False)


def test_host_separable_damping_check():
    """The upload's host check (hostio.cpp host_sep_damp) accepts the
    reference's build_damping fields (golden fixture) with profiles equal to
    the per-axis minima, and declines fields the device check must decide."""
    g = np.load(os.path.join(GOLD, "ref_3d_so8.npz"))
    mdl = S.make_model(list(g["interior"]), float(g["h"]), int(g["nbpml"]), int(g["so"]),
                       g["m_interior"])
    pz, py, px = mdl.padded
    d = np.ascontiguousarray(g["damp"], dtype=np.float64)

    def check(field):
        prof = np.full(pz + py + px, np.nan)
        rc = L.lib().sfdb200_damp_separable(L.dptr(field), pz, py, px, L.dptr(prof))
        assert rc in (0, 1)
        return rc == 1, prof

    ok, prof = check(d)
    assert ok
    cube = d.reshape(pz, py, px)
    mins = np.concatenate([cube.min(axis=(1, 2)), cube.min(axis=(0, 2)), cube.min(axis=(0, 1))])
    assert np.array_equal(prof, mins)
    rebuilt = np.maximum(np.maximum(prof[:pz, None, None], prof[pz:pz + py][None, :, None]),
                         prof[pz + py:][None, None, :])
    assert np.array_equal(rebuilt.reshape(-1), d)
    for bad in (1e-3, -1e-9, np.nan):  # perturbed, negative, non-finite cell
        e = d.copy()
        e[e.size // 2 + 5] = bad
        assert not check(e)[0]
    neg0 = d.copy()
    neg0[(pz // 2 * py + py // 2) * px + px // 2] = -0.0  # equal to 0.0, as on the device
    ok, prof0 = check(neg0)
    assert ok and not np.signbit(prof0).any() and np.array_equal(prof0, prof)
    assert L.lib().sfdb200_damp_separable(L.dptr(d), 0, py, px, L.dptr(prof)) == L.EINVAL

