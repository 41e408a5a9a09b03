"""Two-way file-format interop with the UNMODIFIED reference (SURVEY.md
section 8(f) row 4) and the objective's bitwise agreement.

Files written by the reference's own save_model / save_record
(seismic.cpp:557-614) and dump_grid (runtime.cpp:425-440), called through
oracle/_ref, are read by this repo's seismic.load_model / load_record, and
files this repo writes (seismic.save_model / save_record, cli.dump_grid) are
read by the reference's load_model / load_record.  Raw blobs must be
byte-identical and the JSON sidecars must parse to the same objects."""
import json

import numpy as np
import pytest

import oracle_lib as O
from paper_1608_08658_b200 import cli, seismic as S

pytestmark = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")


def _mi(shape, seed=3):
    rng = np.random.default_rng(seed)
    v = 1500.0 + 3000.0 * rng.random(int(np.prod(shape)))
    return 1.0 / v ** 2


@pytest.mark.parametrize("shape", [[13, 11], [9, 12, 10]])
def test_model_files_both_ways(tmp_path, shape):
    mi = _mi(shape)
    so, nbpml, h = 8, 5, 12.5
    # reference writes -> repo reads
    O.ref_save_model(tmp_path / "ref_model", shape, h, nbpml, so, mi)
    ours = S.load_model(str(tmp_path / "ref_model"), so)
    interior, rh, rn, m_ref, damp_ref = O.ref_load_model(tmp_path / "ref_model", so)
    assert ours.interior == list(interior) and ours.h == rh and ours.nbpml == rn
    assert np.array_equal(ours.m, m_ref.ravel()) and np.array_equal(ours.damp, damp_ref.ravel())
    # repo writes -> reference reads
    model = S.make_model(shape, h, nbpml, so, mi)
    S.save_model(model, str(tmp_path / "our_model"))
    interior, rh, rn, m2, d2 = O.ref_load_model(tmp_path / "our_model", so)
    assert list(interior) == shape and rh == h and rn == nbpml
    assert np.array_equal(m2.ravel(), model.m) and np.array_equal(d2.ravel(), model.damp)
    # the blobs are the same bytes, the headers the same objects
    assert (tmp_path / "ref_model.bin").read_bytes() == (tmp_path / "our_model.bin").read_bytes()
    assert json.loads((tmp_path / "ref_model.json").read_text()) == \
        json.loads((tmp_path / "our_model.json").read_text())


def test_record_files_both_ways(tmp_path):
    rng = np.random.default_rng(5)
    nt, n = 37, 6
    data = rng.standard_normal((nt, n))
    coords = rng.uniform(0.0, 500.0, size=(n, 3))
    O.ref_save_record(tmp_path / "ref_rec", data, 7.5e-4, coords)
    rec, c = S.load_record(str(tmp_path / "ref_rec"))
    assert rec.nt == nt and rec.npoints == n and rec.dt == 7.5e-4
    assert np.array_equal(rec.data, data) and np.array_equal(np.array(c), coords)
    S.save_record(S.ShotRecord(nt, 7.5e-4, n, data), coords.tolist(), str(tmp_path / "our_rec"))
    d2, dt2, c2 = O.ref_load_record(tmp_path / "our_rec")
    assert np.array_equal(d2, data) and dt2 == 7.5e-4 and np.array_equal(c2, coords)
    assert (tmp_path / "ref_rec.bin").read_bytes() == (tmp_path / "our_rec.bin").read_bytes()
    assert json.loads((tmp_path / "ref_rec.json").read_text()) == \
        json.loads((tmp_path / "our_rec.json").read_text())


def test_dump_grid_matches_reference(tmp_path):
    """cli.dump_grid (the CLI's wavefield files) against runtime::dump_grid."""
    rng = np.random.default_rng(6)
    u = rng.standard_normal((3, 10, 9, 11))
    O.ref_dump_grid(tmp_path / "ref_grid", u, 4, 3)
    cli.dump_grid(u, u.shape, 4, 3, str(tmp_path / "our_grid"))
    assert (tmp_path / "ref_grid.bin").read_bytes() == (tmp_path / "our_grid.bin").read_bytes()
    assert json.loads((tmp_path / "ref_grid.json").read_text()) == \
        json.loads((tmp_path / "our_grid.json").read_text())


def test_objective_bitwise_with_reference():
    """seismic.objective (host C, element order) equals seismic::objective bit for
    bit, residual included, on a cfg2-sized slice of a record."""
    rng = np.random.default_rng(7)
    syn = rng.standard_normal(3_000_001)
    obs = syn + 1e-3 * rng.standard_normal(syn.size)
    phi_ref, res_ref = O.ref_objective(syn, obs)
    a = S.ShotRecord(1, 1.0, syn.size, syn.reshape(1, -1))
    b = S.ShotRecord(1, 1.0, syn.size, obs.reshape(1, -1))
    phi, res = S.objective(a, b, want_residual=True)
    assert phi == phi_ref
    assert np.array_equal(res.data.ravel(), res_ref)
    assert S.objective(a, b) == phi_ref
