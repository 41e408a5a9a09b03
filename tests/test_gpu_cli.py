"""The sfd-compatible driver (cli.py, mirroring proj/tools/sfd.cpp:309-355 run and
:445-515 bench) end to end on the B200, its files compared with what the
UNMODIFIED reference produces for the same experiment: seismic::forward through
oracle/_ref on the configuration sfd.cpp's build_experiment (:117-195) makes,
record.bin / wavefield.bin within rel-L2 1e-5, and the reference's own
load_record reading the driver's record files."""
import json

import numpy as np
import pytest

import oracle_lib as O
from paper_1608_08658_b200 import cli

pytestmark = pytest.mark.gpu

SETS = [["--set", "interior=[40,36,44]", "--set", "nbpml=6", "--set", "nt=180",
         "--set", "receivers=12", "--set", "space_order=8"],
        ["--set", "interior=[90,101]", "--set", "nbpml=12", "--set", "time=0.6",
         "--set", "space_order=4", "--set", "save=true", "--set", "velocity=2000"]]


def _reference_forward(sets):
    patch = cli.build_patch("", [s for s in sets if s != "--set"])
    ex = cli.build_experiment(patch)
    m = ex["model"]
    mi = O._f64(np.full(int(np.prod(m.interior)), 1.0 / float(ex["cfg"]["velocity"]) ** 2))
    save = bool(ex["cfg"]["save"])
    u, rec, _ = O.ref_forward(m.interior, m.h, m.nbpml, m.space_order, mi, ex["src_coords"],
                              ex["trace"].reshape(-1, 1), ex["rec_coords"], ex["nt"], ex["dt"],
                              save=save)
    return ex, u, rec


@pytest.mark.parametrize("case", [0, 1])
def test_cli_run_matches_reference_forward(tmp_path, case):
    out = tmp_path / "run"
    assert cli.main(["--out", str(out)] + SETS[case] + ["run"]) == 0
    ex, u_ref, rec_ref = _reference_forward(SETS[case])
    summary = json.load(open(out / "summary.json"))
    assert summary["passed"] and summary["nt"] == ex["nt"] and summary["dt"] == ex["dt"]
    meta = json.load(open(out / "wavefield.json"))
    slots = ex["nt"] + 1 if ex["cfg"]["save"] else 3
    assert meta == {"shape": [slots, *ex["model"].padded], "halo": ex["model"].halo(),
                    "dtype": "float64", "time_slots": slots}
    u = np.fromfile(out / "wavefield.bin").reshape(u_ref.shape)
    assert O.rel_l2(u, u_ref) <= 1e-5
    rec = np.fromfile(out / "record.bin").reshape(rec_ref.shape)
    assert O.rel_l2(rec, rec_ref) <= 1e-5
    # the reference reads the driver's record files
    data, dt, coords = O.ref_load_record(out / "record")
    assert np.array_equal(data, rec) and dt == ex["dt"]
    assert np.array_equal(coords, np.array(ex["rec_coords"]))


def test_cli_bench_rows(tmp_path):
    """bench writes the reference's roofline-row keys (verify.hpp:110-119) for
    the device run and the end-to-end run, and a summary."""
    out = tmp_path / "bench"
    assert cli.main(["--out", str(out)] + SETS[0] + ["bench"]) == 0
    rows = [json.loads(x) for x in open(out / "bench.jsonl")]
    assert [r["plan"] for r in rows] == ["b200-device", "b200-e2e"]
    for r in rows:
        for k in ("kernel", "flops_per_point", "bytes_per_point", "intensity", "seconds",
                  "gflops", "plan", "blocks", "gpts"):
            assert k in r, k
        assert r["seconds"] > 0 and r["gpts"] > 0 and r["kernel"] == "Forward"
    assert rows[0]["gpts"] >= rows[1]["gpts"]
    s = json.load(open(out / "summary.json"))
    assert s["command"] == "bench" and s["passed"] and s["rows"] == 2
