"""The C++ operator mirror (include/sfdb200/seismic.hpp), compiled as a
reference caller would, checked against the oracle."""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu
ROOT = O.ROOT


def test_cpp_operator_api(tmp_path):
    exe = tmp_path / "api_check"
    pkg = os.path.join(ROOT, "paper_1608_08658_b200")
    subprocess.run(["c++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "seismic_api_check.cpp"), "-L", pkg,
                    "-lsfdb200", f"-Wl,-rpath,{pkg}", "-o", str(exe)], check=True)
    res = json.loads(subprocess.run([str(exe), str(tmp_path)], check=True, capture_output=True,
                                    text=True).stdout)
    assert res["refused"] == 1
    rd = lambda n: np.fromfile(tmp_path / f"{n}.bin")  # noqa: E731
    n, nbpml, so, h, nt, dt = 24, 8, 8, 10.0, res["nt"], res["dt"]
    padded, m, damp = O.make_model([n, n, n], h, nbpml, so, rd("m_interior"))
    si, sw = O.locate([n, n, n], h, nbpml, so, [[35.0, 115.5, 117.25]])
    ri, rw = O.locate([n, n, n], h, nbpml, so, rd("rec_coords").reshape(-1, 3))
    wav = rd("wavelet")
    u, r = O.forward(padded, so, h, dt, nt, m, damp, si, sw, wav, ri, rw, save=True)
    assert O.rel_l2(rd("record"), r) <= 1e-5
    assert O.rel_l2(rd("u_hist"), u) <= 1e-5
    resid = rd("residual").reshape(nt, -1)
    g, _ = O.gradient(padded, so, h, dt, nt, m, damp, u, ri, rw, resid)
    assert O.rel_l2(rd("grad"), g) <= 1e-5
    _, s = O.adjoint(padded, so, h, dt, nt, m, damp, si, sw, ri, rw, resid)
    assert O.rel_l2(rd("adj_src"), s) <= 1e-5
