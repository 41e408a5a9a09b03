"""The debug build (libsfdb200_debug.so, -DSFDB200_DEBUG): every global access
the 3-D sweep, its fused sparse work, the P2P peer stores and the 2-D loop make
is checked against the row it addresses (csrc/kernels.cuh SFDB_CHECK); a
failed check is recorded, the access skipped, and the plan fails at download.
This stands in for compute-sanitizer, which is closed on this GPU pool.  The
full -m gpu suite is also run against this build once per round
(SFDB200_LIBRARY=debug, log in profiles/)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import numpy as np
from paper_1608_08658_b200 import _lib as L, configs, seismic as S
assert "debug" in L.lib().sfdb200_version().decode()
w = configs.cfg2(n=24, nt=40, nbpml=6, nrec_side=4)
model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
src, rec = S.locate_points(model, w.src_coords), S.locate_points(model, w.rec_coords)
p = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
           rec.npoints, False, 0)
argv = [np.zeros((3, *model.padded)), model.m, model.damp, src.idx, src.w, w.wavelet,
        rec.idx, rec.w, np.zeros((w.nt, rec.npoints))]
try:
    p.run(argv)
    print("RESULT ok")
except L.SfdError as e:
    print("RESULT error", e.code, e)
"""


def _run(fault, **extra):
    lib = os.path.join(ROOT, "paper_1608_08658_b200", "libsfdb200_debug.so")
    if not os.path.exists(lib):
        pytest.fail("libsfdb200_debug.so missing: make -C paper_1608_08658_b200/csrc debug")
    env = dict(os.environ, SFDB200_LIBRARY="debug", SFDB200_DEBUG_FAULT=str(fault), **extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], capture_output=True, text=True,
                         env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return [x for x in out.stdout.splitlines() if x.startswith("RESULT")][-1]


def test_debug_build_runs_clean():
    assert _run(0) == "RESULT ok"


def test_debug_build_catches_an_out_of_row_access():
    r = _run(1)
    assert r.startswith("RESULT error 2") and "receiver corner outside the sampled row" in r


@pytest.mark.parametrize("group,zc", [(2, 3), (2, 2)])
def test_grouped_order_injects_from_the_owning_item(group, zc):
    """Under the grouped item order the launch position of an item differs from
    its index in the fused injection table (tile + tiles * chunk).  An item must
    add only the corners it stored itself: an atomic from another CTA races with
    the owner's plain store in the same launch and can lose the injection (seen
    as run-to-run differences at 512^3, where the grouped order is the default).
    The debug build checks every fused injection against the injecting item's
    box (kDbgInjectOwner); a build that indexes the table by launch position
    fails this case with "fused injection into a cell another item stores"."""
    assert _run(0, SFDB200_GROUP=str(group), SFDB200_ZCHUNKS=str(zc),
                SFDB200_TILE="4,2,4,4,1") == "RESULT ok"
