"""The B200 backend under the reference's UNMODIFIED operator API.

Runs oracle/_ref/ref_dropin (tests/cpp/ref_dropin.cpp, built against the
unmodified reference library): sfd::seismic::forward / adjoint / gradient and
sfd::verify::adjoint_test, each once with the reference's generic preset (its
own OpenMP C, the oracle) and once with sfdb200::stencilfd_preset, through
the reference's runtime::compile_and_load / KernelArgs / runtime::run
(runtime.cpp:177-250,335-353, seismic.cpp:333-496).  Every output within
rel-L2 1e-5; the descriptors desc_of(KernelIR)
builds equal the ones the JIT driver reads back."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_dropin")

pytestmark = pytest.mark.gpu


def test_reference_operators_through_the_b200_preset(tmp_path):
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/ref_dropin missing: run __graft_entry__.build() where "
                    "/root/reference exists (it travels with the snapshot)")
    env = dict(os.environ, STENCILFD_CACHE_DIR=str(tmp_path), OMP_PROC_BIND="false")
    out = subprocess.run([BIN, ROOT], capture_output=True, text=True, env=env, timeout=1200)
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    log = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(log):
        with open(os.path.join(log, "ref_dropin.jsonl"), "w") as f:
            f.write(out.stdout + out.stderr)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    checks = [x for x in lines if "check" in x]
    assert len(checks) >= 30 and all(x["ok"] for x in checks)
    assert lines[-1] == {"failures": 0}
