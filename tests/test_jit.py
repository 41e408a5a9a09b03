"""CPU tests of bin/sfdb200-jit, the driver that puts the B200 backend under the
reference's UNMODIFIED operators (csrc/jit.cpp).

The kernel sources come from the reference's own codegen::generate
(oracle/_ref, build_*_ir + generate, seismic.cpp:241-331, codegen.cpp:579-629);
the compile command is the one runtime::compile_and_load runs
(runtime.cpp:213-214: `cc -shared -fPIC <preset flags> -o x.so x.c -lm`)."""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle_lib as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1608_08658_b200")
JIT = os.path.join(PKG, "bin", "sfdb200-jit")

pytestmark = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")


def _model(ndim, so):
    interior = [7, 9, 8][:ndim] if ndim == 3 else [11, 9]
    m = np.full(int(np.prod(interior)), 1.0 / 1800.0 ** 2)
    return interior, 7.5, 3, m


def _source(kind, ndim, so, nsrc=2, nrec=3, nt=17, dt=3.7e-4, save=False, plan=0):
    interior, h, nbpml, m = _model(ndim, so)
    return O.ref_generate(kind, interior, h, nbpml, so, m, nsrc, nrec, nt, dt, save, plan)


def _describe(tmp_path, src):
    path = tmp_path / "k.c"
    path.write_text(src)
    out = subprocess.run([JIT, "--describe", str(path)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout)


@pytest.mark.parametrize("ndim", [2, 3])
@pytest.mark.parametrize("so", [2, 4, 8, 12, 16])
@pytest.mark.parametrize("kind,save", [(0, False), (0, True), (1, False), (2, False)])
@pytest.mark.parametrize("plan", [0, 1, 2])
def test_descriptor_read_back(tmp_path, ndim, so, kind, save, plan):
    """Every field the generated source bakes in comes back: kind, extents,
    order, nt, set sizes, save; dt and h to a few ulp (printed literals)."""
    dt = 3.7e-4
    d = _describe(tmp_path, _source(kind, ndim, so, dt=dt, save=save, plan=plan))
    interior, h, nbpml, _ = _model(ndim, so)
    padded = [n + 2 * (nbpml + so // 2) for n in interior]
    assert d["name"] == ["Forward", "Adjoint", "Gradient"][kind]
    assert d["kind"] == kind and d["ndim"] == ndim and d["padded"][:ndim] == padded
    assert d["space_order"] == so and d["nt"] == 17 and d["save"] == int(save)
    assert d["nrec"] == 3 and d["nsrc"] == (0 if kind == 2 else 2)
    assert d["flags"] == (1 if kind == 2 else 0)  # SFDB200_F_GRAD_NO_ROW2
    assert abs(d["dt"] - dt) <= 4e-16 * dt and abs(d["h"] - h) <= 4e-16 * h


@pytest.mark.parametrize("nsrc,nrec", [(0, 4), (3, 0), (0, 0)])
def test_descriptor_empty_sets(tmp_path, nsrc, nrec):
    """Empty source / receiver sets (cfg4 has no receivers): dt then comes
    from the damping coefficient when nothing is injected."""
    for kind in (0, 1):
        d = _describe(tmp_path, _source(kind, 3, 8, nsrc=nsrc, nrec=nrec))
        assert (d["nsrc"], d["nrec"]) == (nsrc, nrec)
        assert abs(d["dt"] - 3.7e-4) <= 4e-16 * 3.7e-4 and abs(d["h"] - 7.5) <= 4e-15


def _preset_flags():
    """sfdb200::stencilfd_preset (include/sfdb200/stencilfd_preset.hpp)."""
    return ["-O2", "-wrapper", JIT, "-DSFDB200_DEVICE=0", "-L" + PKG, "-Wl,--no-as-needed",
            "-lsfdb200", "-Wl,-rpath," + PKG]


def _compile_like_reference(tmp_path, src, flags, cc="cc", env=None):
    c = tmp_path / "0123456789abcdef.c"
    c.write_text(src)
    so = tmp_path / "0123456789abcdef.so"
    cmd = " ".join([cc, "-shared -fPIC"] + flags + ["-o", str(so), str(c), "-lm"])
    out = subprocess.run(cmd, shell=True, capture_output=True, text=True, env=env)
    return out, so


def _dynamic(so):
    return subprocess.run(["readelf", "-d", str(so)], capture_output=True, text=True).stdout


def _symbols(so):
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True, text=True)
    return {line.split()[-1] for line in out.stdout.splitlines() if line.strip()}


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_wrapper_swaps_the_kernel_for_the_shim(tmp_path, kind):
    """With the b200 preset, the reference's own compile command yields a .so
    whose <Name>_call is the sfdb200 shim (the loop nest is gone) and which
    records libsfdb200.so as NEEDED (the dlopen of runtime.cpp:241-248 then
    resolves sfdb200_call; a plain -lsfdb200 before the source would be
    dropped by --as-needed)."""
    name = ["Forward", "Adjoint", "Gradient"][kind]
    out, so = _compile_like_reference(tmp_path, _source(kind, 3, 8), _preset_flags())
    assert out.returncode == 0, out.stderr
    syms = _symbols(so)
    assert name + "_call" in syms and name not in syms
    dyn = _dynamic(so)
    assert "[libsfdb200.so]" in dyn and PKG in dyn
    assert not list(tmp_path.glob("*.sfdb200.*"))  # the shim source is cleaned up


def test_compiler_hook_mode(tmp_path):
    """STENCILFD_CC=sfdb200-jit (the reference's compiler hook) with the
    reference's generic preset flags: the driver adds include / link flags."""
    flags = ["-O3", "-march=native", "-fopenmp", "-ffp-contract=fast"]
    out, so = _compile_like_reference(tmp_path, _source(0, 2, 4), flags, cc=JIT)
    assert out.returncode == 0, out.stderr
    assert "Forward_call" in _symbols(so) and "Forward" not in _symbols(so)
    assert "[libsfdb200.so]" in _dynamic(so)


def test_other_sources_pass_through(tmp_path):
    """A source that is not a generated stencilfd kernel compiles unchanged."""
    src = "#include <math.h>\n\nint twice(int x) { return 2 * x; }\n"
    out, so = _compile_like_reference(tmp_path, src, _preset_flags())
    assert out.returncode == 0, out.stderr
    assert "twice" in _symbols(so)


def test_unsupported_kernel_fails_the_compile(tmp_path):
    """A stencilfd kernel that is not an acoustic operator fails loudly
    (compile_and_load turns the exit code into CompileError)."""
    src = _source(0, 3, 8).replace("damp", "eta")
    out, _ = _compile_like_reference(tmp_path, src, _preset_flags())
    assert out.returncode != 0
    assert "not a seismic forward / adjoint / gradient kernel" in out.stderr + out.stdout


GOLDEN = "/root/reference/proj/tests/golden"


@pytest.mark.skipif(not os.path.isdir(GOLDEN), reason="reference sources not present")
def test_reference_golden_kernels(tmp_path):
    """The reference's own golden emitted C (proj/tests/golden, pinned by its
    acceptance test, acceptance.cpp:228-229): the Forward kernel reads back as
    24^3 padded, so 2, nt 12, one source, two receivers, h = 0.1, dt = 1e-3;
    the sparse-free `Plain` test kernel is not a seismic operator and is refused."""
    d = _describe(tmp_path, open(os.path.join(GOLDEN, "forward_3d_full.c")).read())
    assert (d["name"], d["kind"], d["ndim"], d["padded"]) == ("Forward", 0, 3, [24, 24, 24])
    assert (d["space_order"], d["nt"], d["nsrc"], d["nrec"], d["save"]) == (2, 12, 1, 2, 0)
    assert abs(d["h"] - 0.1) <= 1e-16 and abs(d["dt"] - 1e-3) <= 1e-18
    path = tmp_path / "plain.c"
    path.write_text(open(os.path.join(GOLDEN, "plain_2d_all_off.c")).read())
    out = subprocess.run([JIT, "--describe", str(path)], capture_output=True, text=True)
    assert out.returncode != 0 and "not a seismic" in out.stderr
