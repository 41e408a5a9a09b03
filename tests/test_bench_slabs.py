"""CPU tests of bench.py's per-rank cfg5 inputs (N > 1): each rank generates
only the interior rows its z slab needs and fills only its planes of the
global-shaped model arrays; those planes must equal the full cfg5 model's
(configs.cfg5 + make_model, i.e. the reference's make_model / build_damping)
bit for bit, at a reduced grid size."""
import types

import numpy as np
import pytest

import bench
from paper_1608_08658_b200 import _lib as L, configs, seismic as S


def test_slab_rows_equal_the_whole_grid():
    shape = (40, 12, 10)
    full = configs.smooth_random_velocity(shape, 1, 2.0)
    parts = [(0, 15), (11, 29), (25, 40)]
    lo, hi = [], []

    def collect(a, b):
        lo.append(a)
        hi.append(b)
        return a, b

    for z0, z1 in parts:
        configs.smooth_random_velocity_rows(shape, 1, 2.0, z0, z1, collect)
    g = (min(lo), max(hi))
    for z0, z1 in parts:
        rows = configs.smooth_random_velocity_rows(shape, 1, 2.0, z0, z1, lambda a, b: g)
        assert np.array_equal(rows, full[z0:z1])


@pytest.mark.parametrize("world", [2, 3])
def test_slab_model_planes_equal_the_full_model(world):
    n = 24  # cfg5 at 24^3 interior (+ 40-point layer, so 16)
    full = configs.cfg5(n=n, nt=12, nrec_side=4)
    model = S.make_model(full.interior, full.h, full.nbpml, 16, full.m_interior)
    P = model.padded[0]
    # the rescale range the ranks would all-reduce
    v = configs.smooth_random_velocity((n, n, n), 1, 16.0)
    raw = 1500.0 + 3000.0 * np.random.default_rng(1).random(n ** 3)
    from scipy.ndimage import gaussian_filter1d
    sm = raw.reshape(n, n, n)
    for ax in range(3):
        sm = gaussian_filter1d(sm, 16.0, axis=ax, mode="nearest", truncate=4.0)
    rng_lohi = (float(sm.min()), float(sm.max()))
    args = types.SimpleNamespace(time_steps=10)
    for rank in range(world):
        w, m = bench.slab_problem(L, S, args, world, rank, n=n, minmax=lambda a, b: rng_lohi)
        assert w.dt == full.dt and np.array_equal(w.src_coords, full.src_coords)
        zb, ze = L.slab(P, 16, world, rank)
        z0, z1 = zb - 8, ze + 8
        mv, dv = m.m.reshape(P, P, P), m.damp.reshape(P, P, P)
        assert np.array_equal(mv[z0:z1], model.m.reshape(P, P, P)[z0:z1])
        assert np.array_equal(dv[z0:z1], model.damp.reshape(P, P, P)[z0:z1])
        # nothing outside the slab was written (those pages stay unbacked)
        assert not mv[:z0].any() and not mv[z1:].any()
    assert v.shape == (n, n, n)


def test_reference_sample_is_cropped_to_host_memory(monkeypatch):
    """bench.py's reference arm: on a host that cannot hold the reference's fp64
    grids of the workload, the sample keeps the x / y extents, sources and
    receivers and crops the interior along z (and says so); otherwise the
    workload is untouched."""
    import builtins
    w = configs.cfg2(n=64, nt=12)
    same, note = bench.fit_reference_to_memory(w)
    assert same is w and note == ""
    real_open = builtins.open

    class Meminfo:
        def __enter__(self):
            return iter(["MemTotal: 1 kB\n", "MemAvailable: 600000 kB\n"])

        def __exit__(self, *a):
            return False

    monkeypatch.setattr(builtins, "open",
                        lambda p, *a, **k: Meminfo() if p == "/proc/meminfo" else real_open(p, *a, **k))
    c, note = bench.fit_reference_to_memory(w)
    assert c.interior[1:] == w.interior[1:] and 8 <= c.interior[0] < w.interior[0]
    assert c.m_interior.size == int(np.prod(c.interior)) and "cropped" in note
    full = np.asarray(w.m_interior).reshape(w.interior)
    assert np.array_equal(c.m_interior.reshape(c.interior), full[:c.interior[0]])
    assert 14 * 8 * np.prod(c.padded) <= 0.6 * 600000 * 1024
    assert w.interior[0] == 64  # the caller's workload is not modified
