"""Seeded synthetic stand-ins for BASELINE.json's five configurations
(SURVEY.md §8(d)).  The reference uses no public dataset; these generators
produce inputs with the stated shapes, sizes and value ranges.

Conventions (all configs): coordinates in metres, (z, y, x) order, origin at
the first interior node; h = 10 m, nbpml = 40; m = 1/v^2; Ricker t0 = 1.2/f0
(tools/sfd.cpp:168).  Real inputs are generated in fp64 and rounded to fp32,
and the same rounded values go to the B200 path and to the CPU oracle.

Random velocity: uniform draws v = 1500 + 3000 r from numpy's PCG64 stream
(np.random.default_rng(seed)) in row-major order -- the survey suggests
mt19937_64, but any seeded stream serves, since both sides get the same
values -- then a separable Gaussian (sigma cells, truncated at 4 sigma,
clamp-to-edge) and a min-max rescale to exactly [1500, 4500].
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    ndim: int
    interior: list
    space_order: int
    nt: int                 # trace samples; steps = nt - 2
    dt: float
    m_interior: np.ndarray  # fp32-rounded squared slowness, interior cells
    wavelet: np.ndarray     # [nt][nsrc], fp32-rounded
    src_coords: np.ndarray  # [nsrc][ndim]
    rec_coords: np.ndarray  # [nrec][ndim]
    h: float = 10.0
    nbpml: int = 40
    f0: float = 10.0
    extra: dict = field(default_factory=dict)

    @property
    def steps(self):
        return self.nt - 2

    @property
    def padded(self):
        pad = self.nbpml + self.space_order // 2
        return [n + 2 * pad for n in self.interior]

    @property
    def points_per_step(self):
        return int(np.prod([n + 2 * self.nbpml for n in self.interior]))


def _round32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def _ricker(f0, nt, dt, nsrc=1):
    t0 = 1.2 / f0
    k = np.arange(nt, dtype=np.float64)
    tau = k * dt - t0
    a = np.pi * np.pi * f0 * f0 * tau * tau
    w = (1.0 - 2.0 * a) * np.exp(-a)
    return _round32(np.repeat(w[:, None], nsrc, axis=1))


def smooth_random_velocity(shape, seed, sigma):
    """Uniform random velocity in [1.5, 4.5] km/s, Gaussian-smoothed along every
    axis (scipy's gaussian_filter1d, mode "nearest", truncate 4), rescaled to
    the same range.  Grids above 2^28 points (cfg5) are smoothed on the GPU
    when one is present (the same separable filter as fp64 convolutions);
    scipy's single-threaded pass would take minutes there."""
    rng = np.random.default_rng(seed)
    v = 1500.0 + 3000.0 * rng.random(int(np.prod(shape)), dtype=np.float64)
    v = v.reshape(shape)
    if v.size > (1 << 28) and _cuda_available():
        v = _smooth_on_gpu(v, sigma)
    else:
        from scipy.ndimage import gaussian_filter1d
        for ax in range(len(shape)):
            v = gaussian_filter1d(v, sigma, axis=ax, mode="nearest", truncate=4.0)
    lo, hi = v.min(), v.max()
    return 1500.0 + 3000.0 * (v - lo) / (hi - lo)


def smooth_random_velocity_rows(shape, seed, sigma, z0, z1, minmax=None):
    """Rows [z0, z1) (axis 0) of smooth_random_velocity(shape, seed, sigma)
    without the rest of the grid: the draws of rows [z0 - r, z1 + r) (r = the
    4-sigma filter radius) come straight from the PCG64 stream advanced to
    their offset (one 64-bit draw per value, row-major), the block is smoothed
    like the whole grid (clamp-to-edge only where it touches the grid's ends,
    so rows [z0, z1) see exactly their full filter windows), then cropped.
    minmax(lo, hi) -> (global lo, global hi) supplies the rescale range over
    all rows (e.g. an all-reduce over the ranks that together cover [0, n));
    None: these rows' own range (only right when [z0, z1) is the whole grid)."""
    n0 = shape[0]
    plane = int(np.prod(shape[1:]))
    r = int(4.0 * sigma + 0.5)
    lo, hi = max(0, z0 - r), min(n0, z1 + r)
    bg = np.random.PCG64(seed)
    bg.advance(lo * plane)
    v = 1500.0 + 3000.0 * np.random.Generator(bg).random((hi - lo) * plane, dtype=np.float64)
    v = v.reshape((hi - lo, *shape[1:]))
    if v.size > (1 << 26) and _cuda_available():
        v = _smooth_on_gpu(v, sigma)
    else:
        from scipy.ndimage import gaussian_filter1d
        for ax in range(len(shape)):
            v = gaussian_filter1d(v, sigma, axis=ax, mode="nearest", truncate=4.0)
    v = np.ascontiguousarray(v[z0 - lo:z1 - lo])
    a, b = float(v.min()), float(v.max())
    if minmax is not None:
        a, b = minmax(a, b)
    return 1500.0 + 3000.0 * (v - a) / (b - a)


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except ImportError:
        return False


def _smooth_on_gpu(v, sigma):
    import torch
    import torch.nn.functional as F
    r = int(4.0 * sigma + 0.5)
    x = np.arange(-r, r + 1, dtype=np.float64)
    k = np.exp(-0.5 * (x / sigma) ** 2)
    k = torch.tensor(k / k.sum(), dtype=torch.float64, device="cuda").view(1, 1, -1)
    t = torch.from_numpy(v).cuda()
    for ax in range(t.dim()):
        t = t.movedim(ax, -1).contiguous()
        sh = t.shape
        rows = t.reshape(-1, 1, sh[-1])
        out = torch.empty_like(rows)
        step = max(1, (1 << 26) // sh[-1])  # bounded temporaries
        for i in range(0, rows.shape[0], step):
            out[i:i + step] = F.conv1d(F.pad(rows[i:i + step], (r, r), mode="replicate"), k)
        t = out.reshape(sh).movedim(-1, ax)
        del rows
    out = t.contiguous().cpu().numpy()
    del t
    torch.cuda.empty_cache()
    return out


def _carpet(n_side, span, depth):
    c = (np.arange(n_side) + 0.5) * span / n_side
    yy, xx = np.meshgrid(c, c, indexing="ij")
    return np.stack([np.full(yy.size, depth), yy.ravel(), xx.ravel()], axis=1)


def _crit(m_min, ndim, so, h=10.0):
    """critical_dt exactly as the operators check it (seismic.cpp:187-193)."""
    from . import _lib
    return float(_lib.lib().sfdb200_critical_dt(ndim, h, so, float(m_min)))


def cfg1(n=201, nt=1002, nbpml=40):
    """2-D forward, two-layer velocity, so 4, 101 receivers (BASELINE configs[0])."""
    h = 10.0
    z = np.arange(n) * h
    v = np.where(z < 1000.0, 1500.0, 2500.0)[:, None] * np.ones((1, n))
    m = _round32(1.0 / v ** 2).ravel()
    dt = 0.4 * h / 2500.0
    span = (n - 1) * h
    rec = np.stack([np.full(101, 20.0), np.arange(101) * span / 100.0], axis=1)
    return Workload("cfg1-2d-so4", 2, [n, n], 4, nt, dt, m, _ricker(10.0, nt, dt),
                    np.array([[20.0, min(1000.0, span / 2)]]), rec, h, nbpml, 10.0)


def cfg2(n=256, nt=1002, nbpml=40, nrec_side=256):
    """3-D forward, smooth random velocity, so 8, receiver carpet (BASELINE configs[1])."""
    h = 10.0
    v = smooth_random_velocity((n, n, n), 0, 8.0)
    m = _round32(1.0 / v ** 2).ravel()
    dt = 0.4 * h / 4500.0
    span = (n - 1) * h
    src = np.array([[10.0, span / 2, span / 2]])
    return Workload("cfg2-3d-so8", 3, [n, n, n], 8, nt, dt, m, _ricker(12.0, nt, dt), src,
                    _carpet(nrec_side, span, 20.0), h, nbpml, 12.0)


def cfg2_stacked(copies, n=256, nt=1002, nbpml=40, nrec_side=256):
    """Weak-scaling form of cfg2 for N GPUs: the cfg2 model repeated `copies`
    times along z (interior n*copies x n x n), same source, receivers and
    steps, so every z-slab rank carries one cfg2-sized slab."""
    w = cfg2(n, nt, nbpml, nrec_side)
    if copies == 1:
        return w
    m = np.tile(w.m_interior.reshape(n, n, n), (copies, 1, 1)).ravel()
    return Workload(f"cfg2-3d-so8-x{copies}", 3, [n * copies, n, n], 8, w.nt, w.dt, m,
                    w.wavelet, w.src_coords, w.rec_coords, w.h, nbpml, w.f0)


def cfg3(n=200, nt=802, nbpml=40, nrec_side=200):
    """3-D FWI gradient: background + Gaussian anomaly (BASELINE configs[2]).
    Returns (true workload, background m)."""
    h = 10.0
    vb = smooth_random_velocity((n, n, n), 0, 8.0)
    c = (n - 1) / 2.0
    i = np.arange(n) - c
    r2 = i[:, None, None] ** 2 + i[None, :, None] ** 2 + i[None, None, :] ** 2
    vt = vb + 300.0 * np.exp(-r2 / 20.0 ** 2)
    dt = 0.4 * h / vt.max()
    span = (n - 1) * h
    src = np.array([[10.0, span / 2, span / 2]])
    w = Workload("cfg3-3d-so8-fwi", 3, [n, n, n], 8, nt, dt, _round32(1.0 / vt ** 2).ravel(),
                 _ricker(10.0, nt, dt), src, _carpet(nrec_side, span, 20.0), h, nbpml, 10.0)
    w.extra["m_background"] = _round32(1.0 / vb ** 2).ravel()
    return w


def cfg4(so, n=512, nt=202, nbpml=40):
    """3-D so sweep, linear v(z), no receivers (BASELINE configs[3])."""
    h = 10.0
    z = np.arange(n) * h
    vz = 1500.0 + 3000.0 * z / ((n - 1) * h)
    v = np.broadcast_to(vz[:, None, None], (n, n, n))
    m = _round32(1.0 / v ** 2).ravel()
    dt = min(0.4 * h / 4500.0, _crit(m.min(), 3, so, h))
    span = (n - 1) * h
    src = np.array([[span / 2] * 3])
    return Workload(f"cfg4-3d-so{so}", 3, [n, n, n], so, nt, dt, m, _ricker(15.0, nt, dt), src,
                    np.zeros((0, 3)), h, nbpml, 15.0)


def cfg5(n=1024, nt=502, nbpml=40, nrec_side=512):
    """3-D so 16 forward, 4 sources, 512^2 carpet (BASELINE configs[4])."""
    h = 10.0
    v = smooth_random_velocity((n, n, n), 1, 16.0)
    m = _round32(1.0 / v ** 2).ravel()
    dt = _crit(m.min(), 3, 16, h)
    span = (n - 1) * h
    q = [span / 4, 3 * span / 4]
    src = np.array([[10.0, a, b] for a in q for b in q])
    return Workload("cfg5-3d-so16", 3, [n, n, n], 16, nt, dt, m, _ricker(10.0, nt, dt, 4), src,
                    _carpet(nrec_side, span, 20.0), h, nbpml, 10.0)


def cfg5_rows(z0, z1, minmax, n=1024, nt=502, nbpml=40, nrec_side=512):
    """cfg5 restricted to the interior rows [z0, z1) a z-slab rank needs
    (bench.py --gpus N): m_interior holds those rows only (extra["rows"]), the
    rescale range and dt come from the whole grid through minmax (see
    smooth_random_velocity_rows).  Sources and receivers are the full sets."""
    h = 10.0
    v = smooth_random_velocity_rows((n, n, n), 1, 16.0, z0, z1, minmax)
    m = _round32(1.0 / v ** 2).ravel()
    m_min = _round32(np.array([1.0 / 4500.0 ** 2]))[0]  # v reaches 4500 exactly at the global max
    dt = _crit(m_min, 3, 16, h)
    span = (n - 1) * h
    q = [span / 4, 3 * span / 4]
    src = np.array([[10.0, a, b] for a in q for b in q])
    w = Workload("cfg5-3d-so16", 3, [n, n, n], 16, nt, dt, m, _ricker(10.0, nt, dt, 4), src,
                 _carpet(nrec_side, span, 20.0), h, nbpml, 10.0)
    w.extra["rows"] = (z0, z1)
    return w
