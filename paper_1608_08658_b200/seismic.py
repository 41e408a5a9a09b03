"""Operator-level API mirroring ``sfd::seismic`` (proj/include/stencilfd/seismic.hpp)
on top of the B200 backend.  Same names, argument meaning and error behaviour:

  VelocityModel / make_model / make_constant_model   seismic.hpp:20-42
  build_damping, ricker, critical_dt                  seismic.hpp:48-57
  SparsePoints / locate_points                        seismic.hpp:61-71
  ShotRecord / zero_record                            seismic.hpp:74-81
  RunConfig                                           seismic.hpp:85-89 (device instead of preset)
  history_rows                                        seismic.hpp:93
  forward / adjoint / gradient                        seismic.hpp:104-144
  objective, restrict_interior, add_interior          seismic.hpp:147-156
  save_model / load_model / save_record / load_record seismic.hpp:160-168

Validation raises ValueError (InvalidArgument) where the reference throws
std::invalid_argument, and RuntimeError where it throws runtime::RuntimeError.
Every kernel runs on the B200 through libsfdb200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import json
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L


@dataclass
class VelocityModel:
    interior: list
    h: float = 10.0
    nbpml: int = 10
    space_order: int = 2
    padded: list = field(default_factory=list)
    m: np.ndarray = None
    damp: np.ndarray = None

    def ndim(self):
        return len(self.interior)

    def halo(self):
        return self.space_order // 2

    def pad(self):
        return self.nbpml + self.halo()

    def cells(self):
        return int(np.prod(self.padded))

    def m_min(self):
        return float(np.min(self.m))


@dataclass
class SparsePoints:
    npoints: int = 0
    ndim: int = 0
    idx: np.ndarray = None  # [npoints][ndim] int64
    w: np.ndarray = None    # [npoints][2^ndim]


@dataclass
class ShotRecord:
    nt: int = 0
    dt: float = 0.0
    npoints: int = 0
    data: np.ndarray = None  # [nt][npoints]


@dataclass
class RunConfig:
    device: int = 0


@dataclass
class RunStats:
    seconds: float = 0.0
    gpts: float = 0.0


@dataclass
class ForwardResult:
    record: ShotRecord
    u: np.ndarray            # 3 rolling slots or history_rows(nt) rows, padded shape
    saved: bool
    stats: RunStats


@dataclass
class AdjointResult:
    src_samples: ShotRecord
    v: np.ndarray
    stats: RunStats


@dataclass
class GradientResult:
    grad: np.ndarray         # padded cells
    stats: RunStats


def history_rows(nt):
    return nt + 1


def _interior(interior):
    return L.i64([int(e) for e in interior])


def make_model(interior, h, nbpml, space_order, m_interior) -> VelocityModel:
    interior = list(int(e) for e in interior)
    if not interior:
        raise L.InvalidArgument(L.EINVAL, "model needs at least one dimension")
    if any(e < 3 for e in interior):
        raise L.InvalidArgument(L.EINVAL, "model interior extents must be at least 3")
    if not h > 0:
        raise L.InvalidArgument(L.EINVAL, "grid spacing must be positive")
    if nbpml < 0:
        raise L.InvalidArgument(L.EINVAL, "absorbing-layer width must be non-negative")
    if space_order < 2 or space_order % 2:
        raise L.InvalidArgument(L.EINVAL, "space order must be a positive even number")
    mi = L.f64(m_interior).ravel()
    if mi.size != int(np.prod(interior)):
        raise L.InvalidArgument(L.EINVAL,
                                "squared-slowness field does not match the interior shape")
    if not np.all(mi > 0):
        raise L.InvalidArgument(L.EINVAL, "squared slowness must be positive")
    nd = len(interior)
    pad = nbpml + space_order // 2
    padded = L.i64([e + 2 * pad for e in interior])
    cells = int(np.prod(padded))
    m = np.empty(cells)
    damp = np.empty(cells)
    L.check(L.lib().sfdb200_make_model(nd, L.lptr(_interior(interior)), float(h), int(nbpml),
                                       int(space_order), L.dptr(mi), L.lptr(padded), L.dptr(m),
                                       L.dptr(damp)))
    return VelocityModel(interior, float(h), int(nbpml), int(space_order),
                         [int(p) for p in padded], m, damp)


def make_constant_model(interior, h, nbpml, space_order, velocity) -> VelocityModel:
    if not velocity > 0:
        raise L.InvalidArgument(L.EINVAL, "velocity must be positive")
    n = int(np.prod([int(e) for e in interior]))
    return make_model(interior, h, nbpml, space_order, np.full(n, 1.0 / (velocity * velocity)))


def build_damping(padded, nbpml, halo, h) -> np.ndarray:
    padded = L.i64(padded)
    out = np.empty(int(np.prod(padded)))
    L.check(L.lib().sfdb200_build_damping(len(padded), L.lptr(padded), int(nbpml), int(halo),
                                          float(h), L.dptr(out)))
    return out


def ricker(f0, t0, nt, dt) -> np.ndarray:
    if not f0 > 0:
        raise L.InvalidArgument(L.EINVAL, "peak frequency must be positive")
    if nt < 0:
        raise L.InvalidArgument(L.EINVAL, "sample count must be non-negative")
    out = np.empty(int(nt))
    L.check(L.lib().sfdb200_ricker(float(f0), float(t0), int(nt), float(dt), L.dptr(out)))
    return out


def fd_coefficients2(space_order) -> np.ndarray:
    w = np.empty(space_order + 1)
    L.check(L.lib().sfdb200_fd2(int(space_order), L.dptr(w)))
    return w


def critical_dt(model: VelocityModel) -> float:
    return float(L.lib().sfdb200_critical_dt(model.ndim(), model.h, model.space_order,
                                             model.m_min()))


def locate_points(model: VelocityModel, coords) -> SparsePoints:
    nd = model.ndim()
    rows = [list(c) for c in coords]
    for c in rows:
        if len(c) != nd:
            raise L.InvalidArgument(L.EINVAL,
                                    "coordinate dimensionality does not match the model")
    n = len(rows)
    c = L.f64(rows).reshape(n, nd) if n else np.zeros((0, nd))
    for p in range(n):
        for d in range(nd):
            span = (model.interior[d] - 1) * model.h
            if c[p, d] < 0.0 or c[p, d] > span:
                raise L.InvalidArgument(
                    L.EINVAL, f"point coordinate {c[p, d]} lies outside the physical "
                    f"interior [0, {span}]")
    idx = np.zeros((n, nd), np.int64)
    w = np.zeros((n, 1 << nd))
    L.check(L.lib().sfdb200_locate_points(nd, L.lptr(_interior(model.interior)), model.h,
                                          model.nbpml, model.space_order, n, L.dptr(c),
                                          L.lptr(idx), L.dptr(w)))
    return SparsePoints(n, nd, idx, w)


def zero_record(nt, dt, npoints) -> ShotRecord:
    return ShotRecord(int(nt), float(dt), int(npoints), np.zeros((int(nt), int(npoints))))


def check_dt(model: VelocityModel, dt):
    """seismic.cpp:31-37"""
    if not dt > 0:
        raise L.InvalidArgument(L.EINVAL, "dt must be positive")
    limit = critical_dt(model)
    if dt > limit:
        raise L.InvalidArgument(L.EINVAL,
                                f"dt {dt} exceeds the stable CFL limit {limit}")


def _sparse_args(pts: SparsePoints, nd):
    if pts.npoints == 0:
        return np.zeros((0, nd), np.int64), np.zeros((0, 1 << nd))
    return L.i64(pts.idx), L.f64(pts.w)


def _stats(plan, seconds):
    pts = plan.points_per_step * plan.steps
    return RunStats(seconds, pts / seconds / 1e9 if seconds > 0 else 0.0)


def forward(model: VelocityModel, src: SparsePoints, src_trace, rec: SparsePoints, nt, dt,
            save, cfg: Optional[RunConfig] = None) -> ForwardResult:
    """seismic.cpp:333-380 on the B200."""
    cfg = cfg or RunConfig()
    check_dt(model, dt)
    trace = L.f64(src_trace).ravel()
    if trace.size != nt * src.npoints:
        raise L.InvalidArgument(L.EINVAL, "source trace must hold nt samples per source point")
    nd = model.ndim()
    rows = history_rows(nt) if save else 3
    u = np.empty((rows, *model.padded))
    rec_data = np.empty((int(nt), rec.npoints))
    si, sw = _sparse_args(src, nd)
    ri, rw = _sparse_args(rec, nd)
    plan = L.Plan(L.FORWARD, nd, model.padded, model.space_order, nt, dt, model.h, src.npoints,
                  rec.npoints, save, cfg.device)
    t0 = time.perf_counter()
    plan.run([u, L.f64(model.m), L.f64(model.damp), si, sw, trace, ri, rw, rec_data])
    secs = time.perf_counter() - t0
    record = ShotRecord(int(nt), float(dt), rec.npoints, rec_data)
    out = ForwardResult(record, u, bool(save), _stats(plan, secs))
    plan.close()
    return out


def adjoint(model: VelocityModel, rec: SparsePoints, residual: ShotRecord, src: SparsePoints,
            nt, dt, cfg: Optional[RunConfig] = None) -> AdjointResult:
    """seismic.cpp:382-426 on the B200."""
    cfg = cfg or RunConfig()
    check_dt(model, dt)
    data = L.f64(residual.data).ravel()
    if residual.nt != nt or residual.npoints != rec.npoints or data.size != nt * rec.npoints:
        raise L.InvalidArgument(L.EINVAL,
                                "residual record does not match nt and the receiver set")
    nd = model.ndim()
    v = np.empty((3, *model.padded))
    src_data = np.empty((int(nt), src.npoints))
    si, sw = _sparse_args(src, nd)
    ri, rw = _sparse_args(rec, nd)
    plan = L.Plan(L.ADJOINT, nd, model.padded, model.space_order, nt, dt, model.h, src.npoints,
                  rec.npoints, False, cfg.device)
    t0 = time.perf_counter()
    plan.run([v, L.f64(model.m), L.f64(model.damp), si, sw, src_data, ri, rw, data])
    secs = time.perf_counter() - t0
    out = AdjointResult(ShotRecord(int(nt), float(dt), src.npoints, src_data), v,
                        _stats(plan, secs))
    plan.close()
    return out


def gradient(model: VelocityModel, rec: SparsePoints, residual: ShotRecord, u_history, nt, dt,
             cfg: Optional[RunConfig] = None) -> GradientResult:
    """seismic.cpp:428-496 on the B200 (the row-2 host term is part of the device loop)."""
    cfg = cfg or RunConfig()
    check_dt(model, dt)
    data = L.f64(residual.data).ravel()
    if residual.nt != nt or residual.npoints != rec.npoints or data.size != nt * rec.npoints:
        raise L.InvalidArgument(L.EINVAL,
                                "residual record does not match nt and the receiver set")
    hist = L.f64(u_history).ravel()
    if hist.size != history_rows(nt) * model.cells():
        raise L.InvalidArgument(L.EINVAL, "wavefield history must come from a saved forward run")
    nd = model.ndim()
    v = np.empty((3, *model.padded))
    grad = np.empty(model.padded)
    ri, rw = _sparse_args(rec, nd)
    plan = L.Plan(L.GRADIENT, nd, model.padded, model.space_order, nt, dt, model.h, 0,
                  rec.npoints, False, cfg.device)
    t0 = time.perf_counter()
    plan.run([v, hist, L.f64(model.m), L.f64(model.damp), grad, ri, rw, data])
    secs = time.perf_counter() - t0
    out = GradientResult(grad, _stats(plan, secs))
    plan.close()
    return out


@dataclass
class FwiResult:
    phi: float               # 1/2 sum (syn - obs)^2
    grad: np.ndarray         # padded cells
    record: ShotRecord       # synthetic traces
    history_bytes: int       # device bytes holding the forward wavefield for the gradient
    stats: RunStats          # forward + gradient wall time, gradient steps counted


def fwi_gradient(model: VelocityModel, src: SparsePoints, src_trace, rec: SparsePoints,
                 observed: ShotRecord, nt, dt, checkpoint_interval: Optional[int] = None,
                 cfg: Optional[RunConfig] = None) -> FwiResult:
    """One FWI gradient (the forward(save) -> objective -> gradient chain of
    verify.cpp:179-297 / the cfg3 workload) kept on the device.

    checkpoint_interval: 0 keeps the whole u history in HBM (nt + 1 rows, the
    reference's saved-history semantics); k > 0 keeps restart rows every k steps
    and recomputes each segment during the backward pass (3-D only; SURVEY
    §8(f) row 2, sfdb200_set_checkpointing); None picks ~sqrt(steps) in 3-D."""
    cfg = cfg or RunConfig()
    check_dt(model, dt)
    nd = model.ndim()
    steps = max(0, int(nt) - 2)
    if checkpoint_interval is None:
        checkpoint_interval = max(1, int(round(steps ** 0.5))) if nd == 3 else 0
    k = int(checkpoint_interval)
    if k and nd != 3:
        raise L.InvalidArgument(L.EINVAL, "checkpointing is implemented for 3-D problems")
    trace = L.f64(src_trace).ravel()
    if trace.size != nt * src.npoints:
        raise L.InvalidArgument(L.EINVAL, "source trace must hold nt samples per source point")
    obs = L.f64(observed.data)
    if observed.nt != nt or observed.npoints != rec.npoints:
        raise L.InvalidArgument(L.EINVAL, "observed record does not match nt and the receivers")
    si, sw = _sparse_args(src, nd)
    ri, rw = _sparse_args(rec, nd)
    m, damp = L.f64(model.m), L.f64(model.damp)
    fwd = L.Plan(L.FORWARD, nd, model.padded, model.space_order, nt, dt, model.h, src.npoints,
                 rec.npoints, k == 0, cfg.device)
    g = L.Plan(L.GRADIENT, nd, model.padded, model.space_order, nt, dt, model.h, 0,
               rec.npoints, False, cfg.device)
    try:
        t0 = time.perf_counter()
        syn = np.empty((int(nt), rec.npoints))
        fargv = [None, m, damp, si, sw, trace, ri, rw, syn]
        if k:
            fwd.set_checkpointing(k)
        fwd.upload(fargv)
        fwd.execute()
        fwd.download(fargv)
        resid = syn - obs.reshape(syn.shape)
        phi = 0.5 * float(np.dot(resid.ravel(), resid.ravel()))
        if k:
            g.bind_checkpoints(fwd)
            hist_bytes = fwd.checkpoint_bytes
        else:
            g.bind_history(fwd)
            hist_bytes = history_rows(nt) * int(np.prod(model.padded)) * 4
        grad = np.empty(model.padded)
        g.run([None, None, m, damp, grad, ri, rw, resid])
        secs = time.perf_counter() - t0
        return FwiResult(phi, grad, ShotRecord(int(nt), float(dt), rec.npoints, syn),
                         int(hist_bytes), _stats(g, secs))
    finally:
        g.close()
        fwd.close()


def objective(synthetic: ShotRecord, observed: ShotRecord, want_residual=False):
    """seismic.cpp:498-510: Phi = 1/2 sum (syn - obs)^2 (and the residual record)."""
    a = np.asarray(synthetic.data, np.float64)
    b = np.asarray(observed.data, np.float64)
    if synthetic.nt != observed.nt or synthetic.npoints != observed.npoints or a.size != b.size:
        raise L.InvalidArgument(L.EINVAL, "records disagree in shape")
    shape = a.shape
    a = np.ascontiguousarray(a).ravel()
    b = np.ascontiguousarray(b).ravel()
    d = np.empty(a.size) if want_residual else None
    phi = C.c_double()
    # element order, as the reference accumulates (sfdb200_objective, host C)
    L.check(L.lib().sfdb200_objective(L.dptr(a), L.dptr(b), a.size,
                                      L.dptr(d) if d is not None else None, C.byref(phi)))
    phi = phi.value
    if want_residual:
        d = d.reshape(shape)
        return phi, ShotRecord(synthetic.nt, synthetic.dt, synthetic.npoints, d)
    return phi


def restrict_interior(model: VelocityModel, padded_field) -> np.ndarray:
    f = np.asarray(padded_field, np.float64)
    if f.size != model.cells():
        raise L.InvalidArgument(L.EINVAL, "field does not match the padded shape")
    p = model.pad()
    sl = tuple(slice(p, p + n) for n in model.interior)
    return f.reshape(model.padded)[sl].ravel().copy()


def add_interior(model: VelocityModel, interior_field, scale, padded_field):
    f = np.asarray(interior_field, np.float64)
    if f.size != int(np.prod(model.interior)) or padded_field.size != model.cells():
        raise L.InvalidArgument(L.EINVAL, "field shapes do not match the model")
    p = model.pad()
    sl = tuple(slice(p, p + n) for n in model.interior)
    view = padded_field.reshape(model.padded)
    view[sl] += scale * f.reshape(model.interior)


def save_model(model: VelocityModel, path_prefix):
    """seismic.cpp:557-568: JSON header + raw float64 interior squared slowness."""
    with open(path_prefix + ".json", "w") as fh:
        json.dump({"shape": model.interior, "h": model.h, "nbpml": model.nbpml}, fh, indent=2)
        fh.write("\n")
    restrict_interior(model, model.m).astype("<f8").tofile(path_prefix + ".bin")


def load_model(path_prefix, space_order) -> VelocityModel:
    with open(path_prefix + ".json") as fh:
        hdr = json.load(fh)
    shape = [int(e) for e in hdr["shape"]]
    m = np.fromfile(path_prefix + ".bin", dtype="<f8")
    if m.size != int(np.prod(shape)):
        raise RuntimeError("cannot read " + path_prefix + ".bin")
    return make_model(shape, float(hdr["h"]), int(hdr["nbpml"]), space_order, m)


def save_record(record: ShotRecord, coordinates, path_prefix):
    with open(path_prefix + ".json", "w") as fh:
        json.dump({"nt": record.nt, "dt": record.dt,
                   "coordinates": [list(map(float, c)) for c in coordinates]}, fh, indent=2)
        fh.write("\n")
    np.asarray(record.data, "<f8").tofile(path_prefix + ".bin")


def load_record(path_prefix):
    with open(path_prefix + ".json") as fh:
        hdr = json.load(fh)
    coords = hdr["coordinates"]
    nt, n = int(hdr["nt"]), len(coords)
    data = np.fromfile(path_prefix + ".bin", dtype="<f8")
    if data.size != nt * n:
        raise RuntimeError("cannot read " + path_prefix + ".bin")
    return ShotRecord(nt, float(hdr["dt"]), n, data.reshape(nt, n)), coords
