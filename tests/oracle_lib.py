"""TEST INFRASTRUCTURE: ctypes bindings for the CPU oracle (oracle/libsfdoracle.so,
the C restatement) and, where it was built, the unmodified reference
(oracle/_ref/libsfdref.so).  Only tests/, __graft_entry__.smoke() and bench.py's
CPU legs import this module, and only as the checker / CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "libsfdoracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libsfdref.so")

_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_long)


def _d_ref(x):
    return C.cast(C.pointer(x), _dp)


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _l(a):
    return a.ctypes.data_as(_lp) if a is not None else None


class Problem(C.Structure):
    _fields_ = [("ndim", C.c_int), ("padded", C.c_long * 3), ("space_order", C.c_int),
                ("nt", C.c_long), ("dt", C.c_double), ("h", C.c_double),
                ("nsrc", C.c_long), ("nrec", C.c_long)]


_i, _L, _D, _P = C.c_int, C.c_long, C.c_double, C.c_void_p
_ORACLE_SIGS = {
    "sfdo_fd2": (_i, [_i, _dp]),
    "sfdo_make_model": (_i, [_i, _lp, _D, _L, _i, _dp, _lp, _dp, _dp]),
    "sfdo_locate": (_i, [_i, _lp, _D, _L, _i, _L, _dp, _lp, _dp]),
    "sfdo_ricker": (None, [_D, _D, _L, _D, _dp]),
    "sfdo_critical_dt": (_D, [_i, _D, _i, _D]),
    "sfdo_forward": (_i, [_P, _i, _dp, _dp, _dp, _lp, _dp, _dp, _lp, _dp, _dp]),
    "sfdo_adjoint": (_i, [_P, _dp, _dp, _dp, _lp, _dp, _dp, _lp, _dp, _dp]),
    "sfdo_gradient": (_i, [_P, _dp, _dp, _dp, _dp, _dp, _lp, _dp, _dp]),
    "sfdo_forward_steps": (_i, [_P, _dp, _dp, _dp, _lp, _dp, _dp, _P, _lp, _dp, _dp, _P, _L,
                                _L]),
    "sfdo_sample_row": (_i, [_P, _dp, _L, _lp, _dp, _dp, _P]),
}
_REF_SIGS = {
    "sfdref_fd2": (_i, [_i, _dp]),
    "sfdref_model": (_i, [_i, _lp, _D, _L, _i, _dp, _lp, _dp, _dp]),
    "sfdref_locate": (_i, [_i, _lp, _D, _L, _i, _dp, _L, _dp, _lp, _dp]),
    "sfdref_critical_dt": (_i, [_i, _lp, _D, _L, _i, _dp, _dp]),
    "sfdref_ricker": (_i, [_D, _D, _L, _D, _dp]),
    "sfdref_forward": (_i, [_i, _lp, _D, _L, _i, _dp, _L, _dp, _dp, _L, _dp, _L, _D, _i, _i,
                            _dp, _dp, _dp]),
    "sfdref_adjoint": (_i, [_i, _lp, _D, _L, _i, _dp, _L, _dp, _dp, _L, _dp, _L, _D, _i, _dp,
                            _dp, _dp]),
    "sfdref_gradient": (_i, [_i, _lp, _D, _L, _i, _dp, _L, _dp, _dp, _dp, _L, _D, _i, _dp,
                             _dp]),
    "sfdref_generate": (_i, [_i, _i, _lp, _D, _L, _i, _dp, _L, _L, _L, _D, _i, _i, C.c_char_p,
                             _L, _lp]),
    "sfdref_save_model": (_i, [_i, _lp, _D, _L, _i, _dp, C.c_char_p]),
    "sfdref_load_model": (_i, [C.c_char_p, _i, C.POINTER(_i), _lp, _dp, _lp, _lp, _dp, _dp]),
    "sfdref_save_record": (_i, [_L, _D, _L, _i, _dp, _dp, C.c_char_p]),
    "sfdref_load_record": (_i, [C.c_char_p, _lp, _dp, _lp, C.POINTER(_i), _dp, _dp]),
    "sfdref_dump_grid": (_i, [_dp, _i, _lp, _L, _L, C.c_char_p]),
    "sfdref_objective": (_i, [_dp, _dp, _L, _dp, _dp]),
    "sfdref_problem_create": (_P, [_i, _lp, _D, _L, _i, _dp, _L, _dp, _L, _dp]),
    "sfdref_problem_free": (None, [_P]),
    "sfdref_problem_forward": (_i, [_P, _dp, _L, _D, _dp, _dp]),
}


def _declare(lib, sigs):
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args


_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"], check=True)
        _oracle = C.CDLL(ORACLE_SO)
        _declare(_oracle, _ORACLE_SIGS)
    return _oracle


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        _ref = C.CDLL(REF_SO)
        _ref.sfdref_last_error.restype = C.c_char_p
        _declare(_ref, _REF_SIGS)
    return _ref


def _check_ref(rc):
    if rc != 0:
        raise ValueError(ref().sfdref_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# ---------------------------------------------------------------- oracle port

def fd2(so):
    w = np.zeros(so + 1)
    assert oracle().sfdo_fd2(so, _d(w)) == 0
    return w


def make_model(interior, h, nbpml, so, m_interior):
    interior = _i64(interior)
    nd = len(interior)
    pad = nbpml + so // 2
    padded = _i64(interior + 2 * pad)
    m = np.zeros(int(np.prod(padded)))
    damp = np.zeros_like(m)
    rc = oracle().sfdo_make_model(nd, _l(interior), C.c_double(h), C.c_long(nbpml), so,
                                  _d(_f64(m_interior).ravel()), _l(padded), _d(m), _d(damp))
    if rc:
        raise ValueError("invalid model")
    return padded, m, damp


def locate(interior, h, nbpml, so, coords):
    interior = _i64(interior)
    coords = _f64(coords).reshape(-1, len(interior))
    n, nd = coords.shape
    idx = np.zeros((n, nd), np.int64)
    w = np.zeros((n, 1 << nd))
    if oracle().sfdo_locate(nd, _l(interior), C.c_double(h), C.c_long(nbpml), so, n,
                            _d(coords), _l(idx), _d(w)):
        raise ValueError("point outside the interior")
    return idx, w


def ricker(f0, t0, nt, dt):
    out = np.zeros(nt)
    oracle().sfdo_ricker(C.c_double(f0), C.c_double(t0), C.c_long(nt), C.c_double(dt), _d(out))
    return out


def critical_dt(ndim, h, so, m_min):
    return oracle().sfdo_critical_dt(ndim, C.c_double(h), so, C.c_double(m_min))


def _problem(padded, so, nt, dt, h, nsrc, nrec):
    p = Problem()
    p.ndim = len(padded)
    for i, e in enumerate(padded):
        p.padded[i] = int(e)
    p.space_order, p.nt, p.dt, p.h, p.nsrc, p.nrec = so, nt, dt, h, nsrc, nrec
    return p


def forward(padded, so, h, dt, nt, m, damp, src_idx, src_w, src_data, rec_idx, rec_w, save=False):
    cells = int(np.prod(padded))
    nsrc, nrec = len(src_idx), len(rec_idx)
    u = np.zeros(((nt + 1) if save else 3) * cells)
    rec = np.zeros(nt * nrec)
    p = _problem(padded, so, nt, dt, h, nsrc, nrec)
    rc = oracle().sfdo_forward(C.cast(C.pointer(p), C.c_void_p), int(save), _d(u), _d(_f64(m)), _d(_f64(damp)),
                               _l(_i64(src_idx)), _d(_f64(src_w)), _d(_f64(src_data)),
                               _l(_i64(rec_idx)), _d(_f64(rec_w)), _d(rec))
    assert rc == 0
    return u.reshape(-1, *padded), rec.reshape(nt, nrec)


def adjoint(padded, so, h, dt, nt, m, damp, src_idx, src_w, rec_idx, rec_w, rec_data):
    cells = int(np.prod(padded))
    nsrc, nrec = len(src_idx), len(rec_idx)
    v = np.zeros(3 * cells)
    src = np.zeros(nt * nsrc)
    p = _problem(padded, so, nt, dt, h, nsrc, nrec)
    rc = oracle().sfdo_adjoint(C.cast(C.pointer(p), C.c_void_p), _d(v), _d(_f64(m)), _d(_f64(damp)),
                               _l(_i64(src_idx)), _d(_f64(src_w)), _d(src),
                               _l(_i64(rec_idx)), _d(_f64(rec_w)), _d(_f64(rec_data)))
    assert rc == 0
    return v.reshape(3, *padded), src.reshape(nt, nsrc)


def gradient(padded, so, h, dt, nt, m, damp, u_history, rec_idx, rec_w, rec_data):
    cells = int(np.prod(padded))
    nrec = len(rec_idx)
    v = np.zeros(3 * cells)
    grad = np.zeros(cells)
    p = _problem(padded, so, nt, dt, h, 0, nrec)
    rc = oracle().sfdo_gradient(C.cast(C.pointer(p), C.c_void_p), _d(v), _d(_f64(u_history)), _d(_f64(m)),
                                _d(_f64(damp)), _d(grad), _l(_i64(rec_idx)), _d(_f64(rec_w)),
                                _d(_f64(rec_data)))
    assert rc == 0
    return grad.reshape(padded), v.reshape(3, *padded)


def forward_steps(padded, so, h, dt, nt, u, m, damp, src_idx, src_w, src_data, src_cmask,
                  t_begin, t_end):
    """Sweep + masked injection for t in [t_begin, t_end) on u (3 slots, in place)."""
    p = _problem(padded, so, nt, dt, h, len(src_idx), 0)
    cm = None if src_cmask is None else np.ascontiguousarray(src_cmask, np.uint8)
    rc = oracle().sfdo_forward_steps(C.cast(C.pointer(p), C.c_void_p), _d(u), _d(_f64(m)),
                                     _d(_f64(damp)), _l(_i64(src_idx)), _d(_f64(src_w)),
                                     _d(_f64(src_data)), cm.ctypes.data if cm is not None
                                     else None, None, None, None, None, t_begin, t_end)
    assert rc == 0


def sample_row(padded, so, h, dt, nt, u, t, rec_idx, rec_w, rec_data, rec_mask):
    p = _problem(padded, so, nt, dt, h, 0, len(rec_idx))
    pm = None if rec_mask is None else np.ascontiguousarray(rec_mask, np.uint8)
    rc = oracle().sfdo_sample_row(C.cast(C.pointer(p), C.c_void_p), _d(u), t, _l(_i64(rec_idx)),
                                  _d(_f64(rec_w)), _d(rec_data),
                                  pm.ctypes.data if pm is not None else None)
    assert rc == 0


# ---------------------------------------------------------------- reference

def ref_fd2(so):
    w = np.zeros(so + 1)
    _check_ref(ref().sfdref_fd2(so, _d(w)))
    return w


def ref_model(interior, h, nbpml, so, m_interior):
    interior = _i64(interior)
    nd = len(interior)
    padded = np.zeros(nd, np.int64)
    cells = int(np.prod(interior + 2 * (nbpml + so // 2)))
    m = np.zeros(cells)
    damp = np.zeros(cells)
    _check_ref(ref().sfdref_model(nd, _l(interior), C.c_double(h), C.c_long(nbpml), so,
                                  _d(_f64(m_interior).ravel()), _l(padded), _d(m), _d(damp)))
    return padded, m, damp


def ref_locate(interior, h, nbpml, so, m_interior, coords):
    interior = _i64(interior)
    coords = _f64(coords).reshape(-1, len(interior))
    n, nd = coords.shape
    idx = np.zeros((n, nd), np.int64)
    w = np.zeros((n, 1 << nd))
    _check_ref(ref().sfdref_locate(nd, _l(interior), C.c_double(h), C.c_long(nbpml), so,
                                   _d(_f64(m_interior).ravel()), n, _d(coords), _l(idx), _d(w)))
    return idx, w


def ref_critical_dt(interior, h, nbpml, so, m_interior):
    interior = _i64(interior)
    out = C.c_double()
    _check_ref(ref().sfdref_critical_dt(len(interior), _l(interior), C.c_double(h),
                                        C.c_long(nbpml), so, _d(_f64(m_interior).ravel()),
                                        _d_ref(out)))
    return out.value


def ref_ricker(f0, t0, nt, dt):
    out = np.zeros(nt)
    _check_ref(ref().sfdref_ricker(C.c_double(f0), C.c_double(t0), C.c_long(nt),
                                   C.c_double(dt), _d(out)))
    return out


def ref_forward(interior, h, nbpml, so, m_interior, src_coords, src_trace, rec_coords, nt, dt,
                save=False, portable=False, want_u=True):
    interior = _i64(interior)
    nd = len(interior)
    padded = interior + 2 * (nbpml + so // 2)
    cells = int(np.prod(padded))
    src_coords = _f64(src_coords).reshape(-1, nd)
    rec_coords = _f64(rec_coords).reshape(-1, nd)
    nsrc, nrec = len(src_coords), len(rec_coords)
    u = np.zeros(((nt + 1) if save else 3) * cells) if want_u else None
    rec = np.zeros(nt * nrec)
    secs = C.c_double()
    _check_ref(ref().sfdref_forward(nd, _l(interior), C.c_double(h), C.c_long(nbpml), so,
                                    _d(_f64(m_interior).ravel()), nsrc, _d(src_coords),
                                    _d(_f64(src_trace).ravel()), nrec, _d(rec_coords),
                                    C.c_long(nt), C.c_double(dt), int(save), int(portable),
                                    _d(u), _d(rec), _d_ref(secs)))
    return (u.reshape(-1, *padded) if want_u else None), rec.reshape(nt, nrec), secs.value


def ref_adjoint(interior, h, nbpml, so, m_interior, rec_coords, residual, src_coords, nt, dt,
                portable=False):
    interior = _i64(interior)
    nd = len(interior)
    padded = interior + 2 * (nbpml + so // 2)
    cells = int(np.prod(padded))
    src_coords = _f64(src_coords).reshape(-1, nd)
    rec_coords = _f64(rec_coords).reshape(-1, nd)
    nsrc, nrec = len(src_coords), len(rec_coords)
    v = np.zeros(3 * cells)
    src = np.zeros(nt * nsrc)
    secs = C.c_double()
    _check_ref(ref().sfdref_adjoint(nd, _l(interior), C.c_double(h), C.c_long(nbpml), so,
                                    _d(_f64(m_interior).ravel()), nrec, _d(rec_coords),
                                    _d(_f64(residual).ravel()), nsrc, _d(src_coords),
                                    C.c_long(nt), C.c_double(dt), int(portable), _d(v), _d(src),
                                    _d_ref(secs)))
    return v.reshape(3, *padded), src.reshape(nt, nsrc), secs.value


def ref_gradient(interior, h, nbpml, so, m_interior, rec_coords, residual, u_history, nt, dt,
                 portable=False):
    interior = _i64(interior)
    nd = len(interior)
    padded = interior + 2 * (nbpml + so // 2)
    cells = int(np.prod(padded))
    rec_coords = _f64(rec_coords).reshape(-1, nd)
    grad = np.zeros(cells)
    secs = C.c_double()
    _check_ref(ref().sfdref_gradient(nd, _l(interior), C.c_double(h), C.c_long(nbpml), so,
                                     _d(_f64(m_interior).ravel()), len(rec_coords),
                                     _d(rec_coords), _d(_f64(residual).ravel()),
                                     _d(_f64(u_history).ravel()), C.c_long(nt), C.c_double(dt),
                                     int(portable), _d(grad), _d_ref(secs)))
    return grad.reshape(padded), secs.value


def ref_generate(kind, interior, h, nbpml, so, m_interior, nsrc, nrec, nt, dt, save=False,
                 plan=0):
    """The kernel source the reference's codegen::generate emits (str)."""
    interior = _i64(interior)
    need = C.c_long()
    args = [kind, len(interior), _l(interior), C.c_double(h), C.c_long(nbpml), so,
            _d(_f64(m_interior).ravel()), C.c_long(nsrc), C.c_long(nrec), C.c_long(nt),
            C.c_double(dt), int(save), int(plan)]
    _check_ref(ref().sfdref_generate(*args, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _check_ref(ref().sfdref_generate(*args, buf, need.value, C.byref(need)))
    return buf.value.decode()


class RefProblem:
    """A reference model + sparse sets built once (sfdref_problem_create) and run
    with seismic::forward many times (the reference arm's repeated samples)."""

    def __init__(self, interior, h, nbpml, so, m_interior, src_coords, rec_coords):
        interior = _i64(interior)
        nd = len(interior)
        self.src = _f64(src_coords).reshape(-1, nd)
        self.rec = _f64(rec_coords).reshape(-1, nd)
        self.handle = ref().sfdref_problem_create(
            nd, _l(interior), C.c_double(h), C.c_long(nbpml), so, _d(_f64(m_interior).ravel()),
            len(self.src), _d(self.src), len(self.rec), _d(self.rec))
        if not self.handle:
            raise ValueError(ref().sfdref_last_error().decode())

    def forward(self, src_trace, nt, dt):
        """RunStats.seconds of one seismic::forward call (kernel call incl. first touch)."""
        secs = C.c_double()
        _check_ref(ref().sfdref_problem_forward(self.handle, _d(_f64(src_trace).ravel()),
                                                C.c_long(nt), C.c_double(dt), None,
                                                _d_ref(secs)))
        return secs.value

    def close(self):
        if self.handle:
            ref().sfdref_problem_free(self.handle)
            self.handle = None


def ref_objective(syn, obs):
    """(Phi, residual) from the reference's seismic::objective."""
    syn, obs = _f64(syn).ravel(), _f64(obs).ravel()
    res, phi = np.zeros(syn.size), C.c_double()
    _check_ref(ref().sfdref_objective(_d(syn), _d(obs), syn.size, _d(res), C.byref(phi)))
    return phi.value, res


def ref_save_model(prefix, interior, h, nbpml, so, m_interior):
    interior = _i64(interior)
    _check_ref(ref().sfdref_save_model(len(interior), _l(interior), C.c_double(h),
                                       C.c_long(nbpml), so, _d(_f64(m_interior).ravel()),
                                       str(prefix).encode()))


def ref_load_model(prefix, so):
    """(interior, h, nbpml, padded m, padded damp) as the reference loads them."""
    nd, h, nbpml = C.c_int(), C.c_double(), C.c_long()
    interior, padded = np.zeros(3, np.int64), np.zeros(3, np.int64)
    args = [str(prefix).encode(), so, C.byref(nd), _l(interior), C.byref(h), C.byref(nbpml),
            _l(padded)]
    _check_ref(ref().sfdref_load_model(*args, None, None))
    shape = tuple(int(x) for x in padded[:nd.value])
    m, damp = np.zeros(shape), np.zeros(shape)
    _check_ref(ref().sfdref_load_model(*args, _d(m), _d(damp)))
    return interior[:nd.value].copy(), h.value, nbpml.value, m, damp


def ref_save_record(prefix, data, dt, coords):
    data = _f64(data)
    coords = _f64(coords)
    nt, n = data.shape
    _check_ref(ref().sfdref_save_record(nt, C.c_double(dt), n, coords.shape[1], _d(coords),
                                        _d(data), str(prefix).encode()))


def ref_load_record(prefix):
    """(data [nt][npoints], dt, coords [npoints][ndim]) as the reference loads them."""
    nt, dt, n, nd = C.c_long(), C.c_double(), C.c_long(), C.c_int()
    args = [str(prefix).encode(), C.byref(nt), C.byref(dt), C.byref(n), C.byref(nd)]
    _check_ref(ref().sfdref_load_record(*args, None, None))
    coords = np.zeros((n.value, nd.value))
    data = np.zeros((nt.value, n.value))
    _check_ref(ref().sfdref_load_record(*args, _d(coords), _d(data)))
    return data, dt.value, coords


def ref_dump_grid(prefix, data, halo, time_slots):
    data = _f64(data)
    shape = _i64(data.shape)
    _check_ref(ref().sfdref_dump_grid(_d(data), len(shape), _l(shape), C.c_long(halo),
                                      C.c_long(time_slots), str(prefix).encode()))


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    if a.size != b.size:
        raise ValueError(f"size mismatch {a.size} vs {b.size}")
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a - b))
