"""ctypes binding of the C ABI in include/sfdb200.h (libsfdb200.so, in-tree).

No fallback: if the CUDA library is missing or a call fails, this raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libsfdb200.so")

FORWARD, ADJOINT, GRADIENT = 0, 1, 2
OK, EINVAL, ECUDA, ENOMEM, ENONFINITE = 0, 1, 2, 3, 4


class Desc(C.Structure):
    """sfdb200_desc (include/sfdb200.h)."""

    _fields_ = [("kind", C.c_int), ("ndim", C.c_int), ("padded", C.c_long * 3),
                ("space_order", C.c_int), ("nt", C.c_long), ("dt", C.c_double),
                ("h", C.c_double), ("nsrc", C.c_long), ("nrec", C.c_long), ("save", C.c_int),
                ("device", C.c_int), ("flags", C.c_int)]


F_GRAD_NO_ROW2 = 1  # SFDB200_F_GRAD_NO_ROW2


class SfdError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InvalidArgument(SfdError, ValueError):
    """Mirrors the reference's std::invalid_argument."""


_i, _L, _D, _P = C.c_int, C.c_long, C.c_double, C.c_void_p
_dp, _lp = C.POINTER(C.c_double), C.POINTER(C.c_long)
_SIGS = {
    "sfdb200_call": (_i, [_P, _P]),
    "sfdb200_plan_create": (_i, [_P, _P]),
    "sfdb200_plan_destroy": (_i, [_P]),
    "sfdb200_run": (_i, [_P, _P]),
    "sfdb200_upload": (_i, [_P, _P]),
    "sfdb200_execute": (_i, [_P]),
    "sfdb200_download": (_i, [_P, _P]),
    "sfdb200_bind_history": (_i, [_P, _P]),
    "sfdb200_set_checkpointing": (_i, [_P, _L]),
    "sfdb200_bind_checkpoints": (_i, [_P, _P]),
    "sfdb200_checkpoint_bytes": (_L, [_P]),
    "sfdb200_set_stream": (_i, [_P, _P]),
    "sfdb200_set_timing": (_i, [_P, _i]),
    "sfdb200_stencil_time": (_i, [_P, _dp, _lp]),
    "sfdb200_launches_per_execute": (_L, [_P]),
    "sfdb200_points_per_step": (_L, [_P]),
    "sfdb200_steps": (_L, [_P]),
    "sfdb200_h2d_bytes": (_L, [_P]),
    "sfdb200_plan_info": (_i, [_P, C.c_char_p, _L]),
    "sfdb200_d2h_bytes": (_L, [_P]),
    "sfdb200_comm_unique_id": (_i, [_P]),
    "sfdb200_comm_create": (_i, [_P, _i, _i, _i, _P]),
    "sfdb200_comm_destroy": (_i, [_P]),
    "sfdb200_comm_create_loopback": (_i, [_i, _i, _i, _P]),
    "sfdb200_execute_group": (_i, [_P, _i]),
    "sfdb200_plan_ipc_export": (_i, [_P, _P]),
    "sfdb200_plan_ipc_import": (_i, [_P, _P, _P]),
    "sfdb200_plan_peer_group": (_i, [_P, _i]),
    "sfdb200_p2p_selftest": (_i, [_i]),
    "sfdb200_plan_check": (_i, [_P]),
    "sfdb200_plan_abort": (_i, [_P]),
    "sfdb200_objective": (_i, [_dp, _dp, _L, _dp, _dp]),
    "sfdb200_plan_create_dist": (_i, [_P, _P, _P]),
    "sfdb200_slab": (_i, [_L, _i, _i, _i, _lp, _lp]),
    "sfdb200_plan_slab": (_i, [_P, _lp, _lp, _lp]),
    "sfdb200_slab_owns": (_i, [_L, _i, _i, _i, _L, _i, _lp, _P, _P]),
    "sfdb200_fd2": (_i, [_i, _dp]),
    "sfdb200_make_model": (_i, [_i, _lp, _D, _L, _i, _dp, _lp, _dp, _dp]),
    "sfdb200_build_damping": (_i, [_i, _lp, _L, _L, _D, _dp]),
    "sfdb200_locate_points": (_i, [_i, _lp, _D, _L, _i, _L, _dp, _lp, _dp]),
    "sfdb200_damp_separable": (_i, [_dp, _L, _L, _L, _dp]),
    "sfdb200_ricker": (_i, [_D, _D, _L, _D, _dp]),
    "sfdb200_critical_dt": (_D, [_i, _D, _i, _D]),
    "sfdb200_last_error": (C.c_char_p, []),
    "sfdb200_version": (C.c_char_p, []),
}
EXPORTS = tuple(_SIGS)

_lib = None


DEBUG_LIB_PATH = os.path.join(PKG_DIR, "libsfdb200_debug.so")


def lib_path():
    """libsfdb200.so, or with SFDB200_LIBRARY=debug the build whose kernels
    check every global access they make (csrc/kernels.cuh SFDB_CHECK)."""
    sel = os.environ.get("SFDB200_LIBRARY", "")
    if sel == "debug":
        return DEBUG_LIB_PATH
    if sel.endswith(".so"):  # an experiment build (tools/build_probe.sh)
        return sel if os.path.isabs(sel) else os.path.join(PKG_DIR, sel)
    return LIB_PATH


def lib():
    """Loads libsfdb200.so (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
        lib_ = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib_, name)
            f.restype = res
            f.argtypes = args
        _lib = lib_
    return _lib


def check(rc):
    if rc != OK:
        msg = lib().sfdb200_last_error().decode()
        if rc == EINVAL:
            raise InvalidArgument(rc, msg)
        raise SfdError(rc, msg)


def dptr(a):
    return a.ctypes.data_as(_dp)


def lptr(a):
    return a.ctypes.data_as(_lp)


def argv_of(arrays):
    """void*[] over numpy arrays (None -> NULL), keeping the arrays alive."""
    arr = (C.c_void_p * len(arrays))()
    for i, a in enumerate(arrays):
        arr[i] = None if a is None else a.ctypes.data
    return arr


class Plan:
    """Owning handle of an sfdb200_plan."""

    def __init__(self, kind, ndim, padded, space_order, nt, dt, h, nsrc, nrec, save=False,
                 device=0, comm=None):
        d = Desc()
        d.kind, d.ndim, d.space_order = kind, ndim, space_order
        for i in range(3):
            d.padded[i] = int(padded[i]) if i < len(padded) else 0
        d.nt, d.dt, d.h, d.nsrc, d.nrec = int(nt), float(dt), float(h), int(nsrc), int(nrec)
        d.save, d.device = int(bool(save)), int(device)
        self.desc = d
        h_ = C.c_void_p()
        if comm is None:
            check(lib().sfdb200_plan_create(C.byref(d), C.byref(h_)))
        else:
            check(lib().sfdb200_plan_create_dist(C.byref(d), comm.handle, C.byref(h_)))
        self.handle = h_
        self.comm = comm
        self._keep = None

    def close(self):
        if self.handle:
            lib().sfdb200_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, arrays):
        self._keep = arrays
        check(lib().sfdb200_upload(self.handle, argv_of(arrays)))

    def execute(self):
        check(lib().sfdb200_execute(self.handle))

    def check(self):
        """Waits for the plan's stream; raises if the P2P exchange timed out."""
        check(lib().sfdb200_plan_check(self.handle))

    def abort(self):
        """Marks the P2P exchange broken on this rank and its neighbours now."""
        check(lib().sfdb200_plan_abort(self.handle))

    def download(self, arrays):
        check(lib().sfdb200_download(self.handle, argv_of(arrays)))

    def run(self, arrays):
        self._keep = arrays  # the caller's buffers outlive every copy of the call
        check(lib().sfdb200_run(self.handle, argv_of(arrays)))

    def bind_history(self, forward_plan):
        check(lib().sfdb200_bind_history(self.handle, forward_plan.handle))
        self._hist_fwd = forward_plan  # keep it alive while bound

    def set_checkpointing(self, interval):
        """Forward plans: keep restart rows every `interval` steps (0: off)."""
        check(lib().sfdb200_set_checkpointing(self.handle, int(interval)))

    def bind_checkpoints(self, forward_plan):
        """Gradient plans: recompute the u history from a checkpointing forward plan."""
        check(lib().sfdb200_bind_checkpoints(self.handle, forward_plan.handle))
        self._ck_fwd = forward_plan  # keep it alive while bound

    @property
    def checkpoint_bytes(self):
        return int(lib().sfdb200_checkpoint_bytes(self.handle))

    def set_stream(self, stream_handle):
        check(lib().sfdb200_set_stream(self.handle, C.c_void_p(stream_handle or None)))

    def set_timing(self, on):
        check(lib().sfdb200_set_timing(self.handle, int(bool(on))))

    def stencil_time(self):
        ms = C.c_double()
        n = C.c_long()
        check(lib().sfdb200_stencil_time(self.handle, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def info(self):
        import json
        buf = C.create_string_buffer(1024)
        check(lib().sfdb200_plan_info(self.handle, buf, 1024))
        return json.loads(buf.value.decode())

    def slab(self):
        zb, ze, zo = C.c_long(), C.c_long(), C.c_long()
        check(lib().sfdb200_plan_slab(self.handle, C.byref(zb), C.byref(ze), C.byref(zo)))
        return zb.value, ze.value, zo.value

    @property
    def launches_per_execute(self):
        return lib().sfdb200_launches_per_execute(self.handle)

    @property
    def points_per_step(self):
        return lib().sfdb200_points_per_step(self.handle)

    @property
    def steps(self):
        return lib().sfdb200_steps(self.handle)

    @property
    def h2d_bytes(self):
        return lib().sfdb200_h2d_bytes(self.handle)

    @property
    def d2h_bytes(self):
        return lib().sfdb200_d2h_bytes(self.handle)

    def ipc_export(self) -> bytes:
        """This rank's blob for the fused P2P ghost exchange (sfdb200_plan_ipc_export)."""
        buf = C.create_string_buffer(IPC_BYTES)
        check(lib().sfdb200_plan_ipc_export(self.handle, buf))
        return buf.raw

    def ipc_import(self, lower, upper):
        """Open the neighbours' blobs (None at a slab end) and switch to the P2P
        exchange; raises InvalidArgument (plan keeps NCCL) without peer access."""
        lo = C.create_string_buffer(bytes(lower), IPC_BYTES) if lower is not None else None
        hi = C.create_string_buffer(bytes(upper), IPC_BYTES) if upper is not None else None
        check(lib().sfdb200_plan_ipc_import(self.handle, lo, hi))


class Comm:
    """sfdb200_comm: the z-slab ranks' NCCL communicator (one per GPU process)."""

    def __init__(self, unique_id: bytes, world: int, rank: int, device: int):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        h = C.c_void_p()
        check(lib().sfdb200_comm_create(buf, world, rank, device, C.byref(h)))
        self.handle, self.world, self.rank, self.device = h, world, rank, device

    @classmethod
    def loopback(cls, world: int, rank: int, device: int = 0):
        """An emulated rank for the one-GPU harness (execute_group)."""
        c = cls.__new__(cls)
        h = C.c_void_p()
        check(lib().sfdb200_comm_create_loopback(world, rank, device, C.byref(h)))
        c.handle, c.world, c.rank, c.device = h, world, rank, device
        return c

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().sfdb200_comm_unique_id(buf))
        return buf.raw

    def close(self):
        if self.handle:
            lib().sfdb200_comm_destroy(self.handle)
            self.handle = None


IPC_BYTES = 256  # SFDB200_IPC_BYTES


def peer_group(plans):
    """Loopback harness: the emulated ranks store into each other's ghost
    planes from their boundary sweeps (the fused P2P exchange on one GPU)."""
    arr = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
    check(lib().sfdb200_plan_peer_group(arr, len(plans)))


def execute_group(plans):
    arr = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
    check(lib().sfdb200_execute_group(arr, len(plans)))


def slab(padded_z, space_order, world, rank):
    zb, ze = C.c_long(), C.c_long()
    check(lib().sfdb200_slab(int(padded_z), int(space_order), int(world), int(rank),
                             C.byref(zb), C.byref(ze)))
    return zb.value, ze.value


def slab_owns(padded_z, space_order, world, rank, idx):
    idx = i64(idx)
    n, nd = idx.shape
    cm = np.zeros((n, 1 << nd), np.uint8)
    pm = np.zeros(n, np.uint8)
    check(lib().sfdb200_slab_owns(int(padded_z), int(space_order), int(world), int(rank), n, nd,
                                  lptr(idx), cm.ctypes.data, pm.ctypes.data))
    return cm.astype(bool), pm.astype(bool)


def call(kind, ndim, padded, space_order, nt, dt, h, nsrc, nrec, save, arrays, device=0):
    """sfdb200_call: the `<Name>_call(argv)` drop-in with a descriptor."""
    d = Desc()
    d.kind, d.ndim, d.space_order = kind, ndim, space_order
    for i in range(3):
        d.padded[i] = int(padded[i]) if i < len(padded) else 0
    d.nt, d.dt, d.h, d.nsrc, d.nrec = int(nt), float(dt), float(h), int(nsrc), int(nrec)
    d.save, d.device = int(bool(save)), int(device)
    check(lib().sfdb200_call(C.byref(d), argv_of(arrays)))


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)
