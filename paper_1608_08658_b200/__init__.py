"""B200-native (sm_100a) backend for the damped acoustic stencil hot path of
stencilfd (the Devito paper's seismic operators, arXiv:1608.08658).

The product is libsfdb200.so (C ABI in include/sfdb200.h); this package is the
host-side mirror of the reference's ``sfd::seismic`` operator API over it.
"""
from . import _lib
from .seismic import (AdjointResult, ForwardResult, GradientResult, RunConfig, ShotRecord,
                      SparsePoints, VelocityModel, add_interior, adjoint, build_damping,
                      critical_dt, forward, gradient, history_rows, load_model, load_record,
                      locate_points, make_constant_model, make_model, objective,
                      restrict_interior, ricker, save_model, save_record, zero_record)

__all__ = [
    "AdjointResult", "ForwardResult", "GradientResult", "RunConfig", "ShotRecord",
    "SparsePoints", "VelocityModel", "add_interior", "adjoint", "build_damping", "critical_dt",
    "forward", "gradient", "history_rows", "load_model", "load_record", "locate_points",
    "make_constant_model", "make_model", "objective", "restrict_interior", "ricker",
    "save_model", "save_record", "zero_record", "_lib",
]
