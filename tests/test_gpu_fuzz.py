"""Seeded random operator cases on the B200 against the fp64 oracle: shapes
(odd, non-cubic, thin in any axis), space orders 2-16, 2-D and 3-D, random
smooth velocities, 0-5 sources and 0-40 receivers anywhere in the interior
(edges included), random damping-layer widths, forward (rolling and saved),
adjoint and gradient, each through the public operator API.  Wavefields,
traces and source samples within rel-L2 1e-5 (the north star's gate), the
saved history's slack row and rows 0 / 1 exactly zero, nothing non-finite.
The gradient gets 5e-5 here: it sums u[t] times the second time difference of
the adjoint field, which is smaller than the field by (omega dt)^2 (~6e-3 for
these pulses), so the fp32 rounding of the stored v rows reaches the gradient
amplified by ~1/(omega dt)^2; on the BASELINE configurations' full runs it
stays at 1e-6 .. 2e-6 (tests/test_gpu_protocol.py gates them at 1e-5).  A
600-case run of this file (profiles/r02q/fuzz600.txt) passes every wavefield,
record and adjoint gate; two 2-D so-2 gradients land at 5.1e-5 and 8.8e-5 with
their forward / adjoint fields at 1e-7 / 4e-7 (that floor, tools/fuzz_case.py)."""
import os

import numpy as np
import pytest

import oracle_lib as O
from paper_1608_08658_b200 import seismic as S

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    nd = 3 if seed % 3 else 2
    so = int(rng.choice([2, 4, 6, 8, 10, 12, 14, 16] if nd == 3 else [2, 4, 6, 8]))
    lo, hi = (9, 30) if nd == 3 else (20, 90)
    interior = [int(rng.integers(lo, hi)) for _ in range(nd)]
    h = float(rng.choice([5.0, 10.0, 12.5]))
    nbpml = int(rng.integers(2, 12))
    v = 1500.0 + 2500.0 * rng.random(interior)
    for ax in range(nd):  # a little smoothing so the field is physical
        v = 0.5 * v + 0.25 * (np.roll(v, 1, ax) + np.roll(v, -1, ax))
    m = O._f64((1.0 / v ** 2).astype(np.float32))
    model = S.make_model(interior, h, nbpml, so, m.ravel())
    dt = float(rng.uniform(0.3, 0.9)) * S.critical_dt(model)
    nt = int(rng.integers(20, 90))
    span = [(n - 1) * h for n in interior]
    nsrc, nrec = int(rng.integers(0, 6)), int(rng.integers(0, 41))

    def points(n):
        c = rng.random((n, nd)) * np.array(span)
        if n:  # one point exactly on the far corner of the interior
            c[0] = span
        return c

    src = S.locate_points(model, points(nsrc))
    rec = S.locate_points(model, points(nrec))
    f0 = 0.05 / dt / 4
    wav = O._f64(np.outer(S.ricker(f0, 1.2 / f0, nt, dt), 1.0 + rng.random(nsrc)).astype(np.float32))
    return model, src, rec, wav, nt, dt


def _close(a, b, tol=TOL):
    a, b = np.asarray(a), np.asarray(b)
    assert np.all(np.isfinite(a))
    if not np.any(b):
        return np.array_equal(a, b)
    return O.rel_l2(a, b) <= tol


# SFDB200_FUZZ_CASES widens the campaign (profiles/ keeps the log of a 600-case run)
@pytest.mark.parametrize("seed", range(int(os.environ.get("SFDB200_FUZZ_CASES", "48"))))
def test_random_operator_case(seed):
    model, src, rec, wav, nt, dt = _case(seed)
    P, so, h = model.padded, model.space_order, model.h
    save = seed % 2 == 0
    f = S.forward(model, src, wav, rec, nt, dt, save)
    uo, ro = O.forward(P, so, h, dt, nt, model.m, model.damp, src.idx, src.w, wav, rec.idx,
                       rec.w, save=save)
    assert _close(f.u, uo) and _close(f.record.data, ro)
    if save:
        u = np.asarray(f.u)
        assert not u[0].any() and not u[1].any() and not u[nt].any()
    if rec.npoints:
        # band-limited residual traces (white noise convolved with the source
        # pulse along time, as verify.cpp band_limited_noise builds them): the
        # imaging condition takes the second time derivative of the adjoint
        # field, which white noise injected every step would make the fp32
        # cancellation test of, not of the operator
        white = np.random.default_rng(seed).standard_normal((nt, rec.npoints))
        pulse = S.ricker(0.05 / dt / 4, 1.2 * 4 * dt / 0.05, nt, dt)
        smooth = np.stack([np.convolve(white[:, r], pulse)[:nt] for r in range(rec.npoints)], 1)
        resid = O._f64((smooth / np.abs(smooth).max()).astype(np.float32))
        rs = S.ShotRecord(nt, dt, rec.npoints, resid)
        a = S.adjoint(model, rec, rs, src, nt, dt)
        vo, so_ = O.adjoint(P, so, h, dt, nt, model.m, model.damp, src.idx, src.w, rec.idx,
                            rec.w, resid)
        assert _close(a.v, vo) and _close(a.src_samples.data, so_)
        us = uo if save else O.forward(P, so, h, dt, nt, model.m, model.damp, src.idx, src.w,
                                       wav, rec.idx, rec.w, save=True)[0]
        g = S.gradient(model, rec, rs, us, nt, dt)
        go, _ = O.gradient(P, so, h, dt, nt, model.m, model.damp, us, rec.idx, rec.w, resid)
        assert _close(g.grad, go, 5e-5)
