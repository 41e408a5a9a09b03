"""Physics checks of the reference's own test suite (proj/tests/test_seismic.cpp:
first arrival :190-218, energy decay :243-278, spike time reversal :280-306,
gradient against a directional finite difference :308-360), restated for the
B200 operators.  Tolerances that the reference states for fp64 are re-derived
for fp32 where noted."""
import dataclasses

import numpy as np
import pytest

from paper_1608_08658_b200 import seismic as S

pytestmark = pytest.mark.gpu


def test_first_arrival_matches_ray_travel_time():
    """A 20 Hz pulse from the centre of a 1500 m/s box peaks at a receiver
    450 m away at t0 + 450/1500 (within two cells of travel and two steps),
    and the trace is quiet before the wave can arrive."""
    m = S.make_constant_model([65, 65], 15.0, 12, 4, 1500.0)
    dt = 0.8 * S.critical_dt(m)
    nt, t0 = 220, 0.05
    src = S.locate_points(m, [[32 * 15.0, 32 * 15.0]])
    rec = S.locate_points(m, [[32 * 15.0, 62 * 15.0]])
    f = S.forward(m, src, S.ricker(20.0, t0, nt, dt), rec, nt, dt, False)
    trace = f.record.data[:, 0]
    expected = t0 + 450.0 / 1500.0
    window = int((t0 + 510.0 / 1500.0) / dt)  # before the first boundary bounce
    assert window < nt
    tpeak = int(np.argmax(np.abs(trace[:window])))
    peak = abs(trace[tpeak])
    assert peak > 0
    assert abs(tpeak * dt - expected) < 2.0 * 15.0 / 1500.0 + 2.0 * dt
    quiet = int(np.ceil(0.22 / dt))
    assert np.all(np.abs(trace[:quiet]) < 0.01 * peak)


def _small_model():
    return S.make_constant_model([33, 33], 15.0, 10, 4, 1500.0)


def test_energy_decays_after_the_source_stops():
    """Once the source is quiet no row's energy tops the running peak by more
    than 5 %, and the absorbing layer drains the box over the run."""
    m = _small_model()
    dt = 0.9 * S.critical_dt(m)
    nt, f0 = 220, 25.0
    src = S.locate_points(m, [[240.0, 240.0]])
    rec = S.locate_points(m, [[100.0, 380.0]])
    f = S.forward(m, src, S.ricker(f0, 1.0 / f0, nt, dt), rec, nt, dt, True)
    u = np.asarray(f.u).reshape(nt + 1, -1)[:nt]
    energy = (u * u).sum(axis=1)
    cutoff = int(np.ceil(2.5 / f0 / dt))
    peak = energy[cutoff]
    for t in range(cutoff + 1, nt):
        assert energy[t] <= peak * 1.05, t
        peak = max(peak, energy[t])
    window = 4 * int(np.ceil(1.0 / (f0 * dt)))
    head = energy[cutoff:cutoff + window].max()
    tail = energy[nt - window:].max()
    assert tail <= 0.6 * head


def test_adjoint_of_a_spike_is_the_time_reversed_response():
    """Forward from a spike at A sampled at B, against the adjoint from a
    spike at B sampled at A: adj[rho] == fwd[tk - rho + rho0].  The reference
    asserts 1e-8 of the peak in fp64; fp32 rounding of ~150 steps gives
    ~1e-6, asserted at 2e-5."""
    m = S.make_constant_model([33, 33], 15.0, 10, 2, 1500.0)
    dt = 0.9 * S.critical_dt(m)
    nt, rho0, tk = 150, 20, 120
    a = S.locate_points(m, [[120.0, 150.0]])
    b = S.locate_points(m, [[330.0, 345.0]])
    x = np.zeros((nt, 1))
    x[rho0, 0] = 1.0
    f = S.forward(m, a, x, b, nt, dt, False)
    spike = S.zero_record(nt, dt, 1)
    spike.data[tk, 0] = 1.0
    adj = S.adjoint(m, b, spike, a, nt, dt)
    fwd, back = f.record.data[:, 0], adj.src_samples.data[:, 0]
    peak = np.abs(fwd).max()
    assert peak > 0
    checked = 0
    for rho in range(1, nt - 1):
        tau = tk - rho + rho0
        if tau < 2 or tau >= nt:
            continue
        assert abs(back[rho] - fwd[tau]) <= 2e-5 * peak, rho
        checked += 1
    assert checked > 50


def test_gradient_matches_a_directional_finite_difference():
    """<grad, dm> against (Phi(m + h dm) - Phi(m - h dm)) / 2h within 1 %
    (h = 1e-2 instead of the reference's 1e-3 so the fp32 objectives resolve
    the difference), and a zero residual gives an exactly zero gradient."""
    m = _small_model()
    dt = 0.85 * S.critical_dt(m)
    nt = 130
    src = S.locate_points(m, [[243.7, 40.0]])
    rec = S.locate_points(m, [[100.0, 400.0], [250.0, 401.5], [380.0, 404.9]])
    wav = S.ricker(18.0, 1.0 / 18.0, nt, dt)
    i, j = np.meshgrid(np.arange(33), np.arange(33), indexing="ij")
    r2 = (i - 20.0) ** 2 + (j - 14.0) ** 2
    mi = (1.0 / 1500.0 ** 2) * (1.0 + 0.05 * np.exp(-r2 / 30.0))
    observed = S.forward(S.make_model([33, 33], 15.0, 10, 4, mi.ravel()), src, wav, rec, nt, dt,
                         False).record
    base = S.forward(m, src, wav, rec, nt, dt, True)
    phi0, resid = S.objective(base.record, observed, want_residual=True)
    assert phi0 > 0
    g = S.gradient(m, rec, resid, base.u, nt, dt)
    rng = np.random.default_rng(23)
    dmi = rng.uniform(-1.0, 1.0, 33 * 33) * 2e-8
    dm = np.zeros(m.cells())
    S.add_interior(m, dmi, 1.0, dm)
    gdot = float(np.dot(np.asarray(g.grad).ravel(), dm))
    h = 1e-2
    up = dataclasses.replace(m, m=np.asarray(m.m) + h * dm)
    down = dataclasses.replace(m, m=np.asarray(m.m) - h * dm)
    phi_up = S.objective(S.forward(up, src, wav, rec, nt, dt, False).record, observed)
    phi_down = S.objective(S.forward(down, src, wav, rec, nt, dt, False).record, observed)
    fd = (phi_up - phi_down) / (2.0 * h)
    assert abs(fd - gdot) <= 0.01 * abs(fd)
    g0 = S.gradient(m, rec, S.zero_record(nt, dt, 3), base.u, nt, dt)
    assert np.all(np.asarray(g0.grad) == 0.0)
