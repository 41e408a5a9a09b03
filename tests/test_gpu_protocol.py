"""SURVEY §8(d) parity protocol at FULL step counts on the B200.

Each BASELINE config runs with its full number of time steps on the reduced
grid the survey fixes for the fp64 oracle:

  cfg1  201^2 + 40, so 4, 1000 steps                (full size)
  cfg2  128^3 + 40, so 8, 1000 steps, 128^2 carpet
  cfg3   64^3 + 20, so 8, 800-step forward(save) -> objective -> gradient
  cfg4  128^3 + 40, 200 steps, so in {2, 4, 8, 12, 16}
  cfg5  192^3 + 40, so 16, 500 steps, 4 sources, 96^2 carpet; plus the
        z-slab decomposition over 2 / 4 / 8 emulated ranks, bitwise equal to
        the one-GPU run (no two injection corners collide in cfg5)

The checker is the UNMODIFIED reference (oracle/_ref/libsfdref.so: its own
JIT-compiled OpenMP C through sfd::seismic::forward/adjoint/gradient,
proj/src/seismic.cpp:333-496) when it was built, else the C restatement
(oracle/libsfdoracle.so, pinned to the reference at <= 1e-12 by
tests/test_oracle.py).  Gate (BASELINE.json north_star): rel-L2 <= 1e-5 on
the final three slots, the traces and grad; indices bit-exact.  Every
achieved error is appended to gpurun_out/parity/protocol.jsonl (copied to
profiles/ per round).
"""
import json
import os
import time

import numpy as np
import pytest

import oracle_lib as O
from paper_1608_08658_b200 import _lib as L
from paper_1608_08658_b200 import configs, seismic as S

TOL = 1e-5
pytestmark = pytest.mark.gpu

LOG = os.path.join(O.ROOT, "gpurun_out", "parity", "protocol.jsonl")


def _log(case, **kv):
    os.makedirs(os.path.dirname(LOG), exist_ok=True)
    kv = {k: (float(v) if isinstance(v, (np.floating, float)) else v) for k, v in kv.items()}
    with open(LOG, "a") as fh:
        fh.write(json.dumps({"case": case, "checker": _checker(), **kv}) + "\n")


def _checker():
    return "reference (oracle/_ref)" if O.have_ref() else "C restatement (oracle/libsfdoracle.so)"


def _setup(w):
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    src = S.locate_points(model, w.src_coords)
    rec = S.locate_points(model, w.rec_coords)
    return model, src, rec


def _oracle_forward(w, model, src, rec, save=False):
    """(u, record, checker seconds) from the reference when built, else the port."""
    t0 = time.perf_counter()
    if O.have_ref():
        u, r, _ = O.ref_forward(w.interior, w.h, w.nbpml, w.space_order, w.m_interior,
                                w.src_coords, w.wavelet, w.rec_coords, w.nt, w.dt, save=save)
    else:
        u, r = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                         src.idx, src.w, w.wavelet, rec.idx, rec.w, save=save)
    return u, r, time.perf_counter() - t0


def _oracle_gradient(w, model, rec, resid, hist):
    if O.have_ref():
        g, _ = O.ref_gradient(w.interior, w.h, w.nbpml, w.space_order, w.m_interior,
                              w.rec_coords, resid, hist, w.nt, w.dt)
        return g
    g, _ = O.gradient(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp, hist,
                      rec.idx, rec.w, resid)
    return g


def _check_indices(w, model, src, rec):
    """idx + fp64 weights bit-exact against the reference's locate_points."""
    if not O.have_ref():
        return
    for pts, c in ((src, w.src_coords), (rec, w.rec_coords)):
        if len(c) == 0:
            continue
        idx, wt = O.ref_locate(w.interior, w.h, w.nbpml, w.space_order, w.m_interior, c)
        assert np.array_equal(pts.idx, idx) and np.array_equal(pts.w, wt)


def _last_slots(u, nt):
    """The three rolling slots in time order t = nt-3, nt-2, nt-1."""
    return [u[t % 3] for t in (nt - 3, nt - 2, nt - 1)]


def _forward_case(name, w):
    model, src, rec = _setup(w)
    _check_indices(w, model, src, rec)
    t0 = time.perf_counter()
    f = S.forward(model, src, w.wavelet, rec, w.nt, w.dt, False)
    t_gpu = time.perf_counter() - t0
    uo, ro, t_ora = _oracle_forward(w, model, src, rec)
    errs = [O.rel_l2(a, b) for a, b in zip(_last_slots(f.u, w.nt), _last_slots(uo, w.nt))]
    er = O.rel_l2(f.record.data, ro) if rec.npoints else 0.0
    _log(name, padded=list(map(int, model.padded)), so=w.space_order, steps=w.nt - 2,
         nsrc=src.npoints, nrec=rec.npoints, slot_rel_l2=errs, record_rel_l2=er,
         gpu_call_s=t_gpu, checker_s=t_ora)
    assert max(errs) <= TOL, (name, errs)
    assert er <= TOL, (name, er)
    assert np.all(f.record.data[:2] == 0)
    return f, model, src, rec


def test_protocol_cfg1_full():
    _forward_case("cfg1 201^2+40 so4 1000 steps", configs.cfg1())


def test_protocol_cfg2_128():
    _forward_case("cfg2 128^3+40 so8 1000 steps",
                  configs.cfg2(n=128, nt=1002, nbpml=40, nrec_side=128))


@pytest.mark.parametrize("so", [2, 4, 8, 12, 16])
def test_protocol_cfg4_128(so):
    _forward_case(f"cfg4 128^3+40 so{so} 200 steps", configs.cfg4(so, n=128, nt=202, nbpml=40))


def test_protocol_cfg3_64_fwi_gradient():
    """forward(save) of the true model -> observed; forward(save) of the
    background -> synthetic + history; objective; gradient.  Gated on the
    operators with identical inputs (the reference API's contract: the
    gradient takes the caller's residual and history), and the whole chain
    kept on the device (fwi_gradient, full history and checkpointed) logged
    against the checker's chain."""
    w = configs.cfg3(n=64, nt=802, nbpml=20, nrec_side=64)
    model_t, src, rec = _setup(w)
    _check_indices(w, model_t, src, rec)
    # observed data: the true model through both sides
    ft = S.forward(model_t, src, w.wavelet, rec, w.nt, w.dt, False)
    _, obs, _ = _oracle_forward(w, model_t, src, rec)
    e_obs = O.rel_l2(ft.record.data, obs)
    # background forward with the saved history
    wb = configs.Workload(w.name + "-bg", 3, w.interior, w.space_order, w.nt, w.dt,
                          w.extra["m_background"], w.wavelet, w.src_coords, w.rec_coords, w.h,
                          w.nbpml, w.f0)
    model, _, _ = _setup(wb)
    fb = S.forward(model, src, wb.wavelet, rec, wb.nt, wb.dt, True)
    hist, syn, _ = _oracle_forward(wb, model, src, rec, save=True)
    e_syn = O.rel_l2(fb.record.data, syn)
    e_hist = [O.rel_l2(fb.u[t], hist[t]) for t in (w.nt - 3, w.nt - 2, w.nt - 1)]
    del fb
    phi_o, resid_o = S.objective(S.ShotRecord(w.nt, w.dt, rec.npoints, syn),
                                 S.ShotRecord(w.nt, w.dt, rec.npoints, obs), True)
    g_o = _oracle_gradient(wb, model, rec, resid_o.data, hist)
    # the gradient operator on identical inputs
    t0 = time.perf_counter()
    g = S.gradient(model, rec, resid_o, hist, w.nt, w.dt)
    t_g = time.perf_counter() - t0
    e_grad = O.rel_l2(g.grad, g_o)
    del hist
    # the device-resident chain against the checker's chain
    obs_rec = S.ShotRecord(w.nt, w.dt, rec.npoints, obs)
    chain = S.fwi_gradient(model, src, wb.wavelet, rec, obs_rec, w.nt, w.dt,
                           checkpoint_interval=0)
    ck = S.fwi_gradient(model, src, wb.wavelet, rec, obs_rec, w.nt, w.dt,
                        checkpoint_interval=28)
    e_chain = O.rel_l2(chain.grad, g_o)
    e_chain_phi = abs(chain.phi - phi_o) / phi_o
    e_ck = O.rel_l2(ck.grad, chain.grad)
    _log("cfg3 64^3+20 so8 800-step fwd(save)->objective->gradient",
         padded=list(map(int, model.padded)), steps=w.nt - 2, nrec=rec.npoints,
         observed_record_rel_l2=e_obs, synthetic_record_rel_l2=e_syn, history_last3_rel_l2=e_hist,
         gradient_op_rel_l2=e_grad, gradient_op_s=t_g, chain_grad_rel_l2=e_chain,
         chain_phi_rel=e_chain_phi, checkpointed_vs_full_rel_l2=e_ck,
         residual_norm_over_record_norm=float(np.linalg.norm(resid_o.data) /
                                              np.linalg.norm(syn)))
    assert e_obs <= TOL and e_syn <= TOL and max(e_hist) <= TOL
    assert e_grad <= TOL
    assert e_chain_phi <= 1e-4
    assert e_ck <= 1e-6


def _emulated_forward(w, model, src, rec, world):
    """The z-slab decomposition over `world` emulated ranks on one GPU (the real
    kernels, tables and fused peer stores; ghost planes delivered into each
    other's rows), assembled on the host."""
    import torch
    stream = torch.cuda.Stream()
    comms = [L.Comm.loopback(world, r, 0) for r in range(world)]
    plans, outs = [], []
    wav = O._f64(w.wavelet)
    try:
        for r in range(world):
            p = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                       rec.npoints, False, 0, comm=comms[r])
            p.set_stream(stream.cuda_stream)
            field = np.zeros((3, *model.padded))
            tr = np.zeros((w.nt, rec.npoints))
            plans.append(p)
            outs.append(([field, model.m, model.damp, src.idx, src.w, wav, rec.idx, rec.w, tr],
                         field, tr))
        L.peer_group(plans)
        for p, (argv, _, _) in zip(plans, outs):
            p.upload(argv)
        L.execute_group(plans)
        field = np.zeros((3, *model.padded))
        trace = np.zeros((w.nt, rec.npoints))
        for p, (argv, f, tr) in zip(plans, outs):
            p.download(argv)
            field += f     # every plane / receiver has exactly one owner
            trace += tr
        return field, trace
    finally:
        for p in plans:
            p.close()
        for c in comms:
            c.close()


def test_protocol_cfg5_192_and_slabs(monkeypatch):
    """cfg5 at 192^3 so 16 (500 steps, 4 sources) against the checker, then the
    same problem z-slab-decomposed over 2 / 4 / 8 emulated ranks: bitwise equal
    to the one-GPU run.  One tiling for every plan, so the only
    difference between the runs is the decomposition."""
    monkeypatch.setenv("SFDB200_TILE", "4,2,4,4,1")  # by,ny,stages,rot,pair
    w = configs.cfg5(n=192, nt=502, nbpml=40, nrec_side=96)
    f, model, src, rec = _forward_case("cfg5 192^3+40 so16 500 steps 4 src", w)
    # no two injection corners share a cell (the bitwise precondition)
    cells = [tuple(i + np.array([(c >> 2) & 1, (c >> 1) & 1, c & 1]))
             for i in src.idx for c in range(8)]
    assert len(set(cells)) == len(cells)
    diffs = {}
    for world in (2, 4, 8):
        u, tr = _emulated_forward(w, model, src, rec, world)
        diffs[world] = (float(np.abs(u - f.u).max()), float(np.abs(tr - f.record.data).max()))
    _log("cfg5 192^3 so16 z slabs vs 1 GPU (emulated ranks)", max_abs_diff=diffs)
    for world, (du, dt_) in diffs.items():
        assert du == 0.0 and dt_ == 0.0, (world, du, dt_)


# BASELINE's FULL sizes against the unmodified reference (its OpenMP CPU path
# takes 30-60 s per case at 1-2 Gpts/s on 16 cores): opt-in, SFDB200_FULL_PARITY=1
# (the log of one run is kept under profiles/).  cfg3 and cfg5 at full size need
# a 153 GB fp64 history / 130 GB of host grids in the reference and stay at the
# protocol sizes above.
_full = pytest.mark.skipif(os.environ.get("SFDB200_FULL_PARITY") != "1" or not O.have_ref(),
                           reason="opt-in: SFDB200_FULL_PARITY=1 and the built reference")


@pytest.mark.skipif(not O.have_ref(), reason="needs the built reference (oracle/_ref)")
def test_protocol_cfg2_full_size():
    """BASELINE configs[1] exactly as benched (344^3 padded, 1000 steps, 65,536
    receivers) against the unmodified reference: ~40 s of its CPU path, so this
    one full-size case runs with the default suite."""
    _forward_case("cfg2 FULL 256^3+40 so8 1000 steps 256^2 carpet", configs.cfg2())


@pytest.mark.parametrize("so,tile", [(4, "4,2,4,4,1"), (16, "4,2,4,2,1")])
def test_protocol_grouped_order_wide_grid(monkeypatch, so, tile):
    """A wide, thin grid (24 x 704 x 704 + 40) has more (x, y) tiles than the
    GPU has resident CTA slots, so the grouped item order of the 512^3-and-up
    workloads is active at a size the checker finishes in seconds: three
    sources at mid depth, 2,000 receivers through the volume, three z chunks.
    Against the checker, and three identical runs bit-identical (an injection
    added by a CTA that does not own the cell races with the owner's store)."""
    monkeypatch.setenv("SFDB200_TILE", tile)
    monkeypatch.setenv("SFDB200_ZCHUNKS", "3")
    n, nbpml, h, nt = (24, 704, 704), 40, 10.0, 82
    rng = np.random.default_rng(so)
    v = 1500.0 + 2500.0 * rng.random(n)
    for ax in range(3):
        v = 0.5 * v + 0.25 * (np.roll(v, 1, ax) + np.roll(v, -1, ax))
    m = configs._round32(1.0 / v ** 2).ravel()
    dt = 0.8 * configs._crit(m.min(), 3, so, h)
    sp = np.array([(k - 1) * h for k in n])
    srcs = np.array([0.5, 0.31, 0.72]) * sp + rng.uniform(-40.0, 40.0, (3, 3))
    recs = rng.random((2000, 3)) * sp
    w = configs.Workload(f"wide-24x704x704-so{so}", 3, list(n), so, nt, dt, m,
                         configs._ricker(12.0, nt, dt, 3), srcs, recs, h, nbpml, 12.0)
    f, model, src, rec = _forward_case(f"grouped order: 24x704x704+40 so{so} 80 steps 3 src", w)
    tiles = -(-model.padded[2] // 32) * -(-(model.padded[1] - so) // 16)
    assert tiles > 5 * 148, tiles
    for _ in range(2):
        g = S.forward(model, src, w.wavelet, rec, w.nt, w.dt, False)
        assert np.array_equal(g.u, f.u) and np.array_equal(g.record.data, f.record.data)


@_full
@pytest.mark.parametrize("so", [2, 4, 6, 8, 10, 12, 14, 16])
def test_protocol_cfg4_full_size(so):
    _forward_case(f"cfg4 FULL 512^3+40 so{so} 200 steps", configs.cfg4(so))


@_full
def test_protocol_cfg3_full_size_operators():
    """cfg3 at FULL size (200^3 + 40, so 8, 800 steps, 40,000 receivers).  The
    reference runs its forward and adjoint here (rolling slots); its gradient
    would need the 153 GB fp64 history on the host, so the imaging condition at
    this size is checked through the device chain's own properties:
    checkpointed = full history, and <grad, dm> against a central difference of
    the objective (the reference's Taylor-test idea, verify.cpp)."""
    import dataclasses
    w = configs.cfg3()
    model_t, src, rec = _setup(w)
    _check_indices(w, model_t, src, rec)
    ft = S.forward(model_t, src, w.wavelet, rec, w.nt, w.dt, False)
    ut, obs, _ = _oracle_forward(w, model_t, src, rec)
    e_true = [O.rel_l2(a, b) for a, b in zip(_last_slots(ft.u, w.nt), _last_slots(ut, w.nt))]
    e_obs = O.rel_l2(ft.record.data, obs)
    del ft, ut
    wb = configs.Workload(w.name + "-bg", 3, w.interior, w.space_order, w.nt, w.dt,
                          w.extra["m_background"], w.wavelet, w.src_coords, w.rec_coords, w.h,
                          w.nbpml, w.f0)
    model, _, _ = _setup(wb)
    fb = S.forward(model, src, wb.wavelet, rec, wb.nt, wb.dt, False)
    ub, syn, _ = _oracle_forward(wb, model, src, rec)
    e_bg = [O.rel_l2(a, b) for a, b in zip(_last_slots(fb.u, w.nt), _last_slots(ub, w.nt))]
    e_syn = O.rel_l2(fb.record.data, syn)
    del fb, ub
    # adjoint of the reference's residual, both sides (rolling slots)
    resid = syn - obs
    a = S.adjoint(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), src, w.nt, w.dt)
    vo, so_, _ = O.ref_adjoint(wb.interior, wb.h, wb.nbpml, wb.space_order, wb.m_interior,
                               wb.rec_coords, resid, wb.src_coords, w.nt, w.dt)
    # backward loop t = nt-1 .. 2: the last three steps are t = 4, 3, 2
    e_adj = [O.rel_l2(np.asarray(a.v)[t % 3], vo[t % 3]) for t in (4, 3, 2)]
    e_srcs = O.rel_l2(a.src_samples.data, so_)
    del a, vo
    # the device chain: full history (77 GB in HBM) vs checkpoints, and the
    # directional derivative of the objective
    obs_rec = S.ShotRecord(w.nt, w.dt, rec.npoints, obs)
    chain = S.fwi_gradient(model, src, wb.wavelet, rec, obs_rec, w.nt, w.dt, checkpoint_interval=0)
    ck = S.fwi_gradient(model, src, wb.wavelet, rec, obs_rec, w.nt, w.dt, checkpoint_interval=28)
    e_ck = O.rel_l2(ck.grad, chain.grad)
    phi_ref = 0.5 * float(np.sum(resid * resid))
    e_phi = abs(chain.phi - phi_ref) / phi_ref
    i = np.indices(w.interior)
    bump = np.exp(-sum((i[d] - 0.5 * w.interior[d]) ** 2 for d in range(3)) / (2 * 20.0 ** 2))
    dm = np.zeros(model.cells())
    S.add_interior(model, (np.asarray(wb.m_interior).max() * 0.01 * bump).ravel(), 1.0, dm)
    gdot = float(np.dot(np.asarray(chain.grad).ravel(), dm))
    phis = []
    for sgn in (1.0, -1.0):
        mp = dataclasses.replace(model, m=np.asarray(model.m) + sgn * dm)
        rp = S.forward(mp, src, wb.wavelet, rec, w.nt, w.dt, False).record
        phis.append(S.objective(rp, obs_rec))
    fd = (phis[0] - phis[1]) / 2.0
    _log("cfg3 FULL 200^3+40 so8 800 steps: forward (true, background) + adjoint vs reference; "
         "device chain properties", padded=list(map(int, model.padded)), steps=w.nt - 2,
         nrec=rec.npoints, true_slot_rel_l2=e_true, observed_record_rel_l2=e_obs,
         background_slot_rel_l2=e_bg, synthetic_record_rel_l2=e_syn, adjoint_slot_rel_l2=e_adj,
         adjoint_source_samples_rel_l2=e_srcs, chain_phi_rel=e_phi,
         checkpointed_vs_full_rel_l2=e_ck, grad_dot_dm=gdot, central_difference=fd,
         directional_rel_err=abs(fd - gdot) / abs(fd))
    assert max(e_true + e_bg + e_adj) <= TOL and max(e_obs, e_syn, e_srcs) <= TOL
    # Phi subtracts two records that differ by ~1 % (the anomaly's reflections),
    # so their 5e-7 fp32 error reaches Phi amplified ~100x twice over
    assert e_phi <= 5e-4
    # the two storage schemes run the same kernels on the same rows, and the
    # 40,000 receivers' colliding corners (adjacent receivers share cells) are
    # summed per cell in a fixed order: the gradients are bit-identical
    assert e_ck == 0.0
    assert abs(fd - gdot) <= 0.03 * abs(fd)


@_full
def test_protocol_cfg5_full_size_properties():
    """cfg5 at FULL size (1024^3 + 40 -> 1120^3 padded, so 16, 500 steps, 4
    sources, 512^2 carpet) on one B200.  The reference needs > 130 GB of host
    grids here, so the full size is checked through size-independent
    properties of the linear operator, observed on the receiver carpet plus
    8,192 receivers scattered through the whole volume: identical runs are
    bit-identical (no race in the grouped item order / fused sparse work), and
    the 4-source run equals the sum of the four single-source runs (every
    injection lands exactly once, in the cell that stores it; within the 500
    steps the four wavefronts, 5 km apart, do not yet overlap, so the sum is
    exact rather than equal to rounding)."""
    w = configs.cfg5()
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    rng = np.random.default_rng(5)
    span = (w.interior[0] - 1) * w.h
    vol = rng.random((8192, 3)) * span
    rec = S.locate_points(model, np.concatenate([np.asarray(w.rec_coords), vol]))
    src = S.locate_points(model, w.src_coords)
    nsrc = src.npoints
    wav = np.asarray(w.wavelet, dtype=np.float64).reshape(w.nt, nsrc) * np.array([1.0, -0.7, 1.3, 0.5])
    p = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, nsrc, rec.npoints,
               False, 0)
    try:
        def run(tr):
            out = np.zeros((w.nt, rec.npoints))
            argv = [None, model.m, model.damp, src.idx, src.w, np.ascontiguousarray(tr), rec.idx,
                    rec.w, out]
            p.upload(argv)
            p.execute()
            p.download(argv)
            return out
        all_a = run(wav)
        all_b = run(wav)
        same = bool(np.array_equal(all_a, all_b))
        total = np.zeros_like(all_a)
        for s in range(nsrc):
            one = np.zeros_like(wav)
            one[:, s] = wav[:, s]
            total += run(one)
        e_lin = O.rel_l2(total, all_a)
        e_lin_vol = O.rel_l2(total[:, -8192:], all_a[:, -8192:])
        info = p.info()
    finally:
        p.close()
    _log("cfg5 FULL 1024^3+40 so16 500 steps 4 src: determinism + linearity", padded=list(map(int, model.padded)),
         steps=w.nt - 2, nrec=rec.npoints, identical_runs_bitwise=same,
         superposition_rel_l2=e_lin, superposition_rel_l2_volume_receivers=e_lin_vol,
         record_norm=float(np.linalg.norm(all_a)), sweep=info.get("instantiation"),
         zchunks=info.get("zchunks"))
    assert same
    assert np.all(np.isfinite(all_a)) and np.linalg.norm(all_a[:, -8192:]) > 0
    assert e_lin <= TOL and e_lin_vol <= TOL


@_full
def test_protocol_grouped_order_slab_ranks(monkeypatch):
    """The grouped item order (more tiles than resident slots) together with the
    fused P2P boundary items: a cfg5-shaped slab problem (64 x 768 x 768 + 40,
    so 16, 4 sources at mid depth, 160 steps, receivers through the volume)
    against the reference on one GPU, then z-slab-decomposed over 2 and 4
    emulated ranks, bitwise equal to the one-GPU run."""
    monkeypatch.setenv("SFDB200_TILE", "4,2,4,2,1")
    n, so, nbpml, h, nt = (64, 768, 768), 16, 40, 10.0, 162
    v = configs.smooth_random_velocity(n, 1, 16.0)
    m = configs._round32(1.0 / v ** 2).ravel()
    dt = configs._crit(m.min(), 3, so, h)
    sp = [(k - 1) * h for k in n]
    srcs = np.array([[0.5 * sp[0] + 3.0, a, b] for a in (0.25 * sp[1] + 1.0, 0.75 * sp[1] - 2.0)
                     for b in (0.25 * sp[2] + 4.0, 0.75 * sp[2] - 3.0)])
    rng = np.random.default_rng(11)
    recs = np.concatenate([rng.random((4096, 3)) * np.array(sp),
                           srcs + rng.uniform(-150.0, 150.0, (4, 3)).clip(-0.4 * sp[0], 0.4 * sp[0])])
    w = configs.Workload("cfg5-slab-64x768x768", 3, list(n), so, nt, dt, m,
                         configs._ricker(10.0, nt, dt, 4), srcs, recs, h, nbpml, 10.0)
    f, model, src, rec = _forward_case("grouped order: 64x768x768+40 so16 160 steps 4 src", w)
    tiles = -(-model.padded[2] // 32) * -(-(model.padded[1] - so) // 16)
    assert tiles > 3 * 148, tiles  # more tiles than resident slots: the grouped order is on
    assert np.abs(f.record.data).max() > 0
    diffs = {}
    for world in (2, 4):
        u, tr = _emulated_forward(w, model, src, rec, world)
        diffs[world] = (float(np.abs(u - f.u).max()), float(np.abs(tr - f.record.data).max()))
    _log("grouped order + boundary items: 64x768x768 so16 z slabs vs 1 GPU (emulated ranks)",
         max_abs_diff=diffs, tiles=int(tiles))
    for world, (du, dt_) in diffs.items():
        assert du == 0.0 and dt_ == 0.0, (world, du, dt_)


@_full
def test_protocol_adjoint_and_gradient_chain_512():
    """The adjoint at 512^3 + 40 (so 8, 100 steps: grouped order, thousands of
    fused injection corners from a receiver carpet, fused sampling at the
    sources) against the reference, and the device gradient chain at the same
    size (60 steps, 54 GB history in HBM): checkpointed = full history, and the
    directional derivative of the objective."""
    import dataclasses
    w = configs.cfg4(8, nt=102)
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    sp = (w.interior[0] - 1) * w.h
    rng = np.random.default_rng(7)
    rec_c = np.concatenate([configs._carpet(64, sp, 20.0), rng.random((2048, 3)) * sp])
    src_c = 0.3 * sp + rng.random((3, 3)) * 0.4 * sp
    rec = S.locate_points(model, rec_c)
    src = S.locate_points(model, src_c)
    white = rng.standard_normal((w.nt, rec.npoints))
    pulse = S.ricker(15.0, 1.2 / 15.0, w.nt, w.dt)
    sm = np.stack([np.convolve(white[:, r], pulse)[:w.nt] for r in range(rec.npoints)], 1)
    resid = O._f64((sm / np.abs(sm).max()).astype(np.float32))
    a = S.adjoint(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), src, w.nt, w.dt)
    vo, so_, t_ref = O.ref_adjoint(w.interior, w.h, w.nbpml, w.space_order, w.m_interior, rec_c,
                                   resid, src_c, w.nt, w.dt)
    e_adj = [O.rel_l2(np.asarray(a.v)[t % 3], vo[t % 3]) for t in (4, 3, 2)]
    e_src = O.rel_l2(a.src_samples.data, so_)
    del a, vo
    # gradient chain, 60 steps
    nt = 62
    wav = np.ascontiguousarray(np.asarray(w.wavelet)[:nt].reshape(nt, -1)[:, :1])
    one = S.locate_points(model, np.array([[0.5 * sp, 0.5 * sp, 0.5 * sp]]))
    near = S.locate_points(model, 0.5 * sp + rng.uniform(-120.0, 120.0, (512, 3)))
    i = np.indices(w.interior)
    bump = np.exp(-sum((i[d] - 0.5 * w.interior[d] - 4.0) ** 2 for d in range(3)) / (2 * 6.0 ** 2))
    mt = np.asarray(w.m_interior).reshape(w.interior) * (1.0 + 0.05 * bump)
    true = S.make_model(w.interior, w.h, w.nbpml, w.space_order, configs._round32(mt).ravel())
    obs = S.forward(true, one, wav, near, nt, w.dt, False).record
    chain = S.fwi_gradient(model, one, wav, near, obs, nt, w.dt, checkpoint_interval=0)
    ck = S.fwi_gradient(model, one, wav, near, obs, nt, w.dt, checkpoint_interval=10)
    e_ck = O.rel_l2(ck.grad, chain.grad)
    dm = np.zeros(model.cells())
    S.add_interior(model, (np.asarray(w.m_interior).max() * 0.01 * bump).ravel(), 1.0, dm)
    gdot = float(np.dot(np.asarray(chain.grad).ravel(), dm))
    phis = []
    for sgn in (1.0, -1.0):
        mp = dataclasses.replace(model, m=np.asarray(model.m) + sgn * dm)
        phis.append(S.objective(S.forward(mp, one, wav, near, nt, w.dt, False).record, obs))
    fd = (phis[0] - phis[1]) / 2.0
    _log("adjoint 512^3+40 so8 100 steps vs reference; gradient chain 60 steps",
         padded=list(map(int, model.padded)), nrec=rec.npoints, adjoint_slot_rel_l2=e_adj,
         adjoint_source_samples_rel_l2=e_src, checker_s=t_ref, checkpointed_vs_full_rel_l2=e_ck,
         grad_dot_dm=gdot, central_difference=fd, directional_rel_err=abs(fd - gdot) / abs(fd),
         phi=chain.phi)
    assert max(e_adj) <= TOL and e_src <= TOL
    assert e_ck == 0.0
    assert abs(fd - gdot) <= 0.03 * abs(fd)
