"""GPU test of the z-slab decomposition on ONE GPU: `world` emulated ranks
(loopback communicators) run the real kernels, sparse tables and phase
order in lockstep through sfdb200_execute_group, the ghost exchange done as
device copies of exactly the planes the NCCL path sends.  Assembled, the
result must match the single-GPU run (and the oracle)."""
import numpy as np
import pytest

import oracle_lib as O
from paper_1608_08658_b200 import _lib as L
from paper_1608_08658_b200 import configs, seismic as S

pytestmark = pytest.mark.gpu


def _problem(so=8):
    w = configs.cfg2(n=40, nt=122, nbpml=8, nrec_side=6)
    if so != 8:
        w = configs.cfg4(so, n=40, nt=122, nbpml=8)
    rng = np.random.default_rng(8)
    span = (w.interior[0] - 1) * w.h
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    rec_c = np.vstack([rng.uniform(0.0, span, size=(300, 3)), w.rec_coords])
    src_c = rng.uniform(0.0, span, size=(4, 3))
    for world in (2, 3):  # points right at the slab boundaries
        for r in range(1, world):
            zb, _ = L.slab(model.padded[0], w.space_order, world, r)
            zm = (zb - model.pad()) * w.h
            rec_c = np.vstack([rec_c, [[zm - 7.0, 55.0, 61.0], [zm, 40.0, 70.0]]])
            src_c = np.vstack([src_c, [[zm - 5.0, 80.0, 90.0]]])
    src = S.locate_points(model, src_c)
    rec = S.locate_points(model, rec_c)
    wav = O._f64(np.repeat(w.wavelet[:, :1], len(src_c), axis=1))
    return w, model, src, rec, wav


def _collide(pts):
    """Whether two injection corners of the set share a cell (their fp32 atomics
    then sum in a decomposition-dependent order)."""
    nd = pts.idx.shape[1]
    offs = [np.array([(c >> (nd - 1 - k)) & 1 for k in range(nd)]) for c in range(1 << nd)]
    cells = [tuple(i + o) for i in pts.idx for o in offs]
    return len(set(cells)) != len(cells)


def _same(a, b, tol, collide):
    """Bitwise equal to the one-GPU run when no injection corners collide
    (SURVEY §8(e)), else within tol."""
    return np.array_equal(a, b) if not collide else O.rel_l2(a, b) <= tol


@pytest.fixture
def one_tiling(monkeypatch):
    """The one-GPU plan and the slab plans use one compiled sweep variant, so
    the decomposition is the only difference between the runs."""
    def pin(so):
        monkeypatch.setenv("SFDB200_TILE", "4,2,4,1,1" if so <= 8 else "4,2,4,4,1")
    return pin


def _run_group(kind, w, model, src, rec, wav, world, resid=None, p2p=False, abort=None):
    import torch
    stream = torch.cuda.Stream()
    comms = [L.Comm.loopback(world, r, 0) for r in range(world)]
    plans, outs = [], []
    for r in range(world):
        p = L.Plan(kind, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                   rec.npoints, False, 0, comm=comms[r])
        p.set_stream(stream.cuda_stream)
        field = np.zeros((3, *model.padded))
        if kind == L.FORWARD:
            tr = np.zeros((w.nt, rec.npoints))
            argv = [field, model.m, model.damp, src.idx, src.w, wav, rec.idx, rec.w, tr]
        else:
            tr = np.zeros((w.nt, src.npoints))
            argv = [field, model.m, model.damp, src.idx, src.w, tr, rec.idx, rec.w, resid]
        plans.append(p)
        outs.append((argv, field, tr))
    if p2p:  # fused P2P exchange: boundary sweeps store into the neighbours' rows
        L.peer_group(plans)
    for p, (argv, _, _) in zip(plans, outs):
        p.upload(argv)
    if abort is not None:
        plans[abort].abort()
    L.execute_group(plans)
    if abort is not None:  # every rank of the chain reports the broken exchange
        errors = []
        for p, (argv, _, _) in zip(plans, outs):
            try:
                p.download(argv)
                errors.append(None)
            except L.SfdError as e:
                errors.append(e.code)
        for p in plans:
            p.close()
        for c in comms:
            c.close()
        return errors
    field = np.zeros((3, *model.padded))
    trace = 0
    for p, (argv, f, tr) in zip(plans, outs):
        p.download(argv)
        field += f    # each plane is written by exactly one rank (others stay 0)
        trace = trace + tr
    for p in plans:
        p.close()
    for c in comms:
        c.close()
    return field, trace


@pytest.mark.parametrize("world,p2p", [(2, False), (3, False), (2, True), (3, True)])
def test_emulated_ranks_forward_matches_single_gpu(world, p2p, one_tiling):
    one_tiling(8)
    w, model, src, rec, wav = _problem()
    ref = S.forward(model, src, wav, rec, w.nt, w.dt, False)
    u, tr = _run_group(L.FORWARD, w, model, src, rec, wav, world, p2p=p2p)
    c = _collide(src)
    assert _same(u, ref.u, 1e-6, c) and _same(tr, ref.record.data, 1e-6, c)
    uo, ro = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                       src.idx, src.w, wav, rec.idx, rec.w)
    assert O.rel_l2(u, uo) <= 1e-5 and O.rel_l2(tr, ro) <= 1e-5


@pytest.mark.parametrize("p2p", [False, True])
def test_emulated_ranks_adjoint_so16(p2p, one_tiling):
    one_tiling(16)
    w, model, src, rec, wav = _problem(so=16)
    rng = np.random.default_rng(2)
    resid = O._f64(rng.standard_normal((w.nt, rec.npoints)).astype(np.float32))
    ref = S.adjoint(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), src, w.nt, w.dt)
    v, tr = _run_group(L.ADJOINT, w, model, src, rec, wav, 3, resid, p2p=p2p)
    c = _collide(rec)  # the adjoint injects at the receivers
    assert _same(v, ref.v, 1e-6, c) and _same(tr, ref.src_samples.data, 1e-6, c)


def test_nccl_communicator_single_rank():
    """The real NCCL path as far as one GPU allows: torch.distributed (nccl)
    loads libnccl, libsfdb200 resolves it at run time, builds a 1-rank
    communicator from a unique id and runs a plan over it (no neighbour, so no
    exchange); the result equals the plan without a communicator."""
    import socket

    import torch
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        uid = L.Comm.unique_id()
        assert len(uid) == 128 and any(uid)
        comm = L.Comm(uid, 1, 0, 0)
        w, model, src, rec, wav = _problem()
        outs = []
        for c in (comm, None):
            p = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                       rec.npoints, False, 0, comm=c)
            u = np.zeros((3, *model.padded))
            tr = np.zeros((w.nt, rec.npoints))
            p.run([u, model.m, model.damp, src.idx, src.w, wav, rec.idx, rec.w, tr])
            p.close()
            outs.append((u, tr))
        assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
        # bench.py's pre-timing check of the exchange (N > 1) runs its whole
        # path here: the small problem over the communicator, the sum over
        # ranks, the one-GPU comparison on rank 0.
        import bench
        from paper_1608_08658_b200 import seismic as S
        ok, err = bench.check_exchange(L, S, torch, dist, comm, 0, 1, 0, False)
        assert ok and err <= 1e-6, err
        comm.close()
    finally:
        dist.destroy_process_group()


def test_p2p_injection_in_sent_planes(one_tiling):
    """Sources whose corners lie in the planes the boundary sweeps send: the
    fused P2P exchange must mirror the injected values into the neighbour's
    ghost copy (launch_mirror); equal to the single-GPU run."""
    one_tiling(8)
    w, model, src, rec, wav = _problem()
    R = w.space_order // 2
    pts = []
    span = (model.interior[0] - 1) * w.h
    for world in (2, 3):
        for r in range(1, world):  # the boundary between ranks r-1 and r
            zb, _ = L.slab(model.padded[0], w.space_order, world, r)
            # rank r's first R planes (sent down) and rank r-1's last R (sent up)
            for z in (zb, zb + R - 1, zb - R, zb - 1):
                zc = (z - model.pad()) * w.h + 2.5
                if 0.0 <= zc <= span:
                    pts.append([zc, 100.0, 120.0])
    src = S.locate_points(model, np.array(pts))
    wav = O._f64(np.repeat(w.wavelet[:, :1], len(pts), axis=1))
    ref = S.forward(model, src, wav, rec, w.nt, w.dt, False)
    for world in (2, 3):
        u, tr = _run_group(L.FORWARD, w, model, src, rec, wav, world, p2p=True)
        c = _collide(src)
        assert _same(u, ref.u, 1e-6, c) and _same(tr, ref.record.data, 1e-6, c), world


def test_ipc_export_blob():
    """A dist plan exports its IPC blob (field + step counters); importing a
    blob that is not the neighbour's is refused (the plan keeps NCCL)."""
    w, model, src, rec, wav = _problem()
    comms = [L.Comm.loopback(2, r, 0) for r in range(2)]
    plans = [L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                    rec.npoints, False, 0, comm=c) for c in comms]
    try:
        blobs = [p.ipc_export() for p in plans]
        assert all(len(b) == L.IPC_BYTES and any(b) for b in blobs)
        with pytest.raises(L.InvalidArgument):
            plans[0].ipc_import(None, blobs[0])  # its own blob, not rank 1's
    finally:
        for p in plans:
            p.close()
        for c in comms:
            c.close()


def test_p2p_step_counters():
    """cuStreamWriteValue32 and the polling wait kernel as the P2P exchange uses
    them, on one device; a neighbour that stalls (alive, never publishing) makes
    the waiting rank time out AND poisons the staller, whose next wait returns at
    once; p2p_check then fails on both sides."""
    L.check(L.lib().sfdb200_p2p_selftest(0))


@pytest.mark.parametrize("p2p", [False, True])
def test_emulated_ranks_gradient(p2p):
    """The fused adjoint + imaging-condition kernel over z slabs (boundary
    sweeps exchanging v, the gradient local to each rank): assembled gradient
    equals the single-GPU one."""
    import torch
    w, model, src, rec, wav = _problem()
    u, r = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                     src.idx, src.w, wav, rec.idx, rec.w, save=True)
    resid = O._f64(np.random.default_rng(4).standard_normal(r.shape).astype(np.float32))
    ref = S.gradient(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), u, w.nt, w.dt)
    world = 3
    stream = torch.cuda.Stream()
    comms = [L.Comm.loopback(world, k, 0) for k in range(world)]
    plans, outs = [], []
    for k in range(world):
        p = L.Plan(L.GRADIENT, 3, model.padded, w.space_order, w.nt, w.dt, w.h, 0,
                   rec.npoints, False, 0, comm=comms[k])
        p.set_stream(stream.cuda_stream)
        grad = np.zeros(model.padded)
        argv = [np.zeros((3, *model.padded)), u, model.m, model.damp, grad, rec.idx, rec.w, resid]
        plans.append(p)
        outs.append((argv, grad))
    if p2p:
        L.peer_group(plans)
    for p, (argv, _) in zip(plans, outs):
        p.upload(argv)
    L.execute_group(plans)
    total = np.zeros(model.padded)
    for p, (argv, grad) in zip(plans, outs):
        p.download(argv)
        total += grad
    for p in plans:
        p.close()
    for c in comms:
        c.close()
    # colliding receiver corners are summed with fp32 atomics in an order that
    # depends on the decomposition; the backward time sum amplifies that to a
    # few 1e-6 (the forward / adjoint tests stay below 1e-6)
    assert O.rel_l2(total, ref.grad) <= 5e-6
    go, _ = O.gradient(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp, u,
                       rec.idx, rec.w, resid)
    assert O.rel_l2(total, go) <= 1e-5


def test_p2p_fused_launch_with_persistent_ctas():
    """The fused P2P launch (boundary tiles first, then interior items) walked by
    a few persistent CTAs, each running boundary and interior items in turn."""
    import os
    os.environ["SFDB200_CTAS"] = "5"
    try:
        w, model, src, rec, wav = _problem()
        ref = S.forward(model, src, wav, rec, w.nt, w.dt, False)
        u, tr = _run_group(L.FORWARD, w, model, src, rec, wav, 3, p2p=True)
        assert O.rel_l2(u, ref.u) <= 1e-6 and O.rel_l2(tr, ref.record.data) <= 1e-6
    finally:
        os.environ.pop("SFDB200_CTAS", None)


@pytest.mark.parametrize("world,rank", [(2, 0), (3, 1), (3, 2)])
def test_p2p_abort_fails_every_rank(world, rank):
    """sfdb200_plan_abort on one rank of the fused P2P exchange: it and its
    neighbours skip their peer stores, and every rank adjacent to the abort
    reports SFDB200_ECUDA at download instead of returning stale ghost planes
    as results."""
    w, model, src, rec, wav = _problem()
    errors = _run_group(L.FORWARD, w, model, src, rec, wav, world, p2p=True, abort=rank)
    for r, e in enumerate(errors):
        if abs(r - rank) <= 1:
            assert e == L.ECUDA, (r, errors)


@pytest.mark.parametrize("world", [2, 3])
def test_bench_slab_inputs_through_emulated_ranks(world, one_tiling):
    """bench.py's N > 1 inputs on the device: each rank's slab problem
    (bench.slab_problem: only its rows generated, global-shaped model arrays
    written only in its planes) uploaded into its loopback plan, the ranks run
    in lockstep with the fused P2P stores, assembled -- equal to one GPU on the
    full cfg5-style model (a 40^3 interior here), bitwise (the four sources'
    corners do not collide)."""
    import torch
    import types
    import bench
    from scipy.ndimage import gaussian_filter1d
    one_tiling(16)
    n = 40
    raw = (1500.0 + 3000.0 * np.random.default_rng(1).random(n ** 3)).reshape(n, n, n)
    for ax in range(3):
        raw = gaussian_filter1d(raw, 16.0, axis=ax, mode="nearest", truncate=4.0)
    lohi = (float(raw.min()), float(raw.max()))
    args = types.SimpleNamespace(time_steps=60)
    full = configs.cfg5(n=n, nt=62, nrec_side=8)
    fm = S.make_model(full.interior, full.h, full.nbpml, 16, full.m_interior)
    src, rec = S.locate_points(fm, full.src_coords), S.locate_points(fm, full.rec_coords)
    wav = np.ascontiguousarray(full.wavelet.reshape(full.nt, -1))
    ref = S.forward(fm, src, wav, rec, full.nt, full.dt, False)
    stream = torch.cuda.Stream()
    comms = [L.Comm.loopback(world, r, 0) for r in range(world)]
    plans, outs = [], []
    for r in range(world):
        w, model = bench.slab_problem(L, S, args, world, r, n=n, minmax=lambda a, b: lohi)
        p = L.Plan(L.FORWARD, 3, model.padded, 16, w.nt, w.dt, w.h, src.npoints, rec.npoints,
                   False, 0, comm=comms[r])
        p.set_stream(stream.cuda_stream)
        u, tr = np.zeros((3, *model.padded)), np.zeros((w.nt, rec.npoints))
        argv = [u, model.m, model.damp, src.idx, src.w, np.ascontiguousarray(w.wavelet), rec.idx,
                rec.w, tr]
        plans.append(p)
        outs.append((argv, u, tr))
    L.peer_group(plans)
    for p, (argv, _, _) in zip(plans, outs):
        p.upload(argv)
    L.execute_group(plans)
    u_sum, tr_sum = 0, 0
    for p, (argv, u, tr) in zip(plans, outs):
        p.download(argv)
        u_sum = u_sum + u
        tr_sum = tr_sum + tr
    for p in plans:
        p.close()
    for c in comms:
        c.close()
    assert np.array_equal(u_sum, ref.u) and np.array_equal(tr_sum, ref.record.data)
