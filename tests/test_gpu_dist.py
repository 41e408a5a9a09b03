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


def _run_group(kind, w, model, src, rec, wav, world, resid=None):
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
        p.upload(argv)
        plans.append(p)
        outs.append((argv, field, tr))
    L.execute_group(plans)
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


@pytest.mark.parametrize("world", [2, 3])
def test_emulated_ranks_forward_matches_single_gpu(world):
    w, model, src, rec, wav = _problem()
    ref = S.forward(model, src, wav, rec, w.nt, w.dt, False)
    u, tr = _run_group(L.FORWARD, w, model, src, rec, wav, world)
    assert O.rel_l2(u, ref.u) <= 1e-6
    assert O.rel_l2(tr, ref.record.data) <= 1e-6
    uo, ro = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                       src.idx, src.w, wav, rec.idx, rec.w)
    assert O.rel_l2(u, uo) <= 1e-5 and O.rel_l2(tr, ro) <= 1e-5


def test_emulated_ranks_adjoint_so16():
    w, model, src, rec, wav = _problem(so=16)
    rng = np.random.default_rng(2)
    resid = O._f64(rng.standard_normal((w.nt, rec.npoints)).astype(np.float32))
    ref = S.adjoint(model, rec, S.ShotRecord(w.nt, w.dt, rec.npoints, resid), src, w.nt, w.dt)
    v, tr = _run_group(L.ADJOINT, w, model, src, rec, wav, 3, resid)
    assert O.rel_l2(v, ref.v) <= 1e-6
    assert O.rel_l2(tr, ref.src_samples.data) <= 1e-6


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
        comm.close()
        assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    finally:
        dist.destroy_process_group()
