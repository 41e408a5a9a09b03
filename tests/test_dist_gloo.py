"""Multi-rank (world_size 2 and 3) CPU test of the z-slab decomposition's host
logic with torch.distributed/gloo: the product's slab split (sfdb200_slab)
and ownership rules (sfdb200_slab_owns) drive ranks that step their slabs
with the fp64 oracle, inject only owned corners before the ghost exchange,
exchange the so/2 boundary planes with their z neighbours (the same plane
ranges libsfdb200's NCCL exchange sends), and sample owned receivers after it.
Assembled, the result must equal the single-domain oracle bit for bit."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as O
from paper_1608_08658_b200 import _lib as L
from paper_1608_08658_b200 import configs, seismic as S


def _problem():
    w = configs.cfg2(n=20, nt=70, nbpml=4, nrec_side=5)
    rng = np.random.default_rng(4)
    span = (w.interior[0] - 1) * w.h
    # receivers and sources all over z, incl. exactly on slab boundaries
    rec = rng.uniform(0.0, span, size=(40, 3))
    src = rng.uniform(0.0, span, size=(3, 3))
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    pz = model.padded[0]
    R = w.space_order // 2
    for world in (2, 3):
        for r in range(1, world):
            zb, _ = L.slab(pz, w.space_order, world, r)
            # base plane right before / at the boundary (model frame: z = (idx - pad) h)
            rec = np.vstack([rec, [[(zb - 1 - model.pad()) * w.h + 3.0, 55.0, 61.0],
                                   [(zb - model.pad()) * w.h, 40.0, 70.0]]])
            src = np.vstack([src, [[(zb - 1 - model.pad()) * w.h + 5.0, 80.0, 90.0]]])
    s = S.locate_points(model, src)
    r = S.locate_points(model, rec)
    wav = O._f64(np.repeat(w.wavelet[:, :1], len(src), axis=1))
    return w, model, s, r, wav, R


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _rank_main(rank, world, port, outdir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    import torch
    w, model, src, rec, wav, R = _problem()
    P = model.padded
    zb, ze = L.slab(P[0], w.space_order, world, rank)
    zoff, Pl = zb - R, ze - zb + 2 * R
    lp = [Pl, P[1], P[2]]
    m = model.m.reshape(P)[zoff:zoff + Pl].copy()
    damp = model.damp.reshape(P)[zoff:zoff + Pl].copy()
    shift = np.array([zoff, 0, 0])
    cm, _ = L.slab_owns(P[0], w.space_order, world, rank, src.idx)
    _, pm = L.slab_owns(P[0], w.space_order, world, rank, rec.idx)
    sidx = np.where(cm.any(axis=1)[:, None], src.idx - shift, 0)
    ridx = np.where(pm[:, None], rec.idx - shift, 0)
    u = np.zeros((3, *lp))
    recd = np.zeros((w.nt, rec.npoints))
    for t in range(2, w.nt):
        O.forward_steps(lp, w.space_order, w.h, w.dt, w.nt, u, m, damp, sidx, src.w, wav, cm,
                        t, t + 1)
        slot = u[t % 3]
        reqs, recv = [], []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(slot[R:2 * R].copy()), rank - 1))
            buf = torch.empty(slot[0:R].shape, dtype=torch.float64)
            reqs.append(dist.irecv(buf, rank - 1))
            recv.append((buf, slice(0, R)))
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(slot[Pl - 2 * R:Pl - R].copy()), rank + 1))
            buf = torch.empty(slot[Pl - R:Pl].shape, dtype=torch.float64)
            reqs.append(dist.irecv(buf, rank + 1))
            recv.append((buf, slice(Pl - R, Pl)))
        for q in reqs:
            q.wait()
        for buf, sl in recv:
            slot[sl] = buf.numpy()
        O.sample_row(lp, w.space_order, w.h, w.dt, w.nt, u, t, ridx, rec.w, recd, pm)
    # Assemble: every plane / receiver has exactly one owner -> sums are copies.
    glob = np.zeros((3, *P))
    lo = 0 if rank == 0 else R
    hi = Pl if rank == world - 1 else Pl - R
    glob[:, zoff + lo:zoff + hi] = u[:, lo:hi]
    gt = torch.from_numpy(glob)
    rt = torch.from_numpy(recd)
    dist.all_reduce(gt)
    dist.all_reduce(rt)
    owned = torch.tensor([int(pm.sum()), int(cm.sum())])
    dist.all_reduce(owned)
    if rank == 0:
        np.savez(os.path.join(outdir, f"dist{world}.npz"), u=gt.numpy(), rec=rt.numpy(),
                 owned=owned.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_matches_single_domain(world):
    w, model, src, rec, wav, R = _problem()
    u, r = O.forward(model.padded, w.space_order, w.h, w.dt, w.nt, model.m, model.damp,
                     src.idx, src.w, wav, rec.idx, rec.w)
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_rank_main, args=(world, _free_port(), d), nprocs=world,
                           start_method="spawn")
        res = np.load(os.path.join(d, f"dist{world}.npz"))
    assert list(res["owned"]) == [rec.npoints, 8 * src.npoints]  # one owner each
    assert np.array_equal(res["u"], u)
    assert np.array_equal(res["rec"], r)


def test_slab_split_covers_the_updated_range():
    for pz, so, world in [(344, 8, 8), (1120, 16, 8), (101, 4, 3), (30, 2, 7)]:
        R = so // 2
        ends = []
        for r in range(world):
            zb, ze = L.slab(pz, so, world, r)
            assert ze > zb
            ends.append((zb, ze))
        assert ends[0][0] == R and ends[-1][1] == pz - R
        assert all(ends[i][1] == ends[i + 1][0] for i in range(world - 1))
        sizes = [b - a for a, b in ends]
        assert max(sizes) - min(sizes) <= 1


def _slab_rank(rank, world, port, outdir):
    """bench.py's N > 1 input generation on one gloo rank: its rows, the
    rescale range all-reduced over the ranks, its planes of the model."""
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    import types
    import torch
    import bench
    n = 24
    w, model = bench.slab_problem(L, S, types.SimpleNamespace(time_steps=10), world, rank, n=n)
    P = model.padded[0]
    zb, ze = L.slab(P, 16, world, rank)
    lo = 0 if rank == 0 else zb
    hi = P if rank == world - 1 else ze
    mg = np.zeros((P, P, P))
    dg = np.zeros((P, P, P))
    mg[lo:hi] = model.m.reshape(P, P, P)[lo:hi]
    dg[lo:hi] = model.damp.reshape(P, P, P)[lo:hi]
    mt, dt_ = torch.from_numpy(mg), torch.from_numpy(dg)
    dist.all_reduce(mt)
    dist.all_reduce(dt_)
    if rank == 0:
        np.savez(os.path.join(outdir, "slab.npz"), m=mt.numpy(), damp=dt_.numpy(), dt=w.dt)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bench_slab_inputs_over_gloo_ranks(world):
    """The per-rank cfg5 inputs of bench.py --gpus N, generated on gloo ranks
    (real all-reduce of the rescale range), assemble to the whole model bit
    for bit (configs.cfg5 + make_model, the reference's make_model /
    build_damping)."""
    full = configs.cfg5(n=24, nt=12, nrec_side=4)
    model = S.make_model(full.interior, full.h, full.nbpml, 16, full.m_interior)
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_slab_rank, args=(world, _free_port(), d), nprocs=world,
                           start_method="spawn")
        res = np.load(os.path.join(d, "slab.npz"))
    assert float(res["dt"]) == full.dt
    assert np.array_equal(res["m"].ravel(), model.m)
    assert np.array_equal(res["damp"].ravel(), model.damp)
