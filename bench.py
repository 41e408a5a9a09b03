#!/usr/bin/env python
"""Benchmark of the damped acoustic stencil hot path (BASELINE.json metric:
"Gpts/s (grid-point updates/sec) 3D acoustic so-8; % of HBM roofline; 1/2/4/8 GPU").

One bench step = one full operator run (all nt-2 time steps) over one
synthetic problem.  At N=1 the workload is BASELINE configs[1] (cfg2: 3-D
forward, 256^3 + 40-point damping layer, so 8, 1000 steps, 65,536 receivers).
At N>1 it is BASELINE configs[4] (cfg5: 1024^3 + 40-point layer, so 16, 500
steps, 4 sources, 512^2 receivers) strong-scaled over z slabs, the north
star's parallel-efficiency configuration; each rank generates and uploads
only its slab.  `python bench.py --gpus N` launches the N ranks itself
(torch.distributed.run) when it is not already running under one.

  value    Gpts/s with inputs resident in HBM (plan.execute() only), device-timed
           with CUDA events on the plan's stream, max over ranks
  e2e      the same metric through the C ABI (sfdb200_run) with PAGEABLE host
           fp64 buffers -- the reference hands its kernel std::vectors
           (seismic.cpp:354-361) -- H2D + fp64->fp32, the run, fp32->fp64 + D2H;
           e2e.pinned: the same with pinned buffers (N=1)
  roofline dominant kernel (the 3-D sweep): algorithmic bytes per launch /
           mean launch time; frac at the bytes the kernel needs (16 B/pt with
           separable damping), frac_alg at SURVEY 8(d)'s 20 B/pt (32 gradient)
  cpu_baseline  the unmodified reference (oracle/_ref) on this host's cores,
           full grid, truncated step count

--impl reference runs the reference's own CPU implementation of the path
(oracle/_ref, else the oracle C port) and prints the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# The reference's JIT'd kernels use OpenMP: all host threads, bound close
# (set just before the reference first runs, bind_reference_threads(): an
# OpenMP runtime started earlier with binding would pin this process's main
# thread, and the helper threads it spawns, to one core).
os.environ.setdefault("STENCILFD_THREADS", str(os.cpu_count() or 1))
os.environ.setdefault("STENCILFD_CACHE_DIR", "/tmp/stencilfd-cache")


def bind_reference_threads():
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")

import numpy as np  # noqa: E402

BYTES_PER_POINT = {"forward": 20, "adjoint": 20, "gradient": 32}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None,
                    help="cfg1 | cfg2 | cfg3 (FWI gradient) | cfg4-so{2,4,8,12,16} | cfg5 "
                         "(default: cfg2 at N=1, cfg5 at N>1)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N>1 with cfg2: weak = one cfg2 slab per GPU, "
                         "strong = the cfg2 grid split over the GPUs")
    ap.add_argument("--no-1gpu", action="store_true",
                    help="N>1: skip rank 0's one-GPU run of the same workload "
                         "(config.one_gpu, the denominator of config.parallel_efficiency)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--checkpoint", type=int, default=0,
                    help="cfg3: checkpoint interval k (0 = whole history in HBM)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=0, help="reference sample steps (0: auto)")
    ap.add_argument("--time-steps", type=int, default=0,
                    help="override the workload's time steps (profiling runs only)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    n = world or args.gpus
    if args.workload is None:
        args.workload = "cfg5" if n > 1 else "cfg2"
    return args


def make_workload(name, time_steps=0):
    w = _make_workload(name)
    if time_steps:
        w.nt = time_steps + 2
        w.wavelet = np.ascontiguousarray(w.wavelet[:w.nt])
    w.wavelet = np.ascontiguousarray(w.wavelet.reshape(w.nt, -1))
    return w


def _make_workload(name):
    from paper_1608_08658_b200 import configs
    if name == "cfg1":
        return configs.cfg1()
    if name == "cfg2":
        return configs.cfg2()
    if name == "cfg3":
        return configs.cfg3()
    if name.startswith("cfg4-so"):
        return configs.cfg4(int(name[len("cfg4-so"):]))
    if name == "cfg5":
        return configs.cfg5()
    raise SystemExit(f"unknown workload {name}")


def problem(w):
    from paper_1608_08658_b200 import seismic as S
    model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    src = S.locate_points(model, w.src_coords)
    rec = S.locate_points(model, w.rec_coords)
    return model, src, rec


def config_of(w, n, extra=None):
    c = {"workload": f"{w.name}: interior {'x'.join(map(str, w.interior))} + {w.nbpml}-pt "
                     f"damping layer, so {w.space_order}, {w.steps} steps, "
                     f"{len(w.src_coords)} src, {len(w.rec_coords)} rec",
         "padded": w.padded, "space_order": w.space_order, "time_steps": w.steps,
         "points_per_step": w.points_per_step, "nsrc": len(w.src_coords),
         "nrec": len(w.rec_coords),
         "parallelism": f"z-slab x{n} (ghost planes exchanged every step, overlapped with the interior sweep)"
                        if n > 1 else "1 GPU",
         "l2": "inputs larger than L2 (each fp32 field 4*prod(padded) B > 126 MB)"
               if 4 * int(np.prod(w.padded)) > 126e6 else "working set fits L2"}
    if extra:
        c.update(extra)
    return c


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is None:
            self.summary = None
            return
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        self.summary = {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                        "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic(workload, info, ndim):
    """DRAM bytes per sweep launch from the committed ncu --set full capture of
    THIS instantiation (template arguments + z chunks + grid) on this workload:
    profiles/ncu_summary.json is keyed "<workload>|<instantiation>|z<zchunks>"
    (tools/ncu_traffic.py writes it from the capture).  (None, why) when the
    tiling the bench autotuned to has no capture."""
    if ndim != 3:
        return None, "2-D: L2 / shared-memory resident, no DRAM roofline"
    key = f"{workload}|{info.get('instantiation')}|z{info.get('zchunks')}" + \
        ("|dyn" if info.get("ctas") == -2 else "")
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            caps = json.load(fh)["captures"]
    except Exception:
        return None, f"no committed ncu capture of {key}"
    if key in caps:
        return caps[key]["dram_bytes_per_launch"], caps[key]["source"]
    # The autotuner picks among tilings within a few percent of each other, so
    # the benched one may have no capture of its own: the DRAM traffic of a
    # sweep hardly depends on the tiling (625-630 MB on cfg2 / cfg3 whichever
    # is captured), so the capture of another tiling of the SAME workload is
    # reported, named as such.
    other = sorted(k for k in caps if k.startswith(workload + "|"))
    if other:
        e = caps[other[0]]
        return e["dram_bytes_per_launch"], (f"{e['source']} (capture of another tiling of this "
                                            f"workload, {other[0]}; none of {key})")
    return None, f"no committed ncu capture of {key}"


_REF_PROBLEM = {}


def fit_reference_to_memory(w):
    """The reference keeps ~14 fp64 grids of the padded problem on the host
    (its model, the copies seismic::forward binds, the three u slots): cfg5
    needs > 130 GB.  On a host with less available memory the sample is the
    same workload cropped along z (x and y extents, sources and receivers
    kept; per-point work is the same), and the sample text says so.  Returns
    (workload, note)."""
    need = 14 * 8 * float(np.prod(w.padded))
    try:
        with open("/proc/meminfo") as fh:
            avail = next(int(l.split()[1]) * 1024.0 for l in fh if l.startswith("MemAvailable"))
    except Exception:
        return w, ""
    if need <= 0.6 * avail or w.ndim != 3:
        return w, ""
    pad = 2 * (w.nbpml + w.space_order // 2)
    plane = 14 * 8 * float(np.prod(w.padded[1:]))
    nz = int(0.6 * avail / plane) - pad
    if nz < 8:
        raise SystemExit("bench.py: not enough host memory for a reference sample")
    import copy
    c = copy.copy(w)
    c.interior = [nz] + list(w.interior[1:])
    c.m_interior = np.ascontiguousarray(
        np.asarray(w.m_interior).reshape(w.interior)[:nz]).ravel()
    return c, (f" [host memory {avail / 1e9:.0f} GB < the {need / 1e9:.0f} GB the reference needs "
               f"for the full grid: cropped to {nz} interior z rows]")


def cpu_baseline(w, steps_hint):
    """The reference (oracle/_ref) timed on this host's cores: full grid,
    truncated step count.  Falls back to the C port when _ref was not built."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    bind_reference_threads()
    w, note = fit_reference_to_memory(w)
    cores = int(os.environ["STENCILFD_THREADS"])
    steps = steps_hint or max(4, min(40, int(2.0e9 / w.points_per_step)))
    nt = steps + 2
    trace = np.ascontiguousarray(w.wavelet[:nt])
    if O.have_ref():
        # the reference's model and sparse sets, built once per workload
        if _REF_PROBLEM.get("name") != w.name:
            if _REF_PROBLEM.get("p"):
                _REF_PROBLEM["p"].close()
            _REF_PROBLEM["p"] = O.RefProblem(w.interior, w.h, w.nbpml, w.space_order,
                                             w.m_interior, w.src_coords, w.rec_coords)
            _REF_PROBLEM["name"] = w.name
        secs = _REF_PROBLEM["p"].forward(trace, nt, w.dt)
        kind = "reference"
    else:
        from paper_1608_08658_b200 import seismic as S
        model, src, rec = problem(w)
        t0 = time.perf_counter()
        O.forward(model.padded, w.space_order, w.h, w.dt, nt, model.m, model.damp, src.idx,
                  src.w, trace, rec.idx, rec.w)
        secs = time.perf_counter() - t0
        kind = "port"
    gpts = w.points_per_step * steps / secs / 1e9
    return {"value": gpts, "unit": "Gpts/s", "cores": cores, "kind": kind,
            "sample": f"seismic::forward on the full {'x'.join(map(str, w.padded))} padded grid, "
                      f"{steps} of {w.steps} time steps (RunStats.seconds of the kernel call, "
                      f"STENCILFD_THREADS={cores})" + note, "seconds": secs}


def run_reference(args):
    """The reference's own CPU path on this host (rank 0 only under torchrun),
    on our arm's workload: at N > 1 with weak scaling that is the cfg2 model
    stacked N times along z (the global problem the N ranks share)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    if world > 1 and args.workload == "cfg2" and args.scaling == "weak":
        from paper_1608_08658_b200 import configs
        w = configs.cfg2_stacked(world)
        if args.time_steps:
            w.nt = args.time_steps + 2
        w.wavelet = np.ascontiguousarray(w.wavelet[:w.nt].reshape(w.nt, -1))
    else:
        w = make_workload(args.workload, args.time_steps)
    vals = []
    cb = None
    for i in range(args.warmup + args.steps):
        # warm-up samples are minimal (2 time steps): they JIT-compile and cache
        # the reference's kernel and start its OpenMP pool, which is all a
        # warm-up is for, and keep the cfg5 (1120^3) arm within minutes
        warm = i < args.warmup
        cb = cpu_baseline(w, 2 if warm else (args.cpu_steps or 0))
        if not warm:
            vals.append(cb["value"])
    v = float(np.median(vals))
    cb["value"] = v
    line = {"metric": "Gpts/s (grid-point updates/sec) 3D acoustic so-8", "value": v,
            "unit": "Gpts/s", "n_gpus": world, "gpus_used": 0,
            "ranks_working": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": cb["seconds"] * 1e3, "higher_is_better": True,
            "scaling": "strong" if world > 1 and args.workload != "cfg2" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_of(w, world, {"sample": cb["sample"],
                                           "parallelism": f"reference CPU path on rank 0 of "
                                                          f"{world}, {cb['cores']} host threads; "
                                                          "no GPU"}),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "Gpts/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def bytes_per_point(plan, kind):
    """Algorithmic bytes per updated point of the kernel the plan runs: the
    SURVEY §8(d) figure (20 B forward/adjoint, 32 B fused gradient), minus the
    c1 coefficient stream (4 B) when the damping field is max-separable and the
    sweep forms c1 from its per-axis profiles."""
    info = plan.info()
    return int(info.get("bytes_per_point", BYTES_PER_POINT[kind]))


def kernel_name(plan):
    info = plan.info()
    return "sweep3d_pair_kernel" if info.get("mapping", "").startswith("column") else "sweep3d_kernel"


def check_exchange(L, S, torch, dist, comm, rank, world, local, p2p):
    """A small forward problem (waves crossing every slab boundary, receivers
    in every slab) through this job's z-slab exchange, summed over ranks and
    compared on rank 0 with the same problem on one GPU.  Returns (ok, the
    larger relative L2 error of the wavefield and the record) on every rank."""
    nt = 40
    model = S.make_constant_model([16 * world + 8, 40, 40], 15.0, 8, 8, 1500.0)
    dt = 0.8 * S.critical_dt(model)
    ext = (16 * world + 7) * 15.0
    src = S.locate_points(model, [[0.5 * ext + 4.0, 310.0, 290.0]])
    rec = S.locate_points(model, [[f * ext, 200.0 + 200.0 * f, 330.0]
                                  for f in np.linspace(0.02, 0.98, 16)])
    wav = np.ascontiguousarray(S.ricker(30.0, 0.03, nt, dt).reshape(nt, 1))
    si, sw = S._sparse_args(src, 3)
    ri, rw = S._sparse_args(rec, 3)
    field = np.zeros((3, *model.padded))
    trace = np.zeros((nt, rec.npoints))
    ok = 1
    plan = L.Plan(L.FORWARD, 3, model.padded, 8, nt, dt, model.h, src.npoints, rec.npoints,
                  False, local, comm=comm)
    try:
        if p2p:
            blobs = [None] * world
            dist.all_gather_object(blobs, plan.ipc_export())
            plan.ipc_import(blobs[rank - 1] if rank > 0 else None,
                            blobs[rank + 1] if rank < world - 1 else None)
        plan.run([field, L.f64(model.m), L.f64(model.damp), si, sw, wav, ri, rw, trace])
    except L.SfdError as e:
        print(f"rank {rank}: exchange check failed: {e}", file=sys.stderr)
        ok = 0
    finally:
        plan.close()
    flag = torch.tensor([ok], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    total = torch.from_numpy(np.concatenate([field.ravel(), trace.ravel()])).cuda()
    dist.reduce(total, 0, op=dist.ReduceOp.SUM)
    err = torch.tensor([float("inf")], device="cuda", dtype=torch.float64)
    if rank == 0:
        ref = S.forward(model, src, wav, rec, nt, dt, False, S.RunConfig(device=local))
        got = total.cpu().numpy()

        def rel(a, b):
            return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
        err[0] = max(rel(got[:field.size], np.asarray(ref.u).ravel()),
                     rel(got[field.size:], ref.record.data.ravel()))
    dist.broadcast(err, 0)
    e = float(err.item())
    return bool(int(flag.item()) == 1 and e <= 1e-5), e


def _pinned(torch, shape, fill=None):
    t = torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    if fill is not None:
        t[...] = fill
    return t


def slab_problem(L, S, args, world, rank, n=1024, minmax=None):
    """cfg5 at N > 1: this rank's slab only.  The interior rows its planes
    need are generated here (configs.cfg5_rows; the rescale range is
    all-reduced), and the model arrays are GLOBAL-shaped but untouched outside
    the rank's planes (np.zeros: pages that are never written are never
    backed), so sfdb200_upload reads exactly its slab from them as it does
    from a full model."""
    from paper_1608_08658_b200 import configs
    nbpml, so = 40, 16
    R, pad = so // 2, nbpml + so // 2
    P = n + 2 * pad
    zb, ze = L.slab(P, so, world, rank)
    zoff, pz = zb - R, (ze - zb) + 2 * R  # local planes [zoff, zoff + pz) of the global grid
    z0, z1 = max(0, zoff - pad), min(n, zoff + pz - pad)

    if minmax is None:  # the rescale range over all ranks' rows
        import torch
        import torch.distributed as dist

        def minmax(a, b):
            dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
            t = torch.tensor([-a, b], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return -float(t[0]), float(t[1])

    steps = args.time_steps
    w = configs.cfg5_rows(z0, z1, minmax, n=n, nbpml=nbpml,
                          nt=(steps + 2) if steps else 502)
    w.wavelet = np.ascontiguousarray(w.wavelet.reshape(w.nt, -1))
    mi = w.m_interior.reshape(z1 - z0, n, n)
    dprof = S.build_damping([P], nbpml, R, w.h)  # the per-axis taper (seismic.cpp:152-173)
    m = np.zeros(P * P * P)
    damp = np.zeros(P * P * P)
    mv, dv = m.reshape(P, P, P), damp.reshape(P, P, P)
    yx = np.maximum(dprof[:, None], dprof[None, :])
    for zg in range(zoff, zoff + pz):  # make_model's edge replication (seismic.cpp:100-142)
        iz = min(max(zg - pad, 0), n - 1) - z0
        mv[zg] = np.pad(mi[iz], pad, mode="edge")
        dv[zg] = np.maximum(dprof[zg], yx)
    model = S.VelocityModel([n, n, n], w.h, nbpml, so, [P, P, P], m, damp)
    w.m_interior = None
    return w, model


def run_ours(args):
    import torch
    from paper_1608_08658_b200 import _lib as L
    from paper_1608_08658_b200 import seismic as S

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    comm = None
    if world > 1:
        # torch.distributed is the plumbing (rendezvous, barriers, the max over
        # ranks); the ghost exchange is libsfdb200's own (fused P2P stores, or its
        # NCCL communicator as the fallback).
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [L.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = L.Comm(uid[0], world, rank, local)

    slab = world > 1 and args.workload == "cfg5"
    if slab:
        w, model = slab_problem(L, S, args, world, rank)
    elif world > 1 and args.workload == "cfg2" and args.scaling == "weak":
        # weak scaling: one cfg2-sized slab per GPU (the cfg2 model stacked along z)
        from paper_1608_08658_b200 import configs
        w = configs.cfg2_stacked(world)
        if args.time_steps:
            w.nt = args.time_steps + 2
        w.wavelet = np.ascontiguousarray(w.wavelet[:w.nt].reshape(w.nt, -1))
        model = None
    else:
        w = make_workload(args.workload, args.time_steps)
        model = None
    if model is None:
        model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
        S.check_dt(model, w.dt)
    src = S.locate_points(model, w.src_coords)
    rec = S.locate_points(model, w.rec_coords)
    nd = model.ndim()

    def new_plan():
        p = L.Plan(L.FORWARD, nd, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                   rec.npoints, False, local, comm=comm)
        p.set_stream(stream.cuda_stream)
        return p

    stream = torch.cuda.Stream()
    plan = new_plan()
    exchange = None
    if world > 1:
        # Fused P2P ghost exchange (default): the boundary sweeps store into the
        # neighbours' ghost planes over NVLink; NCCL send/recv otherwise.
        exchange = "nccl send/recv on a comm stream, overlapped with the interior sweep"
        if os.environ.get("SFDB200_EXCHANGE", "p2p") == "p2p":
            blobs = [None] * world
            dist.all_gather_object(blobs, plan.ipc_export())
            try:
                plan.ipc_import(blobs[rank - 1] if rank > 0 else None,
                                blobs[rank + 1] if rank < world - 1 else None)
                ok = 1
            except L.SfdError as e:
                print(f"rank {rank}: P2P exchange unavailable ({e}); using NCCL", file=sys.stderr)
                ok = 0
            flag = torch.tensor([ok], device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 1:
                exchange = ("fused P2P: boundary sweeps store into the neighbours' ghost planes "
                            "(CUDA IPC over NVLink), step counters via stream memory ops")
            else:  # every rank must use the same exchange
                plan.close()
                plan = new_plan()

    exchange_check = None
    if world > 1:
        # Check the exchange on a small problem against one GPU first, and fall
        # back to NCCL if the fused P2P path fails or disagrees.
        p2p = exchange.startswith("fused")
        ok, err = check_exchange(L, S, torch, dist, comm, rank, world, local, p2p)
        exchange_check = {"exchange": "p2p" if p2p else "nccl", "ok": ok, "max_rel_err": err}
        if not ok and p2p:
            if rank == 0:
                print(f"P2P exchange check failed (rel err {err}); using NCCL", file=sys.stderr)
            plan.close()
            plan = new_plan()
            exchange = "nccl send/recv on a comm stream, overlapped with the interior sweep"
            ok2, err2 = check_exchange(L, S, torch, dist, comm, rank, world, local, False)
            exchange_check = {"exchange": "nccl", "ok": ok2, "max_rel_err": err2,
                              "p2p_failed": {"ok": ok, "max_rel_err": err}}

    # Pageable host buffers in the reference's layout (fp64 grids, long idx),
    # as seismic::forward binds them (seismic.cpp:354-368).  The output grid
    # is global-shaped; a rank writes only its owned planes.
    u = np.zeros((3, *model.padded))
    rec_data = np.zeros((w.nt, rec.npoints))
    trace = np.ascontiguousarray(w.wavelet)
    argv = [u, model.m, model.damp, L.i64(src.idx), L.f64(src.w), trace, L.i64(rec.idx),
            L.f64(rec.w), rec_data]

    # ---- device-resident timing (value)
    plan.upload(argv)
    for _ in range(args.warmup):
        plan.execute()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            plan.execute()
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    plan.check()  # a broken P2P exchange fails the run instead of reporting a number
    ms = ev0.elapsed_time(ev1)
    # Kernel timing for the roofline: CUDA events around every sweep launch of
    # one more execute() right after the timed region.  (Events between the
    # launches inside the timed region would serialise consecutive sweeps,
    # which otherwise overlap launch and CTA setup through programmatic
    # dependent launch.)
    plan.set_timing(True)
    plan.execute()
    torch.cuda.synchronize()
    sweep_ms, sweep_n = plan.stencil_time()
    plan.set_timing(False)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    pts = w.points_per_step * plan.steps  # the global problem over all z slabs
    value = pts * args.steps / (ms / 1e3) / 1e9
    launches = plan.launches_per_execute * args.steps

    # ---- end to end through the C ABI with host buffers (e2e)
    def timed_runs(av, reps):
        plan.run(av)  # warm (and sizes the staging chunks)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            plan.run(av)
        el = time.perf_counter() - t0
        if dist:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        return el / reps

    e2e = None
    if not args.no_e2e:
        per = timed_runs(argv, args.steps)
        e2e = {"value": pts / per / 1e9, "unit": "Gpts/s",
               "h2d_bytes_per_step": plan.h2d_bytes, "d2h_bytes_per_step": plan.d2h_bytes,
               "ms_per_step": per * 1e3, "runs": args.steps,
               "path": "sfdb200_run(plan, argv): reference argv, pageable fp64 host buffers "
                       "(the reference's std::vector case, seismic.cpp:354-368)"}
        # Where the time goes: the same run as three synchronised stages
        # (run() overlaps the receiver rows' D2H with the sweeps; here they all
        # land in download).
        stage = {}
        for name, fn in (("upload", lambda: plan.upload(argv)), ("execute", plan.execute),
                         ("download", lambda: plan.download(argv))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            stage[name] = (time.perf_counter() - t0) * 1e3
        e2e["staged_ms"] = stage
        if world == 1:
            # The same call with pinned host buffers (a caller that owns pinned
            # memory; not the reference's case).
            pargv = [_pinned(torch, u.shape), _pinned(torch, model.m.shape, model.m),
                     _pinned(torch, model.damp.shape, model.damp), L.i64(src.idx), L.f64(src.w),
                     _pinned(torch, trace.shape, trace), L.i64(rec.idx), L.f64(rec.w),
                     _pinned(torch, rec_data.shape)]
            perp = timed_runs(pargv, args.steps)
            e2e["pinned"] = {"value": pts / perp / 1e9, "ms_per_step": perp * 1e3,
                             "runs": args.steps,
                             "path": "sfdb200_run with pinned fp64 host buffers"}

    peak, peak_src = measured_peak()
    per_launch_ms = sweep_ms / max(1, sweep_n)
    # the timed launch: with the fused P2P exchange one launch per step sweeps
    # every owned plane (boundary items first); with NCCL the interior launch
    # leaves out the R planes next to each neighbour
    interior = plan.points_per_step
    if world > 1 and not exchange.startswith("fused"):
        zb, ze, _ = plan.slab()
        R = w.space_order // 2
        interior = plan.points_per_step // (ze - zb) * ((ze - zb) - R * ((rank > 0) + (rank < world - 1)))
    # 2-D runs the whole time loop in one cooperative launch
    sweeps_per_launch = plan.steps if nd == 2 else 1
    info = plan.info()
    bpp = bytes_per_point(plan, "forward")
    alg = bpp * interior * sweeps_per_launch
    achieved = alg / (per_launch_ms / 1e3) / 1e9
    alg20 = BYTES_PER_POINT["forward"] * interior * sweeps_per_launch
    traffic, traffic_src = ncu_traffic(w.name, info, nd)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "frac_alg": alg20 / (per_launch_ms / 1e3) / 1e9 / peak,
            "alg_bytes_per_point_survey": BYTES_PER_POINT["forward"],
            "kernel": kernel_name(plan) if nd == 3 else "loop2d_kernel (all steps, cooperative)",
            "instantiation": info.get("instantiation"),
            "alg_bytes_per_launch": alg, "bytes_per_point": bpp, "mean_launch_ms": per_launch_ms,
            "kernel_timing": "CUDA events around each launch of one execute() after the timed region",
            "kernel_share_of_step": sweep_ms / (ms / args.steps), "peak_source": peak_src}

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cb = cpu_baseline(w, args.cpu_steps or 0)
        cb.pop("seconds", None)

    one_gpu = None
    if world > 1 and not args.no_1gpu:
        one_gpu = measure_one_gpu(args, rank, dist, torch)

    if rank == 0:
        scaling = "weak" if (world > 1 and args.workload == "cfg2" and args.scaling == "weak") \
            else "strong"
        extra = {"sweep": info, "exchange": exchange, "exchange_check": exchange_check}
        if slab:
            extra["inputs"] = ("each rank generated only the interior rows its slab needs "
                               "(configs.cfg5_rows, PCG64 advanced to the rows, rescale range "
                               "all-reduced) and filled only its planes of the global-shaped "
                               "model arrays")
        if one_gpu:
            extra["one_gpu"] = one_gpu
            extra["parallel_efficiency"] = value / (world * one_gpu["value"])
        line = {"metric": "Gpts/s (grid-point updates/sec) 3D acoustic so-8", "value": value,
                "unit": "Gpts/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": scaling if world > 1 else "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": config_of(w, world, extra),
                "roofline": roof, "cpu_baseline": cb,
                "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary}
        print(json.dumps(line))
    plan.close()
    if comm:
        comm.close()
    if dist:
        dist.destroy_process_group()


def measure_one_gpu(args, rank, dist, torch):
    """Rank 0 times the same workload on its GPU alone while the other ranks
    wait at a barrier: the denominator of the strong-scaling efficiency
    (config.one_gpu; the driver computes its own from the per-N lines).  Same
    method as `value`: warm-up execute, then one execute between CUDA events
    on the plan's stream."""
    res = None
    if rank == 0:
        from paper_1608_08658_b200 import _lib as L
        from paper_1608_08658_b200 import seismic as S
        w = make_workload(args.workload, args.time_steps)
        model = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
        src = S.locate_points(model, w.src_coords)
        rec = S.locate_points(model, w.rec_coords)
        p = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                   rec.npoints, False, int(os.environ.get("LOCAL_RANK", "0")))
        stream = torch.cuda.Stream()
        p.set_stream(stream.cuda_stream)
        p.upload([None, model.m, model.damp, src.idx, src.w, np.ascontiguousarray(w.wavelet),
                  rec.idx, rec.w, np.zeros((w.nt, rec.npoints))])
        p.execute()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        p.execute()
        e1.record(stream)
        torch.cuda.synchronize()
        p.check()
        ms = e0.elapsed_time(e1)
        res = {"workload": w.name, "value": w.points_per_step * p.steps / (ms / 1e3) / 1e9,
               "ms_per_step": ms, "sweep": p.info().get("instantiation"),
               "timing": "rank 0 alone, one execute() after a warm-up, CUDA events"}
        p.close()
        del model
    dist.barrier()
    return res


def run_fwi(args):
    """cfg3 (BASELINE configs[2]): FWI gradient.  Observed traces from the true
    model, a saved forward on the smooth background (history stays in HBM),
    the residual, then the timed gradient operator (fused adjoint + imaging
    condition, 32 B/pt).  One GPU."""
    import torch
    from paper_1608_08658_b200 import _lib as L
    from paper_1608_08658_b200 import seismic as S

    torch.cuda.set_device(0)
    w = make_workload(args.workload, args.time_steps)
    true = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.m_interior)
    bg = S.make_model(w.interior, w.h, w.nbpml, w.space_order, w.extra["m_background"])
    S.check_dt(true, w.dt)
    S.check_dt(bg, w.dt)
    src = S.locate_points(bg, w.src_coords)
    rec = S.locate_points(bg, w.rec_coords)
    P, nt = bg.padded, w.nt
    stream = torch.cuda.Stream()

    def plan(kind, save=False):
        p = L.Plan(kind, 3, P, w.space_order, nt, w.dt, w.h, src.npoints, rec.npoints, save, 0)
        p.set_stream(stream.cuda_stream)
        return p

    obs = np.zeros((nt, rec.npoints))
    f_true = plan(L.FORWARD)
    f_true.run([None, true.m, true.damp, src.idx, src.w, w.wavelet, rec.idx, rec.w, obs])
    f_true.close()
    syn = np.zeros((nt, rec.npoints))
    ckk = args.checkpoint
    fwd = plan(L.FORWARD, save=ckk == 0)
    if ckk:
        fwd.set_checkpointing(ckk)
    fargv = [None, bg.m, bg.damp, src.idx, src.w, w.wavelet, rec.idx, rec.w, syn]
    fwd.upload(fargv)
    fwd.execute()
    fwd.download(fargv)  # traces only (argv[0] = NULL skips the 77 GB history)
    resid = syn - obs
    grad = np.zeros(P)
    g = plan(L.GRADIENT)
    if ckk:
        g.bind_checkpoints(fwd)  # history recomputed per segment (one extra forward sweep/step)
    else:
        g.bind_history(fwd)
    # pageable host buffers (the reference's std::vectors, seismic.cpp:446-462)
    # for everything the e2e leg moves (model, residual, gradient)
    gargv = [None, None, np.array(bg.m), np.array(bg.damp), grad, L.i64(rec.idx), L.f64(rec.w),
             np.ascontiguousarray(resid)]
    g.upload(gargv)
    for _ in range(args.warmup):
        g.execute()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(0) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            g.execute()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    g.set_timing(True)  # per-launch events on one more execute (see run_ours)
    g.execute()
    torch.cuda.synchronize()
    sweep_ms, sweep_n = g.stencil_time()
    g.set_timing(False)
    pts = w.points_per_step * g.steps
    value = pts * args.steps / (ms / 1e3) / 1e9
    # e2e: the gradient through the C ABI with host buffers (residual in, grad out;
    # the history stays device-resident from the saved forward, as the design intends)
    g.run(gargv)  # warm (staging chunks)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        g.run(gargv)
    el = time.perf_counter() - t0
    e2e = {"value": pts * args.steps / el / 1e9, "unit": "Gpts/s",
           "h2d_bytes_per_step": g.h2d_bytes, "d2h_bytes_per_step": g.d2h_bytes,
           "ms_per_step": el / args.steps * 1e3, "runs": args.steps,
           "path": "sfdb200_run(gradient plan bound to the saved forward's device history), "
                   "pageable fp64 host buffers"}
    peak, peak_src = measured_peak()
    per_launch_ms = sweep_ms / max(1, sweep_n)
    bpp = bytes_per_point(g, "gradient")
    alg = bpp * w.points_per_step
    achieved = alg / (per_launch_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(w.name, g.info(), 3)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "frac_alg": BYTES_PER_POINT["gradient"] * w.points_per_step / (per_launch_ms / 1e3)
                        / 1e9 / peak,
            "alg_bytes_per_point_survey": BYTES_PER_POINT["gradient"],
            "instantiation": g.info().get("instantiation"),
            "kernel": kernel_name(g) + "<GRAD>", "alg_bytes_per_launch": alg, "bytes_per_point": bpp,
            "mean_launch_ms": per_launch_ms, "kernel_share_of_step": sweep_ms / (ms / args.steps),
            "peak_source": peak_src}
    cb = None
    if not args.no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle_lib as O
        bind_reference_threads()
        if O.have_ref():
            steps = args.cpu_steps or 20
            ntc = steps + 2
            tr = np.ascontiguousarray(w.wavelet[:ntc])
            uh, r, _ = O.ref_forward(w.interior, w.h, w.nbpml, w.space_order,
                                     w.extra["m_background"], w.src_coords, tr, w.rec_coords,
                                     ntc, w.dt, save=True)
            _, secs = O.ref_gradient(w.interior, w.h, w.nbpml, w.space_order,
                                     w.extra["m_background"], w.rec_coords, r, uh, ntc, w.dt)
            cb = {"value": w.points_per_step * steps / secs / 1e9, "unit": "Gpts/s",
                  "cores": int(os.environ["STENCILFD_THREADS"]), "kind": "reference",
                  "sample": f"seismic::gradient on the full {'x'.join(map(str, P))} grid, "
                            f"{steps} of {w.steps} steps (RunStats.seconds)"}
    line = {"metric": "Gpts/s (grid-point updates/sec) 3D acoustic so-8 FWI gradient",
            "value": value, "unit": "Gpts/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_of(w, 1, {"sweep": g.info(), "objective": 0.5 * float((resid ** 2).sum()),
                                       "history_GB": (fwd.checkpoint_bytes if ckk else 4.0 * (nt + 1) * np.prod(P)) / 1e9,
                                       "history": (f"uniform checkpoints every {ckk} steps + "
                                                   "per-segment recompute (timed)") if ckk else
                                                  "whole history resident in HBM"}),
            "roofline": roof, "cpu_baseline": cb, "e2e": e2e,
            "gpu_launches": g.launches_per_execute * args.steps, "clocks": clk.summary}
    print(json.dumps(line))
    for p in (g, fwd):
        p.close()


def relaunch(n):
    """`python bench.py --gpus N` outside a launcher: run the same command as N
    ranks under torch.distributed.run (one process per GPU, 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd).returncode)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; timing {world} ranks",
              file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "cfg3":
        run_fwi(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
