"""Command-line driver mirroring the reference's `sfd` tool
(proj/tools/sfd.cpp:26-567) on the B200 backend:

    python -m paper_1608_08658_b200 run    [--config c.json] [--set a.b=v ...] [--out dir]
    python -m paper_1608_08658_b200 bench  ...
    python -m paper_1608_08658_b200 verify adjoint|taylor ...

Same JSON config keys and defaults (sfd.cpp:26-54), `--set` dotted overrides
parsed as JSON with a plain-string fallback (sfd.cpp:58-78), the same output
files (record.{bin,json}, wavefield.{bin,json}, summary.json, bench.jsonl/.csv,
report.jsonl) and exit codes (2 = refused).  The CPU-code-generation keys
(parallel, simd, block_mode, fixed_blocks, blocks, candidates, preset) are
accepted and ignored: the device tiling is autotuned per plan.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time

import numpy as np

from . import _lib as L
from . import seismic as S
from . import verify as V

DEFAULTS = {
    "physics": "acoustic", "interior": [68, 68, 24], "h": 15.0, "nbpml": 13,
    "space_order": 8, "velocity": 1500.0, "model_file": "", "f0": 10.0, "t0": 0.0,
    "time": 1.0, "nt": 0, "dt": 0.0, "amplitude": 1.0, "save": False, "seed": 0,
    "parallel": True, "simd": True, "block_mode": "best-guess", "fixed_blocks": [8, 8],
    "blocks": [], "candidates": [], "preset": "generic", "kernel": "forward", "source": [],
    "receivers": 8, "device": 0,
}


def build_patch(config_path, sets):
    patch = {}
    if config_path:
        with open(config_path) as fh:
            patch = json.load(fh)
    for kv in sets or []:
        if "=" not in kv or kv.startswith("="):
            raise ValueError(f"--set expects key=value, got '{kv}'")
        key, raw = kv.split("=", 1)
        try:
            value = json.loads(raw)
        except json.JSONDecodeError:
            value = raw
        node = patch
        parts = key.split(".")
        for p in parts[:-1]:
            node = node.setdefault(p, {})
        node[parts[-1]] = value
    return patch


def build_experiment(patch):
    """sfd.cpp:117-195"""
    cfg = dict(DEFAULTS)
    cfg.update(patch)
    order = int(cfg["space_order"])
    if cfg["model_file"]:
        model = S.load_model(cfg["model_file"], order)
    else:
        model = S.make_constant_model(cfg["interior"], float(cfg["h"]), int(cfg["nbpml"]), order,
                                      float(cfg["velocity"]))
    dt = float(cfg["dt"]) if float(cfg["dt"]) > 0 else 0.9 * S.critical_dt(model)
    nt = int(cfg["nt"]) if int(cfg["nt"]) > 0 else max(4, int(round(float(cfg["time"]) / dt)) + 1)
    nd = model.ndim()
    span = [(n - 1) * model.h for n in model.interior]
    src_c = list(cfg["source"]) or [0.5 * s for s in span]
    nrec = int(cfg["receivers"])
    rec_c = []
    for p in range(nrec):
        c = [0.0] * nd
        if nd > 1:
            c[0] = 0.7 * span[0]
        for d in range(1, nd - 1):
            c[d] = 0.5 * span[d]
        frac = 0.5 if nrec == 1 else 0.1 + 0.8 * p / (nrec - 1)
        c[nd - 1] = frac * span[nd - 1]
        rec_c.append(c)
    f0 = float(cfg["f0"])
    t0 = float(cfg["t0"]) if float(cfg["t0"]) > 0 else 1.2 / f0
    trace = S.ricker(f0, t0, nt, dt) * float(cfg["amplitude"])
    return {"cfg": cfg, "model": model, "dt": dt, "nt": nt, "src_coords": [src_c],
            "rec_coords": rec_c, "src": S.locate_points(model, [src_c]),
            "rec": S.locate_points(model, rec_c), "trace": trace,
            "run": S.RunConfig(int(cfg["device"]))}


def dump_grid(data, shape, halo, time_slots, prefix):
    """runtime.cpp:425-440: raw float64 + JSON sidecar."""
    np.asarray(data, "<f8").tofile(prefix + ".bin")
    with open(prefix + ".json", "w") as fh:
        json.dump({"shape": list(map(int, shape)), "halo": int(halo), "dtype": "float64",
                   "time_slots": int(time_slots)}, fh, indent=2)
        fh.write("\n")


def write_summary(out, summary):
    with open(os.path.join(out, "summary.json"), "w") as fh:
        json.dump(summary, fh, indent=2)
        fh.write("\n")


def cmd_run(patch, out):
    """sfd.cpp:309-355"""
    ex = build_experiment(patch)
    save = bool(ex["cfg"]["save"])
    f = S.forward(ex["model"], ex["src"], ex["trace"], ex["rec"], ex["nt"], ex["dt"], save,
                  ex["run"])
    S.save_record(f.record, ex["rec_coords"], os.path.join(out, "record"))
    slots = S.history_rows(ex["nt"]) if save else 3
    dump_grid(f.u, [slots, *ex["model"].padded], ex["model"].halo(), slots,
              os.path.join(out, "wavefield"))
    summary = {"command": "run", "passed": True, "entry": "Forward", "plan": "b200",
               "nt": ex["nt"], "dt": ex["dt"], "save": save, "seconds": f.stats.seconds,
               "gpts": f.stats.gpts, "record_peak": float(np.abs(f.record.data).max(initial=0)),
               "wavefield_peak": float(np.abs(f.u).max(initial=0)),
               "record": os.path.join(out, "record.bin"),
               "wavefield": os.path.join(out, "wavefield.bin")}
    write_summary(out, summary)
    print(f"Forward: nt {ex['nt']}, dt {ex['dt']}, {f.stats.seconds} s, {f.stats.gpts} Gpts/s, "
          f"record peak {summary['record_peak']}")
    return 0


def cmd_bench(patch, out):
    """sfd.cpp:445-515: roofline rows for the device run (device-resident and end to end)."""
    ex = build_experiment(patch)
    m, src, rec = ex["model"], ex["src"], ex["rec"]
    nt, dt = ex["nt"], ex["dt"]
    plan = L.Plan(L.FORWARD, m.ndim(), m.padded, m.space_order, nt, dt, m.h, src.npoints,
                  rec.npoints, False, ex["run"].device)
    rec_data = np.zeros((nt, rec.npoints))
    argv = [None, m.m, m.damp, src.idx, src.w, ex["trace"], rec.idx, rec.w, rec_data]
    t0 = time.perf_counter()
    plan.run(argv)  # includes the per-plan autotune
    first = time.perf_counter() - t0
    plan.set_timing(True)
    t0 = time.perf_counter()
    plan.run(argv)
    e2e = time.perf_counter() - t0
    ms, n = plan.stencil_time()
    pts = plan.points_per_step * plan.steps
    sweeps = plan.steps if m.ndim() == 3 else 1
    dev_s = ms / 1e3 * (sweeps / max(1, n)) if m.ndim() == 3 else ms / 1e3
    info = plan.info()
    bpp = int(info.get("bytes_per_point", 20))
    # the device update's arithmetic per point: per
    # radius k, 2 ndim - 1 neighbour adds, the centre term and the tap (FMA = 2);
    # then u1 + c1 (u1 - u2) + c2 lap.
    fpp = (m.space_order // 2) * (2 * m.ndim() + 2) + 5

    def row(plan_name, seconds, **extra):
        # the reference's roofline-row keys (verify.hpp:110-119, verify.cpp:380-392)
        r = {"kernel": "Forward", "flops_per_point": fpp, "bytes_per_point": bpp,
             "intensity": fpp / bpp, "seconds": seconds, "gflops": fpp * pts / seconds / 1e9,
             "plan": plan_name, "blocks": [], "gpts": pts / seconds / 1e9}
        r.update(extra)
        return r

    rows = [row("b200-device", dev_s, gbps=bpp * pts / dev_s / 1e9, config=info),
            row("b200-e2e", e2e, h2d_bytes=plan.h2d_bytes, d2h_bytes=plan.d2h_bytes)]
    with open(os.path.join(out, "bench.jsonl"), "w") as fh:
        for r in rows:
            fh.write(json.dumps(r) + "\n")
    with open(os.path.join(out, "bench.csv"), "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow(["kernel", "plan", "blocks", "seconds", "gflops", "intensity", "gpts"])
        for r in rows:
            wr.writerow([r["kernel"], r["plan"], "", r["seconds"], r["gflops"], r["intensity"],
                         r["gpts"]])
    write_summary(out, {"command": "bench", "passed": True, "rows": len(rows),
                        "seconds": e2e, "gpts": rows[0]["gpts"], "first_run_seconds": first})
    print(f"Forward: device {dev_s:.4f} s ({rows[0]['gpts']:.1f} Gpts/s), "
          f"end to end {e2e:.4f} s ({rows[1]['gpts']:.1f} Gpts/s)")
    plan.close()
    return 0


def cmd_verify(suite, patch, out):
    """sfd.cpp:357-443 (adjoint and taylor suites)."""
    cfg = dict(DEFAULTS)
    cfg.update(patch)
    if suite == "adjoint":
        reports = []
        for dims in ([41, 41], [21, 22, 23]):
            for order in (2, 4, 8):
                reports.append(V.adjoint_test(V.AdjointConfig(interior=dims, space_order=order,
                                                              nt=150)))
        lines = [json.dumps({"suite": "adjoint", **r.__dict__}) for r in reports]
        passed = all(r.passed for r in reports)
    elif suite == "taylor":
        r = V.taylor_test(V.TaylorConfig())
        pts = [p.__dict__ for p in r.points]
        lines = [json.dumps({"suite": "taylor", "phi0": r.phi0, "gdot": r.gdot,
                             "slope0": r.slope0, "slope1": r.slope1, "passed": r.passed,
                             "points": pts}, default=float)]
        passed = r.passed
    else:
        raise ValueError(f"unknown suite '{suite}' (adjoint | taylor)")
    with open(os.path.join(out, "report.jsonl"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    write_summary(out, {"command": "verify", "suite": suite, "passed": passed,
                        "report": os.path.join(out, "report.jsonl")})
    print(f"{suite}: {'PASS' if passed else 'FAIL'}")
    return 0 if passed else 1


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1608_08658_b200",
                                 description="B200 stencil operators (sfd-compatible driver)")
    ap.add_argument("--config", default="")
    ap.add_argument("--set", action="append", default=[])
    ap.add_argument("--out", default="sfd-out")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sub.add_parser("run")
    sub.add_parser("bench")
    v = sub.add_parser("verify")
    v.add_argument("suite", choices=["adjoint", "taylor"])
    args = ap.parse_args(argv)
    os.makedirs(args.out, exist_ok=True)
    try:
        patch = build_patch(args.config, args.set)
        if args.cmd == "run":
            return cmd_run(patch, args.out)
        if args.cmd == "bench":
            return cmd_bench(patch, args.out)
        return cmd_verify(args.suite, patch, args.out)
    except Exception as e:  # sfd.cpp:555-565: refusal -> exit 2 with a summary
        print(f"refused: {e}", file=sys.stderr)
        write_summary(args.out, {"command": "error", "passed": False, "error": str(e)})
        return 2


if __name__ == "__main__":
    sys.exit(main())
