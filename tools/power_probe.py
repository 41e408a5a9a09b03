#!/usr/bin/env python
"""Power / SM clock under sustained load: (a) a device copy at full HBM
bandwidth, (b) the cfg2 forward plan, each for ~N seconds, with nvidia-smi
sampled every 50 ms.  Prints one JSON line per phase."""
import json, os, subprocess, sys, threading, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def sample(stop, out):
    q = "clocks.sm,power.draw,clocks_throttle_reasons.active"
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True).stdout.strip().split(",")
        try:
            out.append((float(r[0]), float(r[1]), int(r[2], 16)))
        except Exception:
            pass
        time.sleep(0.05)


def phase(name, fn, secs):
    import torch
    stop, out = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, out))
    th.start()
    t0 = time.time()
    n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < secs:
        fn()
        n += 1
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    load = out[len(out) // 4:]
    print(json.dumps({"phase": name, "iters": n, "ms_per_iter": e0.elapsed_time(e1) / n,
                      "sm_mhz_median": float(np.median([s[0] for s in load])),
                      "power_w_median": float(np.median([s[1] for s in load])),
                      "power_w_max": max(s[1] for s in load),
                      "capped_frac": sum(1 for s in load if s[2] & 4) / max(1, len(load))}),
          flush=True)


def main():
    import torch
    import bench
    from paper_1608_08658_b200 import _lib as L
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    phase("copy 2 GiB", lambda: [b.copy_(a) for _ in range(10)], secs)
    del a, b
    w = bench.make_workload("cfg2", 200)
    model, src, rec = bench.problem(w)
    argv = [None, L.f64(model.m), L.f64(model.damp), L.i64(src.idx), L.f64(src.w),
            L.f64(w.wavelet), L.i64(rec.idx), L.f64(rec.w), np.empty((w.nt, rec.npoints))]
    plan = L.Plan(L.FORWARD, 3, model.padded, w.space_order, w.nt, w.dt, w.h, src.npoints,
                  rec.npoints, False, 0)
    plan.upload(argv)
    plan.execute()
    torch.cuda.synchronize()
    phase("cfg2 forward, 200 steps/iter", plan.execute, secs)
    print(json.dumps({"cfg": plan.info()}))


if __name__ == "__main__":
    main()
