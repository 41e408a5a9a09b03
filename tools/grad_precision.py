"""Where the fp32 imaging condition loses precision (Gradient).

A 2-D second-order damped acoustic toy (numpy, no GPU) run in fp64 and fp32,
accumulating grad += u * v_tt with v_tt formed two ways:
  A  v_tt = inc - d                (what the kernels compute; inc = c1 d + c2 lap)
  B  v_tt = (c1 - 1) d + c2 lap    (no cancellation between inc and d)
Both give the same fp32 error against fp64 (2.54e-5 rel-L2 here): the floor is
the rounding of the fp32 wavefield rows themselves, whose fresh per-step error
reaches v_tt at full size while v_tt is (omega dt)^2 smaller than v, not the
subtraction.  Run: python tools/grad_precision.py"""
import numpy as np


def run(f, form, n=80, nt=200, cfl=0.5):
    v = np.zeros((n, n), f)
    vp = np.zeros((n, n), f)
    g = np.zeros((n, n))
    c2 = f(cfl ** 2) * np.ones((n, n), f)
    e = np.zeros((n, n))
    for i in range(8):
        w = 0.05 * (8 - i) / 8
        e[i, :] += w
        e[-1 - i, :] += w
        e[:, i] += w
        e[:, -1 - i] += w
    c1 = (f(1) - e.astype(f) * c2).astype(f)
    f0 = 0.05 / 4
    t = np.arange(nt)
    arg = (np.pi * f0 * (t - 1.2 / f0)) ** 2
    wav = (1 - 2 * arg) * np.exp(-arg)
    u = np.random.default_rng(0).standard_normal((nt, n, n))
    for it in range(nt):
        lap = np.zeros((n, n), f)
        lap[1:-1, 1:-1] = ((v[:-2, 1:-1] + v[2:, 1:-1]) + (v[1:-1, :-2] + v[1:-1, 2:])
                           + f(-4) * v[1:-1, 1:-1])
        d = (v - vp).astype(f)
        inc = (c1 * d + c2 * lap).astype(f)
        vtt = (inc - d) if form == "A" else ((c1 - f(1)) * d + c2 * lap)
        g += u[it] * vtt.astype(f)
        vn = (v + inc).astype(f)
        vn[n // 2, n // 2] += f(wav[it])
        vp, v = v, vn
    return g


if __name__ == "__main__":
    g64 = run(np.float64, "A")
    for form in "AB":
        g = run(np.float32, form)
        print(form, np.linalg.norm(g - g64) / np.linalg.norm(g64))
