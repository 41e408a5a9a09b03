#!/usr/bin/env python
"""Generates tests/golden/*.npz by running the UNMODIFIED reference library
(oracle/_ref/libsfdref.so, built from /root/reference/proj/src by
oracle/Makefile) on small seeded problems.  Run in a container that has
/root/reference:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin both the CPU oracle (tests/test_oracle.py) and the B200
backend's host helpers (bit-exact) and operators (rel-L2 gates on the GPU).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
os.environ.setdefault("STENCILFD_CACHE_DIR", "/tmp/stencilfd-cache")

import oracle_lib as O  # noqa: E402


def f32r(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def model_field(shape, seed):
    rng = np.random.default_rng(seed)
    v = 1500.0 + 1500.0 * rng.random(int(np.prod(shape)))
    return f32r(1.0 / v ** 2)


def case_2d():
    interior, h, nbpml, so = [33, 41], 15.0, 10, 4
    mi = model_field(interior, 1)
    src = np.array([[243.7, 40.0]])
    rec = np.array([[100.0, 400.0], [250.0, 401.5], [380.0, 404.9], [0.0, 0.0],
                    [480.0, 600.0]])
    dtc = O.ref_critical_dt(interior, h, nbpml, so, mi)
    nt, dt = 160, 0.85 * dtc
    wav = f32r(O.ref_ricker(18.0, 1.0 / 18.0, nt, dt))
    padded, m, damp = O.ref_model(interior, h, nbpml, so, mi)
    si, sw = O.ref_locate(interior, h, nbpml, so, mi, src)
    ri, rw = O.ref_locate(interior, h, nbpml, so, mi, rec)
    u, r, _ = O.ref_forward(interior, h, nbpml, so, mi, src, wav, rec, nt, dt)
    uh, rh, _ = O.ref_forward(interior, h, nbpml, so, mi, src, wav, rec, nt, dt, save=True)
    rng = np.random.default_rng(7)
    resid = f32r(0.5 * r + 0.05 * np.abs(r).max() * rng.standard_normal(r.shape))
    v, s, _ = O.ref_adjoint(interior, h, nbpml, so, mi, rec, resid, src, nt, dt)
    g, _ = O.ref_gradient(interior, h, nbpml, so, mi, rec, resid, uh, nt, dt)
    np.savez_compressed(os.path.join(HERE, "ref_2d_so4.npz"), interior=interior, h=h,
                        nbpml=nbpml, so=so, m_interior=mi, src_coords=src, rec_coords=rec,
                        nt=nt, dt=dt, wavelet=wav, padded=padded, m=m, damp=damp, src_idx=si,
                        src_w=sw, rec_idx=ri, rec_w=rw, u=u, rec=r, rec_saved=rh,
                        u_hist_tail=uh[nt - 3:], residual=resid, v=v, src_samples=s, grad=g,
                        critical_dt=dtc)


def case_3d():
    interior, h, nbpml, so = [10, 12, 11], 10.0, 3, 8
    mi = model_field(interior, 2)
    src = np.array([[15.0, 55.5, 50.0]])
    rec = np.array([[20.0, 10.0 * j + 3.3, 10.0 * k + 1.7] for j in range(0, 11, 2)
                    for k in range(0, 10, 3)])
    dtc = O.ref_critical_dt(interior, h, nbpml, so, mi)
    nt, dt = 90, 0.9 * dtc
    wav = f32r(O.ref_ricker(25.0, 0.04, nt, dt))
    padded, m, damp = O.ref_model(interior, h, nbpml, so, mi)
    si, sw = O.ref_locate(interior, h, nbpml, so, mi, src)
    ri, rw = O.ref_locate(interior, h, nbpml, so, mi, rec)
    u, r, _ = O.ref_forward(interior, h, nbpml, so, mi, src, wav, rec, nt, dt)
    uh, _, _ = O.ref_forward(interior, h, nbpml, so, mi, src, wav, rec, nt, dt, save=True)
    rng = np.random.default_rng(9)
    resid = f32r(r + 0.1 * np.abs(r).max() * rng.standard_normal(r.shape))
    v, s, _ = O.ref_adjoint(interior, h, nbpml, so, mi, rec, resid, src, nt, dt)
    g, _ = O.ref_gradient(interior, h, nbpml, so, mi, rec, resid, uh, nt, dt)
    np.savez_compressed(os.path.join(HERE, "ref_3d_so8.npz"), interior=interior, h=h,
                        nbpml=nbpml, so=so, m_interior=mi, src_coords=src, rec_coords=rec,
                        nt=nt, dt=dt, wavelet=wav, padded=padded, m=m, damp=damp, src_idx=si,
                        src_w=sw, rec_idx=ri, rec_w=rw, u_last=u[(nt - 1) % 3], rec=r,
                        residual=resid, v_last=v[2 % 3], src_samples=s, grad=g,
                        critical_dt=dtc)


def case_helpers():
    fd = {f"fd2_so{so}": O.ref_fd2(so) for so in range(2, 17, 2)}
    # locate_points edge cases: on-node, mid-cell, the far boundary, random
    interior, h, nbpml, so = [33, 33], 15.0, 10, 4
    mi = np.full(33 * 33, 1.0 / 1500.0 ** 2)
    rng = np.random.default_rng(11)
    pts = np.concatenate([[[60.0, 135.0], [67.5, 142.5], [0.0, 0.0], [480.0, 480.0],
                           [480.0, 0.1]], rng.uniform(0.0, 480.0, size=(200, 2))])
    li, lw = O.ref_locate(interior, h, nbpml, so, mi, pts)
    crit = np.array([O.ref_critical_dt([17, 13], 10.0, 6, o, np.full(17 * 13, 1 / v ** 2))
                     for o in (2, 4, 8, 12, 16) for v in (1500.0, 4500.0)])
    pm, mm, dm = O.ref_model([9, 7], 10.0, 5, 4, 1e-6 * np.arange(1, 64))
    pd, _, dd = O.ref_model([8], 12.5, 8, 4, np.full(8, 1e-7))
    rk = O.ref_ricker(10.0, 0.1, 2001, 1e-4)
    np.savez_compressed(os.path.join(HERE, "ref_helpers.npz"), locate_pts=pts,
                        locate_idx=li, locate_w=lw, crit=crit, model_m=mm, model_damp=dm,
                        model_padded=pm, damp1d=dd, damp1d_padded=pd, ricker=rk, **fd)


if __name__ == "__main__":
    if not O.have_ref():
        raise SystemExit("oracle/_ref/libsfdref.so missing: make -C oracle ref")
    case_helpers()
    case_2d()
    case_3d()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
