// The 3-D sweep kernel template (see kernels.cu for the overview).  Included
// by the per-radius translation units sweep3d_r<R>.cu so the eight radii
// compile in parallel.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <initializer_list>
#include <mutex>
#include <string>
#include <utility>

#include "kernels.cuh"

#ifndef SFDB200_PROBE
#define SFDB200_PROBE 0
#endif

namespace sfdb200 {
namespace detail {

// ---------------------------------------------------------------- PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void named_barrier_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// bar.red.or over the named barrier `id` (`threads` threads): returns, in every
// participating thread, whether any of them passed pred = true.
__device__ __forceinline__ bool named_barrier_or(int id, int threads, bool pred) {
    unsigned int r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\t"
        "barrier.cta.red.or.pred q, %2, %3, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
        : "=r"(r)
        : "r"(static_cast<unsigned int>(pred)), "r"(id), "r"(threads)
        : "memory");
    return r != 0;
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// try_wait with a suspend-time hint: a thread whose phase is not complete
// sleeps until it completes (or the hint, in ns, elapses) instead of spinning
// through the issue slots the other warps of its SM sub-partition need.
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Waits for the stage barrier's phase; a transaction count that can never
// complete (a bug) traps after 20 s instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const uint64_t t0 = global_ns();
    while (!mbar_try_wait(bar, parity))
        if (global_ns() - t0 > 20000000000ull) __trap();
}

// Programmatic dependent launch: the next sweep may be scheduled once every
// CTA of this one has started; it sets up its barriers and tables, then waits
// here until this grid has completed and its stores are visible.
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar))
        : "memory");
}

// Stage layout: [u1 halo box][u1 centre R planes ahead][u2][c2][c1][ut][grad]
// (c1 only without SEP; ut, grad only with GRAD).  SEP (separable damping,
// c1 formed in registers) drops the c1 box and reserves 32 floats for the
// producer's -ez[z] instead.
template <int R, int BY, int NY, bool GRAD, bool SEP = false>
struct Tile {
    static constexpr int TX = 32;
    static constexpr int HALF = BY * NY;  // rows per tile half
    static constexpr int TY = 2 * HALF;
    // TMA box starts must be 16-byte aligned in x: tiles start at multiples of
    // 32 columns and the x halo is widened to RA = roundup(R, 4).
    static constexpr int RA = (R + 3) & ~3;
    static constexpr int BW = TX + 2 * RA;                     // halo row pitch
    static constexpr int HF = ((TY + 2 * R) * BW + 31) & ~31;  // halo floats, 128 B multiple
    static constexpr int CF = TY * TX;                         // centre box floats
    static constexpr int NC = (GRAD ? 6 : 4) - (SEP ? 1 : 0);  // centre boxes per stage
    static constexpr int O_U1C = HF, O_U2 = HF + CF, O_C2 = HF + 2 * CF, O_C1 = HF + 3 * CF;
    static constexpr int O_UT = HF + (SEP ? 3 : 4) * CF, O_GR = O_UT + CF;
    static constexpr int O_NEZ = HF + NC * CF;                 // SEP: -ez[z]
    static constexpr int SF = HF + NC * CF + (SEP ? 32 : 0);   // floats per stage
    // Bytes the TMA boxes of one stage deliver (the mbarrier transaction count).
    static constexpr uint32_t BYTES = static_cast<uint32_t>((TY + 2 * R) * BW + NC * CF) * 4u;
    static constexpr int Q = 2 * R + 1;                        // z-queue length
};

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

template <int V>
struct IC {
    static constexpr int value = V;
};

// ---------------------------------------------------------------- 3-D sweep
//
// Thread (lx, wy) owns column x = x0 + lx and NY rows in EACH half of the
// tile: rows ly0 + j (top) and HALF + ly0 + j (bottom), j < NY.  Every value
// is a float2 {top, bottom}, so the whole update runs on the packed fp32x2
// pipe (FADD2/FFMA2/FMUL2, sm_100): per k and per point pair, 5 FADD2 for the
// six neighbours and 2 FFMA2 for
//     lap += w_k * ((sum of the 2*ndim neighbours at distance k) - 2*ndim*u0)
// (the centred per-k form keeps the fp32 error ~1e-6).  The z
// neighbours live in a register queue of Q = 2R+1 planes; with ROT the z loop
// is unrolled by Q so the queue rotates by renaming (no moves).
//
// Warp-specialised: warp BY of the CTA is the TMA producer; the BY consumer
// warps never wait on each other.  Stage s has a "full" mbarrier (TMA
// transaction bytes) and an "empty" one (one arrival per consumer warp once
// it is done reading the stage), so no CTA-wide barrier runs per plane.

// The fused sparse work, once per CTA and out of the plane loop (so the loop
// carries no calls and no sparse state).  `a` lives in the kernel's parameter
// space (__grid_constant__), so passing it by reference copies nothing.
//
// Samples of the previous step's row (this launch's u1): this CTA's even share
// of the receivers, read from global memory (the row is complete once the
// launch has passed griddepcontrol.wait), summed c = 0..7 left to right.
template <int NT>
__device__ __noinline__ void sample_cta(const SweepArgs& a, long long py, long long pz, int cta,
                                        int nctas, int tid) {
    const int per = (a.smp_n + nctas - 1) / nctas;
    const int e0 = cta * per, e1 = min(e0 + per, a.smp_n);
    for (int e = e0 + tid; e < e1; e += NT) {
        const long long b0 = __ldg(a.smp_base + e);
        if (!SFDB_CHECK(a.dbg, b0 >= 0 && b0 + pz + py + 1 < a.slot, kDbgSample)) continue;
        const float* u = a.u1 + b0;
        const float4 wl = __ldg(reinterpret_cast<const float4*>(a.smp_w) + 2 * e);
        const float4 wh = __ldg(reinterpret_cast<const float4*>(a.smp_w) + 2 * e + 1);
        const float* v = u + pz;
        float acc = wl.x * u[0];
        acc = fmaf(wl.y, u[1], acc);
        acc = fmaf(wl.z, u[py], acc);
        acc = fmaf(wl.w, u[py + 1], acc);
        acc = fmaf(wh.x, v[0], acc);
        acc = fmaf(wh.y, v[1], acc);
        acc = fmaf(wh.z, v[py], acc);
        acc = fmaf(wh.w, v[py + 1], acc);
        a.smp_row[__ldg(a.smp_pt + e)] = acc;
    }
}

// Injections into the corners this CTA stored, after all its planes.
// (debug build: the corner must lie in the box [x0, x0+32) x [y0, y0+ty) x
// [zb, ze) the injecting item stored -- an atomic into a cell another CTA
// stores in the same launch would race with that store)
template <bool GRAD, int NT>
__device__ __noinline__ void inject_cta(const SweepArgs& a, int cta, int tid, int x0 = 0,
                                        int y0 = 0, int zb = 0, int ze = 0, int ty = 0,
                                        long long py = 1, long long pz = 1) {
    const int r0 = __ldg(a.inj_tab + cta), r1 = __ldg(a.inj_tab + cta + 1);
    // One thread per run: the entries of one cell, adjacent and in the
    // reference's (p, c) order (sparse.cpp).  The run is summed in that order
    // and added once, so colliding corners (a receiver carpet at the grid
    // spacing) give the same bits on every run.
    for (int r = r0 + tid; r < r1; r += NT) {
        const int e = __ldg(a.inj_run + r), e1 = __ldg(a.inj_run + r + 1);
        const long long o = __ldg(a.inj_off + e);
        if (!SFDB_CHECK(a.dbg, o >= 0 && o < a.slot, kDbgInject)) continue;
#ifdef SFDB200_DEBUG
        if (ty > 0) {
            const long long cz = o / pz, cy = (o - cz * pz) / py, cx = o - cz * pz - cy * py;
            if (!SFDB_CHECK(a.dbg,
                            cz >= zb && cz < ze && cy >= y0 && cy < y0 + ty && cx >= x0 &&
                                cx < x0 + 32,
                            kDbgInjectOwner))
                continue;
        }
#endif
        float delta = __ldg(a.inj_coef + e) * __ldg(a.inj_row + __ldg(a.inj_pt + e));
        for (int f = e + 1; f < e1; ++f)
            delta += __ldg(a.inj_coef + f) * __ldg(a.inj_row + __ldg(a.inj_pt + f));
        atomicAdd(a.out + o, delta);
        if constexpr (GRAD)
            if (a.inj_gm[e]) atomicAdd(a.grad + o, a.nidt2 * __ldg(a.ut + o) * delta);
    }
}

template <int R, int BY, int NY, int S, bool GRAD, bool ROT>
__global__ void __launch_bounds__(32 * (BY + 1), 4)
    sweep3d_kernel(const __grid_constant__ CUtensorMap tm_uh,
                   const __grid_constant__ CUtensorMap tm_uc,
                   const __grid_constant__ CUtensorMap tm_c1,
                   const __grid_constant__ CUtensorMap tm_c2,
                   const __grid_constant__ CUtensorMap tm_ut,
                   const __grid_constant__ CUtensorMap tm_gr,
                   const __grid_constant__ SweepArgs a, const int Px,
                   const int Py, const long long py, const long long pz) {
    using T = Tile<R, BY, NY, GRAD>;
    constexpr int Q = T::Q;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* smem = reinterpret_cast<float*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * T::SF);
    uint64_t* empty = full + S;
    constexpr int NT = 32 * BY;  // consumer threads

    const int lx = threadIdx.x;
    const int ly0 = threadIdx.y * NY;
    const int tid = threadIdx.y * 32 + lx;
    const int x0 = blockIdx.x * T::TX;
    const int y0 = R + blockIdx.y * T::TY;
    const int zb = a.zlo + blockIdx.z * a.zchunk;
    const int ze = min(zb + a.zchunk, a.zhi);
    if (zb >= ze) return;
    const int n = ze - zb;
    const int x = x0 + lx;

    // Separable damping: the producer also stages -ez[z] in the (then unused)
    // c1 slot of the stage, ordered before the consumers' acquire by the
    // release of its arrive.
    auto issue = [&](int stage, int z, float nez) {
        float* sb = smem + stage * T::SF;
        uint64_t* bar = &full[stage];
        const bool sep = a.ez != nullptr;  // c1 formed from the damping profiles
        if (sep) sb[T::O_C1] = nez;
        mbar_arrive_expect_tx(bar, sep ? T::BYTES - 4u * T::CF : T::BYTES);
        tma_load_4d(sb, &tm_uh, x0 - T::RA, y0 - R, z, a.row_u1, bar);
        tma_load_4d(sb + T::O_U1C, &tm_uc, x0, y0, z + R, a.row_u1, bar);
        tma_load_4d(sb + T::O_U2, &tm_uc, x0, y0, z, a.row_u2, bar);
        if (!sep) tma_load_4d(sb + T::O_C1, &tm_c1, x0, y0, z, 0, bar);
        tma_load_4d(sb + T::O_C2, &tm_c2, x0, y0, z, 0, bar);
        if constexpr (GRAD) {
            tma_load_4d(sb + T::O_UT, &tm_ut, x0, y0, z, a.row_ut, bar);
            tma_load_4d(sb + T::O_GR, &tm_gr, x0, y0, z, 0, bar);
        }
    };

    pdl_trigger();
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], BY);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.y == BY) {  // producer warp: one lane streams the planes
        pdl_wait();
        if (lx == 0) {
            const float* ez = a.ez ? a.ez + zb : nullptr;
            float nxt = ez ? -__ldg(ez) : 0.0f;
            for (int j = 0; j < n; ++j) {
                const int st = j % S;
                const float cur = nxt;
                if (ez && j + 1 < n) nxt = -__ldg(ez + j + 1);
                if (j >= S) mbar_wait(&empty[st], static_cast<uint32_t>((j / S - 1) & 1));
                issue(st, zb + j, cur);
            }
        }
        return;
    }

    const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    // Everything below reads or writes rows the previous sweep touches.
    pdl_wait();
    if (a.smp_base) sample_cta<NT>(a, py, pz, cta, gridDim.x * gridDim.y * gridDim.z, tid);

    // Queue slot of plane zb - R + t is t mod Q.
    // Rows inside the allocation.  Halo and pad cells of a row are stored too:
    // their coefficients are zero and their u1, u2 are zero, so the update
    // writes back exactly 0 (kernels.cu coeffs_kernel).
    float2 q[NY][Q];
    bool va[NY], vb[NY];
#pragma unroll
    for (int j = 0; j < NY; ++j) {
        const int ya_ = y0 + ly0 + j, yb_ = ya_ + T::HALF;
        va[j] = ya_ < Py;
        vb[j] = yb_ < Py;
        const float* ca = a.u1 + static_cast<long long>(ya_) * py + x;
        const float* cb = a.u1 + static_cast<long long>(yb_) * py + x;
#pragma unroll
        for (int t = 0; t < 2 * R; ++t) {
            const long long o = static_cast<long long>(zb - R + t) * pz;
            q[j][t] = f2(va[j] ? __ldg(ca + o) : 0.0f, vb[j] ? __ldg(cb + o) : 0.0f);
        }
    }

    const float2 neg2nd = f2(a.neg2nd, a.neg2nd);
    const float2 mone = f2(-1.0f, -1.0f);
    float2 wk[R + 1];
#pragma unroll
    for (int k = 0; k <= R; ++k) wk[k] = f2(a.w[k], a.w[k]);
    const float2 nidt2 = f2(a.nidt2, a.nidt2);
    // Separable damping: -max(ey[y], ex[x]) of this thread's points (fixed along z).
    const bool sep = a.ez != nullptr;
    float2 nexy[NY];
#pragma unroll
    for (int j = 0; j < NY; ++j) {
        const int ya_ = y0 + ly0 + j, yb_ = ya_ + T::HALF;
        const float exv = sep && x < Px ? __ldg(a.ex + x) : 0.0f;
        nexy[j] = f2(-fmaxf(sep && ya_ < Py ? __ldg(a.ey + ya_) : 0.0f, exv),
                     -fmaxf(sep && yb_ < Py ? __ldg(a.ey + yb_) : 0.0f, exv));
    }

    // Store cursor: byte address of (plane zb + i, row y0 + ly0, column x) in
    // the output row, advanced one plane per iteration; the other rows and
    // the gradient field are fixed byte offsets from it.
    char* cur = reinterpret_cast<char*>(a.out + static_cast<long long>(zb) * pz +
                                        static_cast<long long>(y0 + ly0) * py + x);
    const long long rowb = py * 4, halfb = T::HALF * py * 4, planeb = pz * 4;
    const long long gdiff = GRAD ? reinterpret_cast<char*>(a.grad) - reinterpret_cast<char*>(a.out) : 0;

    int stage = 0;        // pipeline stage of the current plane
    uint32_t phase = 0;   // its full-barrier parity

    // One z plane.  PH is the compile-time phase of plane i within the queue
    // rotation (always 0 without ROT, where the queue is shifted instead).
    auto plane = [&](auto ph_c, const int i) {
        constexpr int PH = decltype(ph_c)::value;
        auto slot = [](int off) { return ((PH + off + R) % Q + Q) % Q; };
        const int st = stage;
        mbar_wait(&full[st], phase);
        const float* H = smem + st * T::SF;
        const float* Cq = H + T::O_U1C;
        const float* U2 = H + T::O_U2;
        const float* C1 = H + T::O_C1;
        const float* C2 = H + T::O_C2;
        const float* UT = H + T::O_UT;
        const float* GR = H + T::O_GR;  // the gradient plane, staged like the rest
        const int ca = ly0 * T::TX + lx, cb = ca + T::HALF * T::TX;

#pragma unroll
        for (int j = 0; j < NY; ++j)
            q[j][slot(R)] = f2(Cq[ca + j * T::TX], Cq[cb + j * T::TX]);

        // y neighbours outside this thread's NY rows (both halves).
        float2 ya[R], yb[R];
        const float* hA = H + ly0 * T::BW + lx + T::RA;   // smem row ly0 <-> tile row ly0 - R
        const float* hB = hA + T::HALF * T::BW;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            ya[k] = f2(hA[k * T::BW], hB[k * T::BW]);
            yb[k] = f2(hA[(NY + R + k) * T::BW], hB[(NY + R + k) * T::BW]);
        }
        const float nez = sep ? C1[0] : 0.0f;  // -ez[z], staged by the producer

#pragma unroll
        for (int j = 0; j < NY; ++j) {
            const float2 c0 = q[j][slot(0)];
            const float* ra = hA + (j + R) * T::BW;
            const float* rb = hB + (j + R) * T::BW;
            float2 lap = f2(0.0f, 0.0f);
#pragma unroll
            for (int k = 1; k <= R; ++k) {
                const int rm = j + R - k, rp = j + R + k;  // smem rows of the y neighbours
                const float2 ym = rm < R ? ya[rm] : (rm < R + NY ? q[rm - R][slot(0)] : yb[rm - R - NY]);
                const float2 yp = rp < R ? ya[rp] : (rp < R + NY ? q[rp - R][slot(0)] : yb[rp - R - NY]);
                const float2 xs = add2(f2(ra[-k], rb[-k]), f2(ra[k], rb[k]));
                const float2 zs = add2(q[j][slot(-k)], q[j][slot(k)]);
                float2 sk = add2(add2(xs, add2(ym, yp)), zs);
                sk = fma2(neg2nd, c0, sk);
                lap = fma2(wk[k], sk, lap);
            }
            const int ia = ca + j * T::TX, ib = cb + j * T::TX;
            const float2 d = fma2(f2(U2[ia], U2[ib]), mone, c0);           // c0 - u2, exact form
            const float2 c2v = f2(C2[ia], C2[ib]);
            // c1 = 1 - e c2, e = damp/dt (separable) or the streamed c1 field
            const float2 c1v = sep ? fma2(f2(fminf(nez, nexy[j].x), fminf(nez, nexy[j].y)), c2v,
                                          f2(1.0f, 1.0f))
                                   : f2(C1[ia], C1[ib]);
            const float2 inc = fma2(c1v, d, mul2(c2v, lap));
            const float2 o = add2(c0, inc);
            char* pa = cur + j * rowb;
            char* pb = pa + halfb;
            if (va[j]) *reinterpret_cast<float*>(pa) = o.x;
            if (vb[j]) *reinterpret_cast<float*>(pb) = o.y;
            if constexpr (GRAD) {
                // grad += -(1/dt^2) u_t (v_t - 2 v_{t+1} + v_{t+2}) = nidt2 * u_t * (inc - d)
                const float2 vtt = fma2(d, mone, inc);
                const float2 coef = mul2(nidt2, f2(UT[ia], UT[ib]));
                if (va[j]) *reinterpret_cast<float*>(pa + gdiff) = fmaf(coef.x, vtt.x, GR[ia]);
                if (vb[j]) *reinterpret_cast<float*>(pb + gdiff) = fmaf(coef.y, vtt.y, GR[ib]);
            }
        }

        cur += planeb;
        if constexpr (!ROT) {
#pragma unroll
            for (int j = 0; j < NY; ++j)
#pragma unroll
                for (int t = 0; t < 2 * R; ++t) q[j][t] = q[j][t + 1];
        }
        // Release the stage to the producer (one arrival per consumer warp).
        __syncwarp();
        if (lx == 0) mbar_arrive(&empty[st]);
        if (++stage == S) {
            stage = 0;
            phase ^= 1u;
        }
    };

    if constexpr (ROT) {
        for (int base = 0; base < n; base += Q) {
            [&]<int... P>(std::integer_sequence<int, P...>) {
                ((base + P < n ? (plane(IC<P>{}, base + P), true) : false) && ...);
            }(std::make_integer_sequence<int, Q>{});
        }
    } else {
        for (int i = 0; i < n; ++i) plane(IC<0>{}, i);
    }
    // Fused Inject once every consumer warp has stored its planes (named
    // barrier over the consumer warps only).
    if (a.inj_tab) {
        named_barrier_sync(1, NT);
        inject_cta<GRAD, NT>(a, cta, tid, x0, y0, zb, ze, T::TY, py, pz);
    }
}

// ---------------------------------------------------------------- pair mapping
//
// Same tile, TMA pipeline, fused sparse work and numerics as sweep3d_kernel,
// but thread (px, gy) of warp wy owns the column PAIR x, x+1 (x = x0 + 2 px)
// in NY consecutive rows r0 + j, r0 = (2 wy + gy) NY.  The float2 lanes are
// the two columns, so every shared-memory read is an 8-byte LDS.64 (a
// half-warp reads 128 contiguous bytes: conflict-free) and one x window of
// 2R + 2 floats per row serves both points: per updated point the kernel
// reads (2R + 2)/2 + 2R/NY + 4 floats of shared memory instead of
// 2R + 2R/NY + 4, which is what bounds high space orders.  Odd
// x offsets straddle two loaded pairs; the compiler pairs them with moves.
__device__ __forceinline__ float2 ld2(const float* p) {
    return *reinterpret_cast<const float2*>(p);
}
__device__ __forceinline__ void st2(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }

// Unrolling of the z loop, z_unroll(R, ROTV): cfg.rot 1 = by Q (the queue
// rotates by renaming), 0 = none (the queue shifts by one plane per plane),
// k >= 2 = by k (the queue shifts by k planes every k planes).
template <int R, int ROTV>
constexpr int z_unroll() { return ROTV == 1 ? 2 * R + 1 : (ROTV == 0 ? 1 : ROTV); }

// Items: CTA c runs the (x tile, y tile, z chunk) items c, c + gridDim.x, ...
// (item = x tile fastest, then y tile, then z chunk: the hardware's own CTA
// order, so tiles sweep z in step and halos stay in L2).  By default the grid
// has one CTA per item; with fewer (persistent) CTAs the producer streams the
// next item's planes while the consumers finish the current one, so the ring
// never drains between items (measured: on cfg2 no faster than the hardware
// handing items to free slots, and slower whenever items per CTA are not
// integral, so it is a tuning / test option).  With UN a multiple of S each
// item's first plane is aligned to stage 0 by empty "skip" stages, so every
// unrolled plane phase has a fixed stage and compile-time shared-memory offsets.
template <int R, int BY, int NY, int S, bool GRAD, int MINB, int UN, bool SEP>
__global__ void __launch_bounds__(32 * (BY + 1), MINB)
    sweep3d_pair_kernel(const __grid_constant__ CUtensorMap tm_uh,
                        const __grid_constant__ CUtensorMap tm_uc,
                        const __grid_constant__ CUtensorMap tm_c1,
                        const __grid_constant__ CUtensorMap tm_c2,
                        const __grid_constant__ CUtensorMap tm_ut,
                        const __grid_constant__ CUtensorMap tm_gr,
                        const __grid_constant__ SweepArgs a, const int Px, const int Py,
                        const long long py, const long long pz, const int ntx, const int nty,
                        const int nitems) {
    using T = Tile<R, BY, NY, GRAD, SEP>;
    constexpr int Q = T::Q;
    constexpr int WL = (R + 1) & ~1;  // x window [x - WL, x + 1 + WL], 8-byte aligned
    const bool dyn = SEP && a.item_ctr != nullptr;  // dynamic persistent mode
    constexpr bool SST = UN % S == 0;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* smem = reinterpret_cast<float*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * T::SF);
    uint64_t* empty = full + S;
    constexpr int NT = 32 * BY;

    const int lx = threadIdx.x;
    const int tid = threadIdx.y * 32 + lx;
    // item -> tile origin (x0, y0), z range [zb, ze) and direction: planes
    // z0, z0 + dz, ... (dz = -1: the chunk streams downward, a.zdown).  The
    // first a.nbi items are the P2P boundary tiles (SweepArgs::nbi); their side
    // is returned in bs (-1 for interior items).
    // `tab` is the item's index in the fused sparse tables (sparse.cpp owner_of:
    // boundary items first, then tile + tiles * chunk) -- NOT the launch
    // position when the grouped order renumbers the interior items.
    auto decode = [&](int item, int& x0, int& y0, int& zb, int& ze, int& z0, int& dz, int& bs,
                      int& tab) {
        bs = -1;
        int tz = 0;
        tab = item;
        if (item < a.nbi) {
            const int tiles = ntx * nty, grp = item / tiles;
            bs = a.bside[grp];
            item -= grp * tiles;
        } else {
            item -= a.nbi;
        }
        const int tiles = ntx * nty;
        if (bs < 0 && a.group > 0) {  // grouped order (SweepArgs::group)
            const int zc = (nitems - a.nbi) / tiles;
            const int g = item / (a.group * zc);
            const int base = g * a.group;
            const int gn = min(a.group, tiles - base);
            const int rem = item - base * zc;
            tz = rem / gn;
            item = base + (rem - tz * gn) + tz * tiles;  // back to tile-major numbering
            tab = a.nbi + item;
        }
        const int r = item / ntx;
        x0 = (item - r * ntx) * T::TX;
        if (bs < 0) tz = r / nty;
        y0 = R + (r - tz * nty) * T::TY;
        if (bs >= 0) {
            zb = a.bz[bs];
            ze = zb + a.blen;
        } else {
            zb = a.zlo + tz * a.zchunk;
            ze = min(zb + a.zchunk, a.zhi);
        }
        const bool dn = bs < 0 && tz < 64 && ((a.zdown >> tz) & 1ull);
        z0 = dn ? ze - 1 : zb;
        dz = dn ? -1 : 1;
    };

    pdl_trigger();
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], BY);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.y == BY) {  // producer warp: one lane streams every item's stages
        pdl_wait();
        if (lx == 0) {
            uint32_t j = 0;  // stage sequence number across items
            auto acquire = [&]() {
                const int st = static_cast<int>(j % S);
                if (j >= S) mbar_wait(&empty[st], ((j / S) - 1) & 1);
                return st;
            };
            // Dynamic mode: items from the counter, each item's index staged
            // with its first plane; the last fetch of the launch resets it.
            auto fetch = [&]() -> int {
                const unsigned long long v = atomicAdd(a.item_ctr, 1ull);
                if (v + 1 == static_cast<unsigned long long>(nitems) + gridDim.x)
                    atomicExch(a.item_ctr, 0ull);
                return v < static_cast<unsigned long long>(nitems) ? static_cast<int>(v) : nitems;
            };
            auto align = [&]() {
                if constexpr (SST) {
                    while (j % S != 0) {  // skip stage: completes on the arrive alone
                        mbar_arrive(&full[acquire()]);
                        ++j;
                    }
                }
            };
            for (int item = dyn ? fetch() : blockIdx.x; item < nitems;
                 item = dyn ? fetch() : item + gridDim.x) {
                int x0, y0, zb, ze, z0, dz, bs, tab;
                decode(item, x0, y0, zb, ze, z0, dz, bs, tab);
                const int n = ze - zb;
                if (n <= 0) continue;
                align();
                const float* ezp = SEP ? a.ez + z0 : nullptr;
                float nxt = 0.0f;
                if constexpr (SEP) nxt = -__ldg(ezp);
#pragma unroll 1
                for (int i = 0; i < n; ++i) {
                    const float cur = nxt;
                    if constexpr (SEP)
                        if (i + 1 < n) nxt = -__ldg(ezp + dz * (i + 1));
                    const int st = acquire();
                    float* sb = smem + st * T::SF;
                    uint64_t* bar = &full[st];
                    const int z = z0 + dz * i;
                    {
                        const long long planes = a.slot / pz;
                        SFDB_CHECK(a.dbg, z >= 0 && z < planes && z + dz * R >= 0 &&
                                              z + dz * R < planes,
                                   kDbgTmaPlane);
                    }
                    // SEP: -ez[z] (and in dynamic mode the item index, with the
                    // item's first plane) ride in the stage, ordered before the
                    // consumers' acquire by the release of this arrive.
                    if constexpr (SEP) {
                        sb[T::O_NEZ] = cur;
                        if (dyn && i == 0) sb[T::O_NEZ + 1] = __int_as_float(item);
                    }
                    mbar_arrive_expect_tx(bar, T::BYTES);
                    tma_load_4d(sb, &tm_uh, x0 - T::RA, y0 - R, z, a.row_u1, bar);
                    tma_load_4d(sb + T::O_U1C, &tm_uc, x0, y0, z + dz * R, a.row_u1, bar);
                    tma_load_4d(sb + T::O_U2, &tm_uc, x0, y0, z, a.row_u2, bar);
                    if constexpr (!SEP) tma_load_4d(sb + T::O_C1, &tm_c1, x0, y0, z, 0, bar);
                    tma_load_4d(sb + T::O_C2, &tm_c2, x0, y0, z, 0, bar);
                    if constexpr (GRAD) {
                        tma_load_4d(sb + T::O_UT, &tm_ut, x0, y0, z, a.row_ut, bar);
                        tma_load_4d(sb + T::O_GR, &tm_gr, x0, y0, z, 0, bar);
                    }
                    ++j;
                }
            }
            if (dyn) {  // end of work: a stage holding index -1, no transfer
                align();
                const int st = acquire();
                smem[st * T::SF + T::O_NEZ + 1] = __int_as_float(-1);
                mbar_arrive(&full[st]);
                ++j;
            }
        }
        return;
    }

    pdl_wait();
    if (a.smp_base) sample_cta<NT>(a, py, pz, blockIdx.x, gridDim.x, tid);

    const int px = lx & 15, gy = lx >> 4;
    const int r0 = (threadIdx.y * 2 + gy) * NY;  // first tile row of this thread
    const int cidx = r0 * T::TX + 2 * px;
    constexpr bool ROT = UN == Q;
    constexpr int QS = ROT ? Q : Q + UN - 1;  // queue slots
    const float2 neg2nd = f2(a.neg2nd, a.neg2nd);
    const float2 mone = f2(-1.0f, -1.0f);
    float2 wk[R + 1];
#pragma unroll
    for (int k = 0; k <= R; ++k) wk[k] = f2(a.w[k], a.w[k]);
    const float2 nidt2 = f2(a.nidt2, a.nidt2);
    const long long rowb = py * 4, planeb = pz * 4;
    const long long gdiff = GRAD ? reinterpret_cast<char*>(a.grad) - reinterpret_cast<char*>(a.out) : 0;
    uint32_t j = 0;  // stage sequence number, as the producer's

    auto align = [&]() {
        if constexpr (SST) {
            while (j % S != 0) {
                const int st = static_cast<int>(j % S);
                mbar_wait(&full[st], (j / S) & 1);
                __syncwarp();
                if (lx == 0) mbar_arrive(&empty[st]);
                ++j;
            }
        }
    };
    for (int item = blockIdx.x;; item += gridDim.x) {
        if (dyn) {  // the next item's index rides in its first stage
            align();
            const int st = static_cast<int>(j % S);
            mbar_wait(&full[st], (j / S) & 1);
            item = __float_as_int(smem[st * T::SF + T::O_NEZ + 1]);
            if (item < 0) break;
        } else if (item >= nitems) {
            break;
        }
        int x0, y0, zb, ze, z0, dz, bs, tab;
        decode(item, x0, y0, zb, ze, z0, dz, bs, tab);
        const int n = ze - zb;
        if (n <= 0) continue;
        align();
        const int x = x0 + 2 * px;
        // Queue slot of plane z0 + dz (t - R) is t (t < 2R), loaded directly
        // (the loads overlap the producer filling the ring with the item's
        // first planes; staging them through the ring delays those planes).
        // Streaming down mirrors the queue; the per-k sums q[-k] + q[+k] are
        // commutative, so both directions give the same bits.
        float2 q[NY][QS];
#pragma unroll
        for (int jj = 0; jj < NY; ++jj) {
            const int y = y0 + r0 + jj;
            const float* c = a.u1 + static_cast<long long>(y) * py + x;
#pragma unroll
            for (int t = 0; t < 2 * R; ++t) {
                const long long o = static_cast<long long>(z0 + dz * (t - R)) * pz;
                const bool in = SFDB_CHECK(
                    a.dbg, y >= Py || (c + o >= a.u1 && c + o + 2 <= a.u1 + a.slot), kDbgQueue);
                q[jj][t] = y < Py && in ? __ldg(reinterpret_cast<const float2*>(c + o))
                                        : f2(0.0f, 0.0f);
            }
        }
        // Store only the 32-byte sectors that hold updated cells (whole sectors:
        // a partial one costs L2 a DRAM fill).  The halo / pitch cells left out
        // are zeroed once and stay zero: their coefficients are zero and no
        // sparse corner lies there.
        bool vy[NY];
        float2 nexy[NY];  // SEP: -max(ey[y], ex[x]) of this thread's points (fixed along z)
#pragma unroll
        for (int jj = 0; jj < NY; ++jj) {
            const int y = y0 + r0 + jj;
            vy[jj] = y < Py - R && (x & ~7) + 8 > R && (x & ~7) < Px - R;
            const float eyv = SEP && y < Py ? __ldg(a.ey + y) : 0.0f;
            nexy[jj] = f2(-fmaxf(eyv, SEP && x < Px ? __ldg(a.ex + x) : 0.0f),
                          -fmaxf(eyv, SEP && x + 1 < Px ? __ldg(a.ex + x + 1) : 0.0f));
        }
        char* cur = reinterpret_cast<char*>(a.out + static_cast<long long>(z0) * pz +
                                            static_cast<long long>(y0 + r0) * py + x);

        int stage = static_cast<int>(j % S);  // 0 with SST
        uint32_t phase = (j / S) & 1;
        auto plane = [&](auto ph_c, const int i) {
            constexpr int PH = decltype(ph_c)::value;
            auto slot = [](int off) { return ROT ? ((PH + off + R) % Q + Q) % Q : PH + R + off; };
            const int st = SST ? PH % S : stage;
            mbar_wait(&full[st], phase);
            const float* H = smem + st * T::SF;
            const float* Cq = H + T::O_U1C;
            const float* U2 = H + T::O_U2;
            const float* C1 = H + T::O_C1;
            const float* C2 = H + T::O_C2;
            const float* UT = H + T::O_UT;
            const float* GR = H + T::O_GR;
#pragma unroll
            for (int jj = 0; jj < NY; ++jj) q[jj][slot(R)] = ld2(Cq + cidx + jj * T::TX);

            const float* hp = H + (r0 + R) * T::BW + T::RA + 2 * px;  // (row r0, column x)
            const float nez = SEP ? H[T::O_NEZ] : 0.0f;  // -ez[z], staged by the producer
            // x windows of every row, then the k loop outermost: the y
            // neighbours outside this thread's rows (yu[m] = row r0 - 1 - m,
            // yd[m] = row r0 + NY + m) are loaded at k = m + 1 and stay live for
            // NY iterations only, instead of all 2R of them for the whole plane.
            // SFDB200_PROBE (experiments only, tools/build_probe.sh; wrong results):
            // 1 = no x / y shared-memory reads, 2 = no y reads, 3 = no x reads.
            constexpr bool PX = SFDB200_PROBE == 0 || SFDB200_PROBE == 2;
            constexpr bool PY = SFDB200_PROBE == 0 || SFDB200_PROBE == 3;
            float w[NY][2 * WL + 2];
#pragma unroll
            for (int jj = 0; jj < NY; ++jj)
#pragma unroll
                for (int m = 0; m <= WL; ++m) {
                    const float2 v = PX ? ld2(hp + jj * T::BW - WL + 2 * m) : f2(0.0f, 0.0f);
                    w[jj][2 * m] = v.x;
                    w[jj][2 * m + 1] = v.y;
                }
            float2 yu[R], yd[R];
            // Two partial sums (odd / even k) halve the dependent FFMA2 chain.
            float2 lap[NY], lap2[NY];
#pragma unroll
            for (int jj = 0; jj < NY; ++jj) lap[jj] = lap2[jj] = f2(0.0f, 0.0f);
#pragma unroll
            for (int k = 1; k <= R; ++k) {
                yu[k - 1] = PY ? ld2(hp - k * T::BW) : f2(0.0f, 0.0f);
                yd[k - 1] = PY ? ld2(hp + (NY - 1 + k) * T::BW) : f2(0.0f, 0.0f);
#pragma unroll
                for (int jj = 0; jj < NY; ++jj) {
                    const float2 c0 = q[jj][slot(0)];
                    const float2 ym =
                        jj - k >= 0 ? q[(jj - k) >= 0 ? jj - k : 0][slot(0)] : yu[k - jj - 1];
                    const float2 yp =
                        jj + k < NY ? q[(jj + k) < NY ? jj + k : 0][slot(0)] : yd[jj + k - NY];
                    // (x - k, x + 1 - k) straddles two loaded pairs when WL - k is
                    // odd: two scalar adds (same rounding) instead of moves that
                    // re-pair the operands for one packed add
                    const float2 xs =
                        ((WL - k) & 1)
                            ? f2(__fadd_rn(w[jj][WL - k], w[jj][WL + k]),
                                 __fadd_rn(w[jj][WL - k + 1], w[jj][WL + k + 1]))
                            : add2(f2(w[jj][WL - k], w[jj][WL - k + 1]),
                                   f2(w[jj][WL + k], w[jj][WL + k + 1]));
                    const float2 zs = add2(q[jj][slot(-k)], q[jj][slot(k)]);
                    float2 sk = add2(add2(xs, add2(ym, yp)), zs);
                    sk = fma2(neg2nd, c0, sk);
                    if (R >= 5 && (k & 1) == 0)
                        lap2[jj] = fma2(wk[k], sk, lap2[jj]);
                    else
                        lap[jj] = fma2(wk[k], sk, lap[jj]);
                }
            }

#pragma unroll
            for (int jj = 0; jj < NY; ++jj) {
                const float2 c0 = q[jj][slot(0)];
                const float2 lp = R >= 5 ? add2(lap[jj], lap2[jj]) : lap[jj];
                const int ci = cidx + jj * T::TX;
                const float2 d = fma2(ld2(U2 + ci), mone, c0);
                const float2 c2v = ld2(C2 + ci);
                const float2 c1v =
                    SEP ? fma2(f2(fminf(nez, nexy[jj].x), fminf(nez, nexy[jj].y)), c2v,
                               f2(1.0f, 1.0f))
                        : ld2(C1 + ci);
                const float2 inc = fma2(c1v, d, mul2(c2v, lp));
                const float2 o = add2(c0, inc);
                char* pj = cur + jj * rowb;
                const bool inb = SFDB_CHECK(
                    a.dbg,
                    !vy[jj] || (reinterpret_cast<float*>(pj) >= a.out &&
                                reinterpret_cast<float*>(pj) + 2 <= a.out + a.slot),
                    kDbgStore);
                if (vy[jj] && inb) st2(reinterpret_cast<float*>(pj), o);
                if constexpr (GRAD) {
                    const float2 vtt = fma2(d, mone, inc);
                    const float2 coef = mul2(nidt2, ld2(UT + ci));
                    if (vy[jj] && inb)
                        st2(reinterpret_cast<float*>(pj + gdiff), fma2(coef, vtt, ld2(GR + ci)));
                }
            }
            if (dz > 0)
                cur += planeb;
            else
                cur -= planeb;

            __syncwarp();
            if (lx == 0) mbar_arrive(&empty[st]);
            if constexpr (SST) {
                if constexpr (PH % S == S - 1) phase ^= 1u;
            } else if (++stage == S) {
                stage = 0;
                phase ^= 1u;
            }
        };

        for (int base = 0; base < n; base += UN) {
            [&]<int... PP>(std::integer_sequence<int, PP...>) {
                ((base + PP < n ? (plane(IC<PP>{}, base + PP), true) : false) && ...);
            }(std::make_integer_sequence<int, UN>{});
            if constexpr (!ROT) {  // drop the UN oldest planes
#pragma unroll
                for (int jj = 0; jj < NY; ++jj)
#pragma unroll
                    for (int t = 0; t < 2 * R; ++t) q[jj][t] = q[jj][t + UN];
            }
        }
        j += static_cast<uint32_t>(n);
        // Fused Inject once every consumer warp has stored this item's planes
        // (named barrier over the consumer warps only).
        // The table entry is the item's own (`tab`), so every corner is added
        // by the CTA that stored it, after its store.  (Indexing by the launch
        // position made another CTA add it under the grouped order: its atomic
        // raced with the owner's plain store and an injection could be lost.)
        if (a.inj_tab && __ldg(a.inj_tab + tab + 1) > __ldg(a.inj_tab + tab)) {
            named_barrier_sync(1, NT);
            inject_cta<GRAD, NT>(a, tab, tid, x0, y0, zb, ze, T::TY, py, pz);
        }
        // Fused P2P ghost exchange (boundary items only): after the item's
        // injections, each thread re-sends the values it stored (read back
        // through L2) to the neighbour's ghost planes; the last boundary item
        // of the launch then publishes the step to the neighbours' counters.
        // Nothing goes to the neighbours once the exchange is broken (a
        // neighbour timed out): the flag is read by one thread and reduced
        // over the consumer warps, so the whole CTA takes the same branch.
        if (bs >= 0 &&
            !named_barrier_or(1, NT, tid == 0 && a.broken &&
                                         *reinterpret_cast<const volatile unsigned int*>(a.broken))) {
            // (the barrier also orders the injections (atomics) before the re-send)
            const long long pd = a.pdelta[bs];
            const char* c = reinterpret_cast<const char*>(
                a.out + static_cast<long long>(z0) * pz + static_cast<long long>(y0 + r0) * py + x);
            // the R planes at the neighbour's end of the item (it streams up)
            for (int i = bs == 0 ? 0 : n - R; i < (bs == 0 ? R : n); ++i) {
                const char* cp = c + static_cast<long long>(i) * planeb;
#pragma unroll
                for (int jj = 0; jj < NY; ++jj)
                    if (vy[jj]) {
                        const float* src = reinterpret_cast<const float*>(cp + jj * rowb);
                        const float2 v = __ldcg(reinterpret_cast<const float2*>(src));
                        float* dst = reinterpret_cast<float*>(const_cast<char*>(cp + jj * rowb) + pd);
                        if (SFDB_CHECK(a.dbg,
                                       !a.peer_row[bs] ||
                                           (dst >= a.peer_row[bs] &&
                                            dst + 2 <= a.peer_row[bs] + a.peer_slot[bs]),
                                       kDbgPeerStore))
                            st2(dst, v);
                    }
            }
            if (a.done) {
                __threadfence_system();  // this thread's peer stores, system-wide
                named_barrier_sync(1, NT);
                if (tid == 0 && atomicAdd(a.done, 1u) + 1u == a.done_target) {
                    __threadfence_system();
                    for (int sd = 0; sd < 2; ++sd)
                        if (a.sig[sd])
                            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.sig[sd]),
                                         "r"(a.sig_value)
                                         : "memory");
                }
            }
        }
    }
}

// Directions of the z chunks (SweepArgs::zdown) for a launch of `tiles` x
// `zchunks` items, item = tile + tiles * chunk, `slots` resident at a time.
// A chunk runs in wave (middle item) / slots.  The boundary between chunks k
// and k+1 is read once from DRAM when the two read its planes at the same
// time: same wave and both start there (k down, k+1 up) or both end there
// (k up, k+1 down); k one wave before k+1 and both up (k ends where k+1
// starts); k one wave after k+1 and both down.  Exhaustive over <= 12 chunks.
inline unsigned long long zdown_mask(int tiles, int zchunks, long long slots) {
    if (zchunks < 2 || zchunks > 12 || slots < 1) return 0;
    int wave[12];
    for (int k = 0; k < zchunks; ++k)
        wave[k] = static_cast<int>((static_cast<long long>(tiles) * k + tiles / 2) / slots);
    int best = -1;
    unsigned long long pick = 0;
    for (unsigned long long m = 0; m < (1ull << zchunks); ++m) {
        int ok = 0;
        for (int k = 0; k + 1 < zchunks; ++k) {
            const bool dk = (m >> k) & 1, dn = (m >> (k + 1)) & 1;
            if (wave[k] == wave[k + 1]) ok += dk != dn;
            else if (wave[k] + 1 == wave[k + 1]) ok += !dk && !dn;
            else if (wave[k] == wave[k + 1] + 1) ok += dk && dn;
        }
        if (ok > best) {
            best = ok;
            pick = m;
        }
    }
    return pick;
}

// The kernel template as ncu names it (detail::g_describe).
inline std::string kernel_name(const char* base, std::initializer_list<int> args) {
    std::string s = std::string(base) + "<";
    int k = 0;
    for (int a : args) s += (k++ ? ", " : "") + std::to_string(a);
    return s + ">";
}

// Shared-memory carveout of the sweep kernels.  The gradient kernels ask for
// the whole array as shared memory: with the driver's choice cfg3's gradient
// sweep ran 4 CTAs per SM where its registers allow 5 (115 vs 110 us per
// sweep, +3-5 % Gpts/s, profiles/r02p).  The forward kernels are register-
// limited at the driver's carveout and keep it (all-shared measured neutral
// to -2 %, the smaller L1).  SFDB200_CARVEOUT (percent; -1 = the driver's
// choice) overrides both.
template <typename K>
cudaError_t set_sweep_attrs(K kern, size_t smem, bool grad) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    static const int env = [] {
        const char* v = std::getenv("SFDB200_CARVEOUT");
        return v && *v ? std::atoi(v) : -2;
    }();
    const int pct = env != -2 ? env : grad ? static_cast<int>(cudaSharedmemCarveoutMaxShared) : -1;
    if (pct < 0) return cudaSuccess;
    return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

// occ != nullptr: report resident CTAs per SM instead of launching.
template <int R, int BY, int NY, int S, bool GRAD>
cudaError_t launch3d_t(const FieldGeom& g, const SweepConfig& cfg, const SweepMaps& m,
                       const SweepArgs& a, cudaStream_t s, int* occ) {
    auto kern = sweep3d_kernel<R, BY, NY, S, GRAD, true>;
    if (g_describe) {
        *g_describe = kernel_name("sweep3d_kernel", {R, BY, NY, S, GRAD, 1});
        return cudaSuccess;
    }
    const size_t smem = sweep3d_smem_bytes(R, cfg, GRAD);
    cudaError_t e = set_sweep_attrs(kern, smem, GRAD);
    if (e != cudaSuccess) return e;
    if (occ) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, 32 * (BY + 1), smem);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cfg.tiles_x, cfg.tiles_y, cfg.zchunks);
    lc.blockDim = dim3(32, BY + 1);  // BY consumer warps + the TMA producer warp
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = cfg.pdl ? 1 : 0;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, kern, m.uh, m.uc, m.c1, m.c2, m.ut, m.gr, a, g.Px, g.Py,
                              g.py, g.pz);
}

constexpr int kMaxDevices = 64;


template <int R, int BY, int NY, int S, bool GRAD, int MINB, int UN, bool SEP>
cudaError_t launch3d_pair_t(const FieldGeom& g, const SweepConfig& cfg, const SweepMaps& m,
                            const SweepArgs& a, cudaStream_t s, int* occ) {
    auto kern = sweep3d_pair_kernel<R, BY, NY, S, GRAD, MINB, UN, SEP>;
    if (g_describe) {
        *g_describe = kernel_name("sweep3d_pair_kernel", {R, BY, NY, S, GRAD, MINB, UN, SEP});
        return cudaSuccess;
    }
    if (!occ && (a.ez != nullptr) != SEP) return cudaErrorInvalidValue;  // layout mismatch
    const size_t smem = sweep3d_smem_bytes(R, cfg, GRAD);
    // Per instantiation and device: CTAs per SM at this smem size (the
    // max-smem attribute and the occupancy are per device; concurrent
    // sfdb200_call threads share the cache under its mutex).
    struct Occ {
        std::mutex mu;
        int resident[kMaxDevices] = {};
        int sms[kMaxDevices] = {};
        size_t smem[kMaxDevices] = {};
    };
    static Occ cache;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    int resident = 0, sms = 0;
    {
        std::lock_guard<std::mutex> lk(cache.mu);
        if (occ || cache.smem[dev] != smem) {
            e = set_sweep_attrs(kern, smem, GRAD);
            if (e != cudaSuccess) return e;
            int r = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, kern, 32 * (BY + 1), smem);
            if (e != cudaSuccess) return e;
            if (occ) {
                *occ = r;
                return cudaSuccess;
            }
            int n = 0;
            if ((e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
                return e;
            cache.resident[dev] = r;
            cache.sms[dev] = n;
            cache.smem[dev] = smem;
        }
        resident = cache.resident[dev];
        sms = cache.sms[dev];
    }
    if (resident < 1) return cudaErrorInvalidConfiguration;
    const int nitems = cfg.tiles_x * cfg.tiles_y * cfg.zchunks + a.nbi;  // + P2P boundary tiles
    // cfg.ctas: 0 = one CTA per item (the hardware hands items to free slots
    // dynamically), > 0 = that many persistent CTAs, < 0 = one per resident slot.
    // (the dynamic mode needs the separable stage layout's spare slot for the
    // item index; without it, or without a counter, one CTA per item)
    const bool dyn = cfg.ctas == -2 && SEP && a.item_ctr;
    const int ctas = cfg.ctas > 0           ? std::min(cfg.ctas, nitems)
                     : (cfg.ctas == -1 || dyn) ? std::min(nitems, resident * sms)
                                               : nitems;
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(static_cast<unsigned>(ctas));  // CTA c: items c, c + ctas, ...
    lc.blockDim = dim3(32, BY + 1);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = cfg.pdl ? 1 : 0;
    lc.attrs = at;
    lc.numAttrs = 1;
    SweepArgs b = a;
    if (!dyn) b.item_ctr = nullptr;
    const long long slots = static_cast<long long>(resident) * sms;
    const int tiles = cfg.tiles_x * cfg.tiles_y;
    // cfg.group > 1 overrides the group size (test knob: the grouped order on
    // grids smaller than the resident slots)
    const long long gsize = cfg.group > 1 ? cfg.group : slots;
    b.group = cfg.group && ctas == nitems && cfg.zchunks > 1 && tiles > gsize
                  ? static_cast<int>(gsize)
                  : 0;
    b.zdown = b.group ? 0 : zdown_mask(tiles, cfg.zchunks, ctas < nitems ? ctas : slots);
    return cudaLaunchKernelEx(&lc, kern, m.uh, m.uc, m.c1, m.c2, m.ut, m.gr, b, g.Px, g.Py,
                              g.py, g.pz, cfg.tiles_x, cfg.tiles_y, nitems);
}

template <int R, bool GRAD>
cudaError_t launch3d_r(const FieldGeom& g, const SweepConfig& cfg, const SweepMaps& m,
                       const SweepArgs& a, cudaStream_t s, int* occ) {
    // (by, ny, stages) variants compiled for every radius (see kSweepVariants).
    // Pair-mapping variants (by, ny, stages); the register budget (resident
    // CTAs the kernel is compiled for) follows from the z queue, ny (2R+1)
    // float2 per thread.
    constexpr int MB2 = R <= 4 ? 4 : 3;  // ny = 2, 4 warps
// BOTH: also compiled for streamed c1 (non-separable damping); the other
// variants exist for the separable layout only.
#define SFDB_P(BY, NY, S, MINB, ROTV, BOTH)                                                   \
    if (cfg.pair && cfg.by == BY && cfg.ny == NY && cfg.stages == S && cfg.rot == ROTV) {     \
        if (cfg.sep)                                                                          \
            return launch3d_pair_t<R, BY, NY, S, GRAD, MINB, z_unroll<R, ROTV>(), true>(      \
                g, cfg, m, a, s, occ);                                                        \
        if constexpr (BOTH)                                                                   \
            return launch3d_pair_t<R, BY, NY, S, GRAD, MINB, z_unroll<R, ROTV>(), false>(     \
                g, cfg, m, a, s, occ);                                                        \
        return cudaErrorInvalidConfiguration;                                                 \
    }
    constexpr int MB3 = R <= 4 ? 4 : 3;
    SFDB_P(4, 2, 4, MB2, 0, 1)
    SFDB_P(4, 2, 3, MB3, 0, 0)
    SFDB_P(4, 1, 4, 4, 0, 0)
    SFDB_P(4, 2, 4, MB2, 1, 0)
    SFDB_P(4, 2, 3, MB3, 1, 0)
    SFDB_P(8, 2, 3, (R <= 4 ? 2 : 1), 1, 0)
    // eight consumer warps, one row per thread: a 32 x 16 tile with a third
    // of the y halo of the 32 x 8 one (the gradient's six staged boxes)
    if constexpr (R <= 4) {
        SFDB_P(8, 1, 4, 3, 0, 1)
        SFDB_P(8, 1, 3, 3, 0, 1)
    }
    // partial unrolls (queue shifted every 2 / 3 / 4 / 5 / 8 planes); five
    // stages fit four CTAs per SM only in the separable layout
    SFDB_P(4, 2, 4, MB2, 2, 0)
    SFDB_P(4, 2, 4, MB2, 4, 1)
    SFDB_P(4, 2, 5, MB2, 0, 0)
    SFDB_P(4, 2, 5, MB2, 5, 0)
    if constexpr (R >= 5) SFDB_P(4, 2, 4, MB2, 8, 0)
    if constexpr (R <= 4) {
        SFDB_P(4, 2, 3, 4, 3, 0)
        SFDB_P(4, 2, 4, 4, 3, 0)
        SFDB_P(4, 2, 3, 4, 4, 0)
    }
#undef SFDB_P
    if (cfg.pair) return cudaErrorInvalidConfiguration;
#define SFDB_V(BY, NY, S)                                              \
    if (cfg.by == BY && cfg.ny == NY && cfg.stages == S)               \
        return launch3d_t<R, BY, NY, S, GRAD>(g, cfg, m, a, s, occ);
    if constexpr (R <= 4) {  // two rows per half: the queue fits the registers
        SFDB_V(4, 2, 4)
        SFDB_V(4, 2, 3)
        SFDB_V(4, 2, 6)
    }
    SFDB_V(4, 1, 4)
    SFDB_V(4, 1, 3)
    SFDB_V(4, 1, 6)
#undef SFDB_V
    return cudaErrorInvalidConfiguration;
}

}  // namespace detail
}  // namespace sfdb200
