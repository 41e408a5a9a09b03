// sm_100a kernels for the damped acoustic stencil hot path.
//
// Reference semantics (what each kernel replaces):
//   sweep3d / sweep2d  the emitted spatial sweep, proj/src/codegen.cpp:348-417
//                      (golden proj/tests/golden/forward_3d_full.c:41-50); the
//                      damping term is fused (it is part of the solved update)
//   GRAD variant       the second assignment of build_gradient_ir,
//                      proj/src/seismic.cpp:311-318, in summation-by-parts form
//   inject             Inject sparse op, codegen.cpp:436-449 / interpreter.cpp:135-149
//   sample             Sample sparse op, codegen.cpp:450-458 / interpreter.cpp:150-160
//
// Design: the 3-D sweep is a 2.5-D z-streaming stencil.  A CTA
// owns a 32 x TY column of (y, x) and marches along z.  Per z-plane one thread
// issues TMA box loads (cp.async.bulk.tensor) into a ring of shared-memory
// stages guarded by mbarriers: the u1 plane with its R-wide x/y halo, the u1
// centre box R planes ahead (feeds the per-thread register queue that holds
// the 2R+1 z-neighbours), and the u2 / c1 / c2 (and u_t) centre boxes.  Every
// HBM byte is read once per step (halo re-reads hit L2), the output is stored
// straight from registers with 128-byte coalesced rows.
#include "kernels.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <utility>

namespace cg = cooperative_groups;

namespace sfdb200 {
namespace {

// ---------------------------------------------------------------- 2-D sweep
// 2-D fields are small (cfg1: 285^2 cells = 0.3 MB per row, L2-resident):
// one thread per point, neighbours through L1.

template <int R, bool GRAD>
__global__ void __launch_bounds__(256) sweep2d_kernel(const SweepArgs a, const int Px,
                                                       const long long pz) {
    const int x = R + blockIdx.x * 32 + threadIdx.x;
    const int z = R + blockIdx.y * 8 + threadIdx.y;
    if (x >= Px - R || z >= a.zhi) return;
    const long long o = static_cast<long long>(z) * pz + x;
    const float* u1 = a.u1 + o;
    const float c0 = __ldg(u1);
    float lap = 0.0f;
#pragma unroll
    for (int k = 1; k <= R; ++k) {
        float s = (__ldg(u1 - k) + __ldg(u1 + k)) + (__ldg(u1 - k * pz) + __ldg(u1 + k * pz));
        s = fmaf(a.neg2nd, c0, s);
        lap = fmaf(a.w[k], s, lap);
    }
    const float d = c0 - __ldg(a.u2 + o);
    const float inc = fmaf(__ldg(a.c1 + o), d, __ldg(a.c2 + o) * lap);
    a.out[o] = c0 + inc;
    if constexpr (GRAD) a.grad[o] = fmaf(a.nidt2 * __ldg(a.ut + o), inc - d, a.grad[o]);
}

// ---------------------------------------------------------------- 2-D time loop
// 2-D problems are small (cfg1: 78,961 updated points, 0.3 MB per row, all in
// L2), so a launch per step would be launch-bound.  One cooperative launch
// runs every step: each CTA owns a contiguous range of updated points; per
// step it samples its share of the previous row's receivers, sweeps its
// points, applies the injections whose corner it owns (after a CTA barrier,
// in the reference's (p, c) order, atomics for collisions) and meets the rest
// of the grid at grid.sync().  Field rows are written inside the launch, so
// they are read with ld.global.cg (L2, never a stale L1 line); c1, c2 and the
// history are read-only.

template <int R, bool GRAD>
__global__ void __launch_bounds__(256) loop2d_kernel(const Loop2dArgs a) {
    cg::grid_group grid = cg::this_grid();
    const int cta = blockIdx.x;
    const int tid = threadIdx.x;
    const int nth = blockDim.x;
    const int nx = a.Px - 2 * R;
    const long long p0 = static_cast<long long>(cta) * a.per_cta;
    const long long p1 = min(p0 + a.per_cta, a.npts);
    const bool fwd = a.kind == 0;
    const long steps = a.nt > 2 ? a.nt - 2 : 0;
    const int e_begin = a.inj_n ? a.inj_begin[cta] : 0;
    const int e_end = a.inj_n ? a.inj_begin[cta + 1] : 0;
    auto sample = [&](const float* field, long row) {
        const long q0 = static_cast<long>(cta) * a.smp_per_cta;
        const long q1 = min(q0 + a.smp_per_cta, a.smp_cnt);
        for (long q = q0 + tid; q < q1; q += nth) {
            float acc = 0.0f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const long long o = a.smp_off[4 * q + c];
                if (SFDB_CHECK(a.dbg, o >= 0 && o < a.slot, kDbg2d))
                    acc = fmaf(__ldg(a.smp_w + 4 * q + c), __ldcg(field + o), acc);
            }
            a.smp_trace[row * a.smp_n + a.smp_pt[q]] = acc;
        }
    };
    long prev_row = -1;
    const float* prev_out = nullptr;
    for (long i = 0; i < steps; ++i) {
        const long t = fwd ? 2 + i : a.nt - 1 - i;
        long r0, r1, r2;
        if (fwd && a.save) {
            r0 = t; r1 = t - 1; r2 = t - 2;
        } else if (fwd) {
            r0 = t % 3; r1 = (t - 1) % 3; r2 = (t - 2) % 3;
        } else {
            r0 = t % 3; r1 = (t + 1) % 3; r2 = (t + 2) % 3;
        }
        float* out = a.field + r0 * a.slot;
        const float* u1 = a.field + r1 * a.slot;
        const float* u2 = a.field + r2 * a.slot;
        const float* ut = GRAD ? a.hist + t * a.slot : nullptr;
        if (prev_out && a.smp_cnt) sample(prev_out, prev_row);
        for (long long p = p0 + tid; p < p1; p += nth) {
            const long long z = R + p / nx, x = R + p % nx;
            const long long o = z * a.pz + x;
            const float c0 = __ldcg(u1 + o);
            float lap = 0.0f;
#pragma unroll
            for (int k = 1; k <= R; ++k) {
                float s = (__ldcg(u1 + o - k) + __ldcg(u1 + o + k)) +
                          (__ldcg(u1 + o - k * a.pz) + __ldcg(u1 + o + k * a.pz));
                s = fmaf(a.neg2nd, c0, s);
                lap = fmaf(a.w[k], s, lap);
            }
            const float d = c0 - __ldcg(u2 + o);
            const float inc = fmaf(__ldg(a.c1 + o), d, __ldg(a.c2 + o) * lap);
            out[o] = c0 + inc;
            if constexpr (GRAD) a.grad[o] = fmaf(a.nidt2 * __ldg(ut + o), inc - d, a.grad[o]);
        }
        if (e_end > e_begin) {
            __syncthreads();
            const long irow = fwd ? t - 1 : t;
            for (int e = e_begin + tid; e < e_end; e += nth) {
                const long long o = a.inj_off[e];
                if (!SFDB_CHECK(a.dbg, o >= 0 && o < a.slot, kDbg2d)) continue;
                const float delta = a.inj_coef[e] * __ldg(a.inj_trace + irow * a.inj_n + a.inj_pt[e]);
                atomicAdd(out + o, delta);
                if constexpr (GRAD)
                    if (a.inj_gm[e]) atomicAdd(a.grad + o, a.nidt2 * __ldg(ut + o) * delta);
            }
        }
        grid.sync();
        prev_row = fwd ? t : t - 1;
        prev_out = out;
    }
    if (prev_out && a.smp_cnt) sample(prev_out, prev_row);
}

// ---------------------------------------------------------------- sparse ops

__global__ void inject_kernel(float* __restrict__ field, const long long* __restrict__ off,
                              const float* __restrict__ coef, const int* __restrict__ pt,
                              const float* __restrict__ row, long n, float* __restrict__ grad,
                              const float* __restrict__ ut,
                              const unsigned char* __restrict__ gmask, float nidt2) {
    const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const long long o = off[i];
    const float delta = coef[i] * row[pt[i]];
    atomicAdd(field + o, delta);
    if (grad && gmask[i]) atomicAdd(grad + o, nidt2 * ut[o] * delta);
}

// P2P step counters (p2p.cpp): one thread polls until both counters reach
// `value` (cyclic compare), sleeping between polls.  A neighbour that never
// publishes (its process died, it stalls, or the mapping is wrong) sets the
// sticky `broken` flag after timeout_ns instead of trapping, and the flag is
// also written into both neighbours' broken flags (pb0, pb1, through their IPC
// mappings): every rank of the chain then stops its peer stores and step
// publications (the sweep checks the flag) and its waits return at once, so
// no rank runs ahead into ghost rows a neighbour still reads, and every
// rank's p2p_check / download reports the failed exchange.
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* f) {
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    return v;
}

__global__ void wait_flags_kernel(const unsigned int* f0, const unsigned int* f1,
                                  unsigned int value, unsigned long long timeout_ns,
                                  unsigned int* broken, unsigned int* pb0, unsigned int* pb1) {
    auto poison = [&] {
        atomicExch(broken, 1u);
        __threadfence_system();
        for (unsigned int* pb : {pb0, pb1})
            if (pb) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pb), "r"(1u) : "memory");
    };
    if (ld_acquire_sys(broken)) {
        poison();
        return;
    }
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (const unsigned int* f : {f0, f1}) {
        if (!f) continue;
        for (;;) {
            if (static_cast<int>(ld_acquire_sys(f) - value) >= 0) break;
            __nanosleep(200);
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns || ld_acquire_sys(broken)) {
                poison();
                return;
            }
        }
    }
}

// grad += v2 u2 / dt^2 over the updated region [R, P - R) of every dim
// (plan.cu grad_row2_fixup: takes the t = 2 term back out of the gradient).
__global__ void grad_row2_kernel(float* __restrict__ grad, const float* __restrict__ v2,
                                 const float* __restrict__ u2, float idt2, FieldGeom g) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int z = blockIdx.z;
    if (x < g.R || x >= g.Px - g.R || z < g.R || z >= g.Pz - g.R) return;
    if (g.ndim == 3 && (y < g.R || y >= g.Py - g.R)) return;
    const long long c = z * g.pz + y * g.py + x;
    grad[c] = fmaf(v2[c] * u2[c], idt2, grad[c]);
}

template <int C>
__global__ void sample_kernel(const float* __restrict__ field, const long long* __restrict__ off,
                              const float* __restrict__ w, const int* __restrict__ pt,
                              float* __restrict__ row, long n, int corners) {
    const long p = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    if (p >= n) return;
    const int nc = C > 0 ? C : corners;
    float v[C > 0 ? C : 8];
    float acc = 0.0f;
    if constexpr (C > 0) {
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = __ldg(field + __ldg(off + p * C + c));
#pragma unroll
        for (int c = 0; c < C; ++c) acc = fmaf(__ldg(w + p * C + c), v[c], acc);
    } else {
        for (int c = 0; c < nc; ++c) acc = fmaf(w[p * nc + c], field[off[p * nc + c]], acc);
    }
    row[pt ? pt[p] : p] = acc;
}

// ---------------------------------------------------------------- conversions

// 3-D (R > 0): the coefficients of the x/y halo cells (never updated) are
// zero, so the sweep may store its result there unconditionally: with
// u1 = u2 = 0 on the halo the update yields exactly 0 (sweep3d.cuh).
template <class M>
__global__ void coeffs_kernel(const M* __restrict__ m, const double* __restrict__ damp,
                              double dt, float* __restrict__ c1, float* __restrict__ c2,
                              long long cells, int Px, int XP, int Py, int R) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= cells) return;
    const long long r = i / Px, x = i - r * Px;
    const long long y = r % Py;
    if (R > 0 && (x < R || x >= Px - R || y < R || y >= Py - R)) {
        c1[r * XP + x] = 0.0f;
        c2[r * XP + x] = 0.0f;
        return;
    }
    const double a = static_cast<double>(m[i]) / (dt * dt);
    const double b = damp[i] / (2.0 * dt);
    c1[r * XP + x] = static_cast<float>((a - b) / (a + b));
    c2[r * XP + x] = static_cast<float>(1.0 / (a + b));
}

// The same coefficients from m and host-checked separable damp profiles
// (pz, py, px as doubles; hostio.cpp host_sep_damp): the damp value of every
// cell is max(pz[z], py[y], px[x]), bit for bit the caller's (checked).
// M = float: m arrived narrowed on the host, which happens only when every
// value is exactly representable (hostio.cpp copy_h2d_narrow), so
// static_cast<double>(m[i]) is the caller's fp64 value and the coefficients
// are bit for bit the ones from the fp64 upload.
template <class M>
__global__ void coeffs_sep_kernel(const M* __restrict__ m, const double* __restrict__ prof,
                                  double dt, float* __restrict__ c1, float* __restrict__ c2,
                                  long long cells, int Px, int XP, int Py, int Pz, int R) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= cells) return;
    const long long r = i / Px, x = i - r * Px;
    const long long z = r / Py, y = r - z * Py;
    if (x < R || x >= Px - R || y < R || y >= Py - R) {
        c1[r * XP + x] = 0.0f;
        c2[r * XP + x] = 0.0f;
        return;
    }
    const double dmp = fmax(fmax(prof[z], prof[Pz + y]), prof[Pz + Py + x]);
    const double a = static_cast<double>(m[i]) / (dt * dt);
    const double b = dmp / (2.0 * dt);
    c1[r * XP + x] = static_cast<float>((a - b) / (a + b));
    c2[r * XP + x] = static_cast<float>(1.0 / (a + b));
}

// ---- separable damping profiles (see SweepArgs::ez) ----------------------
// Non-negative doubles order like their bit patterns, so the per-axis minima
// are 64-bit atomicMin on the bits; any other input fails the exact check.
__global__ void prof_fill_kernel(unsigned long long* a, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = 0x7FF0000000000000ull;  // +inf
}

constexpr int kProfRows = 16;

__global__ void prof_min_kernel(const double* __restrict__ damp, int Pz, int Py, int Px,
                                unsigned long long* pz, unsigned long long* py,
                                unsigned long long* px) {
    const int z = blockIdx.y, y0 = blockIdx.x * kProfRows;
    const int ny = min(kProfRows, Py - y0);
    unsigned long long rmin[kProfRows];
#pragma unroll
    for (int r = 0; r < kProfRows; ++r) rmin[r] = ~0ull;
    for (int x = threadIdx.x; x < Px; x += blockDim.x) {
        unsigned long long cmin = ~0ull;
#pragma unroll
        for (int r = 0; r < kProfRows; ++r) {
            if (r < ny) {
                const unsigned long long v = __double_as_longlong(
                    damp[(static_cast<long long>(z) * Py + y0 + r) * Px + x]);
                cmin = min(cmin, v);
                rmin[r] = min(rmin[r], v);
            }
        }
        atomicMin(px + x, cmin);
    }
    unsigned long long plane = ~0ull;
#pragma unroll
    for (int r = 0; r < kProfRows; ++r) {
        unsigned long long v = rmin[r];
        for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
        if ((threadIdx.x & 31) == 0 && r < ny) atomicMin(py + y0 + r, v);
        plane = min(plane, v);
    }
    if ((threadIdx.x & 31) == 0) atomicMin(pz + z, plane);
}

__global__ void prof_check_kernel(const double* __restrict__ damp, int Pz, int Py, int Px,
                                  const unsigned long long* pz, const unsigned long long* py,
                                  const unsigned long long* px, unsigned int* mismatch) {
    const long long n = static_cast<long long>(Pz) * Py * Px;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long zy = i / Px;
        const int x = static_cast<int>(i - zy * Px);
        const int z = static_cast<int>(zy / Py), y = static_cast<int>(zy - static_cast<long long>(z) * Py);
        const double r = fmax(fmax(__longlong_as_double(pz[z]), __longlong_as_double(py[y])),
                              __longlong_as_double(px[x]));
        const double v = damp[i];
        if (!(v == r) || !(v >= 0.0)) *mismatch = 1u;
    }
}

__global__ void prof_out_kernel(const unsigned long long* a, int n, double dt, float* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = static_cast<float>(__longlong_as_double(a[i]) / dt);
}

// dense [rows][Px] -> pitched [rows][XP] (with a type conversion)
template <class S, class D>
__global__ void pitch_kernel(const S* __restrict__ src, D* __restrict__ dst, long long n, int Px,
                             int XP) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const long long r = i / Px, x = i - r * Px;
    dst[r * XP + x] = static_cast<D>(src[i]);
}

// pitched [rows][XP] -> dense [rows][Px]
template <class S, class D>
__global__ void unpitch_kernel(const S* __restrict__ src, D* __restrict__ dst, long long n, int Px,
                               int XP) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const long long r = i / Px, x = i - r * Px;
    dst[i] = static_cast<D>(src[r * XP + x]);
}

__global__ void nonfinite_kernel(const float* __restrict__ a, long long n,
                                 unsigned long long* counter) {
    unsigned long long bad = 0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        bad += !isfinite(a[i]);
    bad = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(bad));
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(counter, bad);
}

unsigned grid_for(long long n, int block) {
    return static_cast<unsigned>((n + block - 1) / block);
}

}  // namespace

size_t sweep3d_smem_bytes(int R, const SweepConfig& cfg, bool grad) {
    const int TY = cfg.ty();
    const int BW = cfg.bw(R);
    const int HF = ((TY + 2 * R) * BW + 31) & ~31;
    const int CF = TY * 32;
    // sweep3d.cuh Tile: the separable layout drops the c1 box and keeps 32
    // floats for -ez[z]
    const bool sep = cfg.pair && cfg.sep;
    const int SF = HF + ((grad ? 6 : 4) - (sep ? 1 : 0)) * CF + (sep ? 32 : 0);
    return static_cast<size_t>(cfg.stages) * SF * 4 + cfg.stages * 16 + 128;
}

static cudaError_t dispatch3d(const FieldGeom& g, const SweepConfig& cfg, const SweepMaps& m,
                              const SweepArgs& a, bool grad, cudaStream_t s, int* occ) {
#define SFDB_R_CASE(RR)                                                   \
    case RR:                                                              \
        return sweep3d_r##RR(g, cfg, m, a, grad, s, occ);
    switch (g.R) {
        SFDB_R_CASE(1)
        SFDB_R_CASE(2)
        SFDB_R_CASE(3)
        SFDB_R_CASE(4)
        SFDB_R_CASE(5)
        SFDB_R_CASE(6)
        SFDB_R_CASE(7)
        SFDB_R_CASE(8)
        default:
            return cudaErrorInvalidValue;
    }
#undef SFDB_R_CASE
}

cudaError_t launch_sweep3d(const FieldGeom& g, const SweepConfig& cfg, const SweepMaps& m,
                           const SweepArgs& a, bool grad, cudaStream_t s) {
    return dispatch3d(g, cfg, m, a, grad, s, nullptr);
}

std::string sweep3d_instantiation(const FieldGeom& g, const SweepConfig& cfg, bool grad) {
    std::string name;
    SweepMaps m{};
    SweepArgs a{};
    detail::g_describe = &name;
    const cudaError_t e = dispatch3d(g, cfg, m, a, grad, nullptr, nullptr);
    detail::g_describe = nullptr;
    return e == cudaSuccess ? name : std::string();
}

cudaError_t sweep3d_occupancy(const FieldGeom& g, const SweepConfig& cfg, bool grad,
                              int* blocks_per_sm) {
    SweepMaps m{};
    SweepArgs a{};
    return dispatch3d(g, cfg, m, a, grad, nullptr, blocks_per_sm);
}

cudaError_t launch_sweep2d(const FieldGeom& g, const SweepArgs& a, bool grad, cudaStream_t s) {
    const dim3 block(32, 8);
    const dim3 grid(grid_for(g.Px - 2 * g.R, 32), grid_for(g.Pz - 2 * g.R, 8));
#define SFDB_R_CASE(RR)                                                          \
    case RR:                                                                     \
        if (grad)                                                                \
            sweep2d_kernel<RR, true><<<grid, block, 0, s>>>(a, g.Px, g.pz);      \
        else                                                                     \
            sweep2d_kernel<RR, false><<<grid, block, 0, s>>>(a, g.Px, g.pz);     \
        break;
    switch (g.R) {
        SFDB_R_CASE(1)
        SFDB_R_CASE(2)
        SFDB_R_CASE(3)
        SFDB_R_CASE(4)
        SFDB_R_CASE(5)
        SFDB_R_CASE(6)
        SFDB_R_CASE(7)
        SFDB_R_CASE(8)
        default:
            return cudaErrorInvalidValue;
    }
#undef SFDB_R_CASE
    return cudaGetLastError();
}

cudaError_t launch_loop2d(const Loop2dArgs& a, int R, bool grad, int ctas, cudaStream_t s) {
    void* args[] = {const_cast<Loop2dArgs*>(&a)};
    void* fn = nullptr;
#define SFDB_R_CASE(RR)                                                                     \
    case RR:                                                                                \
        fn = grad ? reinterpret_cast<void*>(loop2d_kernel<RR, true>)                        \
                  : reinterpret_cast<void*>(loop2d_kernel<RR, false>);                      \
        break;
    switch (R) {
        SFDB_R_CASE(1)
        SFDB_R_CASE(2)
        SFDB_R_CASE(3)
        SFDB_R_CASE(4)
        SFDB_R_CASE(5)
        SFDB_R_CASE(6)
        SFDB_R_CASE(7)
        SFDB_R_CASE(8)
        default:
            return cudaErrorInvalidValue;
    }
#undef SFDB_R_CASE
    if (ctas < 0) {  // query: co-resident CTAs per SM
        int occ = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, 0);
        return e != cudaSuccess ? e : (occ > 0 ? cudaSuccess : cudaErrorInvalidConfiguration);
    }
    return cudaLaunchCooperativeKernel(fn, dim3(ctas), dim3(256), args, 0, s);
}

int loop2d_blocks_per_sm(int R, bool grad) {
    void* fn = nullptr;
#define SFDB_R_CASE(RR)                                                                     \
    case RR:                                                                                \
        fn = grad ? reinterpret_cast<void*>(loop2d_kernel<RR, true>)                        \
                  : reinterpret_cast<void*>(loop2d_kernel<RR, false>);                      \
        break;
    switch (R) {
        SFDB_R_CASE(1)
        SFDB_R_CASE(2)
        SFDB_R_CASE(3)
        SFDB_R_CASE(4)
        SFDB_R_CASE(5)
        SFDB_R_CASE(6)
        SFDB_R_CASE(7)
        SFDB_R_CASE(8)
        default:
            return 0;
    }
#undef SFDB_R_CASE
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, 0) != cudaSuccess) return 0;
    return occ;
}

cudaError_t launch_inject(float* field, const long long* off, const float* coef, const int* pt,
                          const float* row, long n, float* grad, const float* ut,
                          const unsigned char* gmask, float nidt2, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    inject_kernel<<<grid_for(n, 128), 128, 0, s>>>(field, off, coef, pt, row, n, grad, ut, gmask,
                                                   nidt2);
    return cudaGetLastError();
}

cudaError_t launch_grad_row2(float* grad, const float* v2, const float* u2, float idt2,
                             const FieldGeom& g, cudaStream_t s) {
    const dim3 grid((g.Px + 127) / 128, g.Py, g.Pz);
    grad_row2_kernel<<<grid, 128, 0, s>>>(grad, v2, u2, idt2, g);
    return cudaGetLastError();
}

cudaError_t launch_wait_flags(const unsigned int* f0, const unsigned int* f1, unsigned int value,
                              unsigned long long timeout_ns, unsigned int* broken,
                              unsigned int* peer_broken0, unsigned int* peer_broken1,
                              cudaStream_t s) {
    wait_flags_kernel<<<1, 1, 0, s>>>(f0, f1, value, timeout_ns, broken, peer_broken0,
                                      peer_broken1);
    return cudaGetLastError();
}

cudaError_t launch_sample(const float* field, const long long* off, const float* w,
                          const int* pt, float* row, long npoints, int corners, cudaStream_t s) {
    if (npoints == 0) return cudaSuccess;
    const unsigned grid = grid_for(npoints, 128);
    if (corners == 8)
        sample_kernel<8><<<grid, 128, 0, s>>>(field, off, w, pt, row, npoints, corners);
    else if (corners == 4)
        sample_kernel<4><<<grid, 128, 0, s>>>(field, off, w, pt, row, npoints, corners);
    else
        sample_kernel<0><<<grid, 128, 0, s>>>(field, off, w, pt, row, npoints, corners);
    return cudaGetLastError();
}

template <class M>
cudaError_t launch_coeffs_t(const FieldGeom& g, const M* m, const double* damp, double dt,
                            float* c1, float* c2, cudaStream_t s) {
    const long long cells = static_cast<long long>(g.Pz) * g.Py * g.Px;
    coeffs_kernel<<<grid_for(cells, 256), 256, 0, s>>>(m, damp, dt, c1, c2, cells, g.Px, g.XP,
                                                        g.Py, g.ndim == 3 ? g.R : 0);
    return cudaGetLastError();
}

cudaError_t launch_coeffs(const FieldGeom& g, const double* m, const double* damp, double dt,
                          float* c1, float* c2, cudaStream_t s) {
    return launch_coeffs_t(g, m, damp, dt, c1, c2, s);
}
cudaError_t launch_coeffs(const FieldGeom& g, const float* m, const double* damp, double dt,
                          float* c1, float* c2, cudaStream_t s) {
    return launch_coeffs_t(g, m, damp, dt, c1, c2, s);
}

template <class M>
cudaError_t launch_coeffs_sep_t(const FieldGeom& g, const M* m, const double* prof, double dt,
                                float* c1, float* c2, float* ez, float* ey, float* ex,
                                cudaStream_t s) {
    const long long cells = static_cast<long long>(g.Pz) * g.Py * g.Px;
    coeffs_sep_kernel<<<grid_for(cells, 256), 256, 0, s>>>(m, prof, dt, c1, c2, cells, g.Px, g.XP,
                                                            g.Py, g.Pz, g.R);
    const auto* bits = reinterpret_cast<const unsigned long long*>(prof);
    prof_out_kernel<<<grid_for(g.Pz, 256), 256, 0, s>>>(bits, g.Pz, dt, ez);
    prof_out_kernel<<<grid_for(g.Py, 256), 256, 0, s>>>(bits + g.Pz, g.Py, dt, ey);
    prof_out_kernel<<<grid_for(g.Px, 256), 256, 0, s>>>(bits + g.Pz + g.Py, g.Px, dt, ex);
    return cudaGetLastError();
}
cudaError_t launch_coeffs_sep(const FieldGeom& g, const double* m, const double* prof, double dt,
                              float* c1, float* c2, float* ez, float* ey, float* ex,
                              cudaStream_t s) {
    return launch_coeffs_sep_t(g, m, prof, dt, c1, c2, ez, ey, ex, s);
}
cudaError_t launch_coeffs_sep(const FieldGeom& g, const float* m, const double* prof, double dt,
                              float* c1, float* c2, float* ez, float* ey, float* ex,
                              cudaStream_t s) {
    return launch_coeffs_sep_t(g, m, prof, dt, c1, c2, ez, ey, ex, s);
}

cudaError_t launch_damp_profiles(const double* damp, int Pz, int Py, int Px, double dt,
                                 unsigned long long* scratch, float* ez, float* ey, float* ex,
                                 unsigned int* mismatch, cudaStream_t s) {
    unsigned long long* pz = scratch;
    unsigned long long* py = pz + Pz;
    unsigned long long* px = py + Py;
    const int n = Pz + Py + Px;
    cudaError_t e = cudaMemsetAsync(mismatch, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    prof_fill_kernel<<<grid_for(n, 256), 256, 0, s>>>(scratch, n);
    prof_min_kernel<<<dim3((Py + kProfRows - 1) / kProfRows, Pz), 256, 0, s>>>(damp, Pz, Py, Px,
                                                                                 pz, py, px);
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    prof_check_kernel<<<4 * sms, 256, 0, s>>>(damp, Pz, Py, Px, pz, py, px, mismatch);
    prof_out_kernel<<<grid_for(Pz, 256), 256, 0, s>>>(pz, Pz, dt, ez);
    prof_out_kernel<<<grid_for(Py, 256), 256, 0, s>>>(py, Py, dt, ey);
    prof_out_kernel<<<grid_for(Px, 256), 256, 0, s>>>(px, Px, dt, ex);
    return cudaGetLastError();
}

cudaError_t launch_to_f32(const FieldGeom& g, const double* src, float* dst, long long rows,
                          cudaStream_t s) {
    const long long n = rows * g.Pz * g.Py * g.Px;
    if (n == 0) return cudaSuccess;
    pitch_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, g.Px, g.XP);
    return cudaGetLastError();
}

cudaError_t launch_to_f64(const FieldGeom& g, const float* src, double* dst, long long rows,
                          cudaStream_t s) {
    const long long n = rows * g.Pz * g.Py * g.Px;
    if (n == 0) return cudaSuccess;
    unpitch_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, g.Px, g.XP);
    return cudaGetLastError();
}

cudaError_t launch_pitch_f32(const FieldGeom& g, const float* src, float* dst, long long rows,
                             cudaStream_t s) {
    const long long n = rows * g.Pz * g.Py * g.Px;
    if (n == 0) return cudaSuccess;
    pitch_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, g.Px, g.XP);
    return cudaGetLastError();
}

cudaError_t launch_unpitch_f32(const FieldGeom& g, const float* src, float* dst, long long rows,
                               cudaStream_t s) {
    const long long n = rows * g.Pz * g.Py * g.Px;
    if (n == 0) return cudaSuccess;
    unpitch_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, g.Px, g.XP);
    return cudaGetLastError();
}

cudaError_t launch_dense_to_f32(const double* src, float* dst, long long n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    pitch_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, 1, 1);
    return cudaGetLastError();
}

cudaError_t launch_dense_to_f64(const float* src, double* dst, long long n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    unpitch_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, 1, 1);
    return cudaGetLastError();
}

cudaError_t launch_count_nonfinite(const float* a, long long n, unsigned long long* counter,
                                   cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    nonfinite_kernel<<<592, 256, 0, s>>>(a, n, counter);
    return cudaGetLastError();
}

}  // namespace sfdb200
