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

#include <cmath>
#include <utility>

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

__global__ void coeffs_kernel(const double* __restrict__ m, const double* __restrict__ damp,
                              double dt, float* __restrict__ c1, float* __restrict__ c2,
                              long long cells, int Px, int XP) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= cells) return;
    const long long r = i / Px, x = i - r * Px;
    const double a = m[i] / (dt * dt);
    const double b = damp[i] / (2.0 * dt);
    c1[r * XP + x] = static_cast<float>((a - b) / (a + b));
    c2[r * XP + x] = static_cast<float>(1.0 / (a + b));
}

__global__ void to_f32_kernel(const double* __restrict__ src, float* __restrict__ dst,
                              long long n, int Px, int XP) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const long long r = i / Px, x = i - r * Px;
    dst[r * XP + x] = static_cast<float>(src[i]);
}

__global__ void to_f64_kernel(const float* __restrict__ src, double* __restrict__ dst,
                              long long n, int Px, int XP) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const long long r = i / Px, x = i - r * Px;
    dst[i] = static_cast<double>(src[r * XP + x]);
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
    const int SF = HF + (grad ? 6 : 4) * CF;
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

cudaError_t launch_inject(float* field, const long long* off, const float* coef, const int* pt,
                          const float* row, long n, float* grad, const float* ut,
                          const unsigned char* gmask, float nidt2, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    inject_kernel<<<grid_for(n, 128), 128, 0, s>>>(field, off, coef, pt, row, n, grad, ut, gmask,
                                                   nidt2);
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

cudaError_t launch_coeffs(const FieldGeom& g, const double* m, const double* damp, double dt,
                          float* c1, float* c2, cudaStream_t s) {
    const long long cells = static_cast<long long>(g.Pz) * g.Py * g.Px;
    coeffs_kernel<<<grid_for(cells, 256), 256, 0, s>>>(m, damp, dt, c1, c2, cells, g.Px, g.XP);
    return cudaGetLastError();
}

cudaError_t launch_to_f32(const FieldGeom& g, const double* src, float* dst, long long rows,
                          cudaStream_t s) {
    const long long n = rows * g.Pz * g.Py * g.Px;
    if (n == 0) return cudaSuccess;
    to_f32_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, g.Px, g.XP);
    return cudaGetLastError();
}

cudaError_t launch_to_f64(const FieldGeom& g, const float* src, double* dst, long long rows,
                          cudaStream_t s) {
    const long long n = rows * g.Pz * g.Py * g.Px;
    if (n == 0) return cudaSuccess;
    to_f64_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, g.Px, g.XP);
    return cudaGetLastError();
}

cudaError_t launch_dense_to_f32(const double* src, float* dst, long long n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    to_f32_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, 1, 1);
    return cudaGetLastError();
}

cudaError_t launch_dense_to_f64(const float* src, double* dst, long long n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    to_f64_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, 1, 1);
    return cudaGetLastError();
}

cudaError_t launch_count_nonfinite(const float* a, long long n, unsigned long long* counter,
                                   cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    nonfinite_kernel<<<592, 256, 0, s>>>(a, n, counter);
    return cudaGetLastError();
}

}  // namespace sfdb200
