// 2-D time loop in ONE thread-block cluster (sm_90+ clusters, distributed
// shared memory), the default 2-D path when the wavefield fits the cluster's
// shared memory (cfg1: 285 x 288 floats per row; kernels.cuh Cluster2dArgs).
//
// Replaces, for 2-D problems, the emitted sweep + inject + sample of one
// operator call (proj/src/codegen.cpp:348-462, time loop :464-547).
//
// Why: a 2-D step is ~80 K points (1.6 MB of traffic, L2-resident), so one
// launch per step is launch-bound and a grid-wide barrier per step (the
// cooperative loop2d_kernel) costs ~3 us.  Here the 3 time slots of the field
// live in shared memory, split in row bands over the cluster's CTAs; a step is
//   sweep (registers + local smem)  ->  CTA barrier  ->  inject (smem atomics)
//   ->  CTA barrier  ->  push the R edge rows into the neighbours' halo rows
//   (DSMEM stores)  ->  cluster barrier  ->  sample (local smem)
// so the only cross-SM synchronisation is the hardware cluster barrier.
//
// Thread mapping: a thread owns a column pair (x, x+1) (float2, packed fp32x2
// math as in the 3-D kernels) in a strip of NZ rows of its CTA's band; its
// c1, c2, previous-step values (u2) and gradient live in registers for the
// whole run, so per step it reads only the u1 stencil window from smem.  The
// arithmetic is operation for operation that of loop2d_kernel.
#include "kernels.cuh"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace sfdb200 {
namespace {

// Threads per CTA and rows per thread strip: 768 x 4 for forward / adjoint
// (more warps to hide the shared-memory and FFMA2 latencies of the short
// per-step chains), 512 x 8 for the gradient (its per-point registers).
template <bool GRAD> struct Shape { static constexpr int NT = GRAD ? 512 : 768, NZ = GRAD ? 8 : 4; };
constexpr int kMaxR = 4;      // register windows sized for so <= 8

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 ld2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void st2(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }

__device__ __forceinline__ void cluster_barrier() {
    asm volatile(
        "barrier.cluster.arrive.release.aligned;\n"
        "barrier.cluster.wait.acquire.aligned;\n" ::
            : "memory");
}

// n floats (n % 4 == 0, 16-byte aligned) from src to dst by the whole CTA.
__device__ __forceinline__ void copy4(float* dst, const float* src, int n) {
    const float4* s = reinterpret_cast<const float4*>(src);
    float4* d = reinterpret_cast<float4*>(dst);
    for (int i = threadIdx.x; i < n / 4; i += blockDim.x) d[i] = s[i];
}

template <int R, bool GRAD>
__global__ void __launch_bounds__(Shape<GRAD>::NT, 1) cluster2d_kernel(const Cluster2dArgs a) {
    constexpr int kThreads = Shape<GRAD>::NT, kNZ = Shape<GRAD>::NZ;
    cg::cluster_group cl = cg::this_cluster();
    const int c = static_cast<int>(cl.block_rank());
    const int tid = threadIdx.x;
    const int XP = a.XP;
    int zb, ze;
    cluster2d_band(a.Pz, R, a.nc, c, &zb, &ze);
    const int nb = ze - zb;
    const int sslot = (a.nbmax + 2 * R) * XP;  // floats per time slot (band + halo rows)
    extern __shared__ __align__(16) float sm[];
    float* gcorr = sm + 3 * sslot;              // GRAD: injection terms of the gradient
    const int ntot = 3 * sslot + (GRAD ? a.nbmax * XP : 0);
    for (int i = tid; i < ntot / 4; i += kThreads)
        reinterpret_cast<float4*>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);

    // Stage this CTA's sparse tables (soff, coef, pt, gm | soff[4], w[4], pt).
    const int ib = a.inj_n ? a.inj_begin[c] : 0, ie = a.inj_n ? a.inj_begin[c + 1] : 0;
    const int sb = a.smp_n ? a.smp_begin[c] : 0, se = a.smp_n ? a.smp_begin[c + 1] : 0;
    int* si = reinterpret_cast<int*>(sm + ntot);             // [inj_cap][4]
    int* ss = si + 4 * a.inj_cap;                             // [smp_cap][9]
    const int ni = min(ie - ib, a.inj_cap), nsm = min(se - sb, a.smp_cap);
    for (int e = tid; e < ni; e += kThreads) {
        si[4 * e] = a.inj_soff[ib + e];
        si[4 * e + 1] = __float_as_int(a.inj_coef[ib + e]);
        si[4 * e + 2] = a.inj_pt[ib + e];
        si[4 * e + 3] = GRAD ? a.inj_gm[ib + e] : 0;
    }
    for (int e = tid; e < nsm; e += kThreads) {
        for (int q = 0; q < 4; ++q) {
            ss[9 * e + q] = a.smp_soff[4 * (sb + e) + q];
            ss[9 * e + 4 + q] = __float_as_int(a.smp_w[4 * (sb + e) + q]);
        }
        ss[9 * e + 8] = a.smp_pt[sb + e];
    }

    // This thread's column pair and row strip; halo / pad columns get zero
    // coefficients, so their update is exactly 0 (as in the 3-D kernels).
    const int xa = R & ~1;
    const int npairs = (a.Px - R - xa + 1) / 2;
    const int ns = (nb + kNZ - 1) / kNZ;
    const bool active = tid < npairs * ns;
    const int x = xa + 2 * (active ? tid % npairs : 0);
    const int rb0 = (active ? tid / npairs : 0) * kNZ;
    const int nzr = active ? min(kNZ, nb - rb0) : 0;
    const bool vx0 = x >= R && x < a.Px - R, vx1 = x + 1 >= R && x + 1 < a.Px - R;
    float2 c1[kNZ], c2[kNZ], prev[kNZ], g[kNZ], utv[kNZ];
#pragma unroll
    for (int j = 0; j < kNZ; ++j) {
        c1[j] = c2[j] = prev[j] = g[j] = utv[j] = f2(0.f, 0.f);
        if (j < nzr) {
            const long long o = static_cast<long long>(zb + rb0 + j) * XP + x;
            c1[j] = f2(vx0 ? __ldg(a.c1 + o) : 0.f, vx1 ? __ldg(a.c1 + o + 1) : 0.f);
            c2[j] = f2(vx0 ? __ldg(a.c2 + o) : 0.f, vx1 ? __ldg(a.c2 + o + 1) : 0.f);
        }
    }
    float2 wk[R + 1];
#pragma unroll
    for (int k = 0; k <= R; ++k) wk[k] = f2(a.w[k], a.w[k]);
    const float2 neg2nd = f2(a.neg2nd, a.neg2nd);
    const float2 nidt2 = f2(a.nidt2, a.nidt2);
    const float2 mone = f2(-1.f, -1.f);

    const bool fwd = a.kind == 0;
    const long steps = a.nt > 2 ? a.nt - 2 : 0;
    float* up = c > 0 ? cl.map_shared_rank(sm, c - 1) : nullptr;
    float* dn = c < a.nc - 1 ? cl.map_shared_rank(sm, c + 1) : nullptr;
    int zb_up = 0, ze_up = 0;
    if (c > 0) cluster2d_band(a.Pz, R, a.nc, c - 1, &zb_up, &ze_up);
    // rows this CTA writes back: its band, plus the global halo rows at the ends
    const int wr0 = c == 0 ? 0 : R, wr1 = R + nb + (c == a.nc - 1 ? R : 0);
    const int grow0 = zb - R;  // global row of smem row 0

    if constexpr (GRAD) {
        if (steps > 0 && nzr > 0) {
            const float* ut = a.ut + (a.nt - 1) * a.slot;
#pragma unroll
            for (int j = 0; j < kNZ; ++j)
                if (j < nzr) utv[j] = __ldg(reinterpret_cast<const float2*>(
                                 ut + static_cast<long long>(zb + rb0 + j) * XP + x));
        }
    }
    __syncthreads();
    cluster_barrier();  // every CTA zeroed before the first halo push

    constexpr int WL = (R + 1) & ~1;
    for (long i = 0; i < steps; ++i) {
        const long t = fwd ? 2 + i : a.nt - 1 - i;
        const int r0 = static_cast<int>(t % 3);
        const int r1 = static_cast<int>(fwd ? (t - 1) % 3 : (t + 1) % 3);
        float* out = sm + r0 * sslot;
        const float* u1 = sm + r1 * sslot;
        // The first injection entry of this thread: its trace sample (and u_t)
        // are loaded now so the global latency hides behind the sweep.
        const long irow = fwd ? t - 1 : t;
        float tv = 0.f, uv = 0.f;
        if (tid < ni) {
            tv = __ldg(a.inj_trace + irow * a.inj_n + si[4 * tid + 2]);
            if constexpr (GRAD)
                if (si[4 * tid + 3]) uv = __ldg(a.ut + t * a.slot + a.inj_goff[ib + tid]);
        }
        if (nzr > 0) {
            float2 zw[kNZ + 2 * R];  // u1 column pair, rows rb0 - R .. rb0 + kNZ + R - 1
#pragma unroll
            for (int m = 0; m < kNZ + 2 * R; ++m)
                zw[m] = m < nzr + 2 * R ? ld2(u1 + (rb0 + m) * XP + x) : f2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < kNZ; ++j) {
                if (j < nzr) {
                    const float* row = u1 + (rb0 + j + R) * XP + x;
                    float w[2 * WL + 2];
#pragma unroll
                    for (int m = 0; m <= WL; ++m) {
                        const float2 v = ld2(row - WL + 2 * m);
                        w[2 * m] = v.x;
                        w[2 * m + 1] = v.y;
                    }
                    const float2 c0 = zw[j + R];
                    float2 lap = f2(0.f, 0.f);
#pragma unroll
                    for (int k = 1; k <= R; ++k) {
                        // misaligned pairs: two scalar adds (same rounding) instead of
                        // re-pairing moves + one packed add, as in the 3-D pair sweep
                        const float2 xs = ((WL - k) & 1)
                                              ? f2(__fadd_rn(w[WL - k], w[WL + k]),
                                                   __fadd_rn(w[WL - k + 1], w[WL + k + 1]))
                                              : add2(f2(w[WL - k], w[WL - k + 1]),
                                                     f2(w[WL + k], w[WL + k + 1]));
                        const float2 zs = add2(zw[j + R - k], zw[j + R + k]);
                        float2 s = add2(xs, zs);
                        s = fma2(neg2nd, c0, s);
                        lap = fma2(wk[k], s, lap);
                    }
                    const float2 d = fma2(prev[j], mone, c0);
                    const float2 inc = fma2(c1[j], d, mul2(c2[j], lap));
                    st2(out + (rb0 + j + R) * XP + x, add2(c0, inc));
                    if constexpr (GRAD) g[j] = fma2(mul2(nidt2, utv[j]), fma2(d, mone, inc), g[j]);
                    prev[j] = c0;
                }
            }
        }
        __syncthreads();
        if (ie > ib) {  // inject (codegen.cpp:436-449), collisions by shared atomics
            if (tid < ni) {
                const float delta = __int_as_float(si[4 * tid + 1]) * tv;
                atomicAdd(out + si[4 * tid], delta);
                if constexpr (GRAD)
                    if (si[4 * tid + 3])
                        atomicAdd(gcorr + si[4 * tid] - R * XP, a.nidt2 * uv * delta);
            }
            const float* ut = GRAD ? a.ut + t * a.slot : nullptr;
            for (int e = ib + ni + tid; e < ie; e += kThreads) {  // beyond the staged ones
                const float delta = a.inj_coef[e] * __ldg(a.inj_trace + irow * a.inj_n + a.inj_pt[e]);
                atomicAdd(out + a.inj_soff[e], delta);
                if constexpr (GRAD)
                    if (a.inj_gm[e])
                        atomicAdd(gcorr + a.inj_soff[e] - R * XP,
                                  a.nidt2 * __ldg(ut + a.inj_goff[e]) * delta);
            }
            __syncthreads();
        }
        // Edge rows into the neighbours' halo rows of the same slot.
        if (up) copy4(up + r0 * sslot + (ze_up - zb_up + R) * XP, out + R * XP, R * XP);
        if (dn) copy4(dn + r0 * sslot, out + nb * XP, R * XP);
        if (a.save)  // forward history row t (codegen.cpp save_every = 1)
            copy4(a.hist + t * a.slot + static_cast<long long>(grow0 + wr0) * XP,
                  out + wr0 * XP, (wr1 - wr0) * XP);
        if constexpr (GRAD) {
            if (i + 1 < steps && nzr > 0) {  // u_t of the next (earlier) step
                const float* ut = a.ut + (t - 1) * a.slot;
#pragma unroll
                for (int j = 0; j < kNZ; ++j)
                    if (j < nzr) utv[j] = __ldg(reinterpret_cast<const float2*>(
                                     ut + static_cast<long long>(zb + rb0 + j) * XP + x));
            }
        }
        cluster_barrier();
        if (se > sb) {  // sample (codegen.cpp:450-458), corners summed in order
            const long srow = fwd ? t : t - 1;
            for (int e = tid; e < se - sb; e += kThreads) {
                float acc = 0.f;
                if (e < nsm) {
                    const int* q9 = ss + 9 * e;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        acc = fmaf(__int_as_float(q9[4 + q]), out[q9[q]], acc);
                    a.smp_trace[srow * a.smp_n + q9[8]] = acc;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        acc = fmaf(__ldg(a.smp_w + 4 * (sb + e) + q), out[a.smp_soff[4 * (sb + e) + q]], acc);
                    a.smp_trace[srow * a.smp_n + a.smp_pt[sb + e]] = acc;
                }
            }
        }
    }
    if (!a.save)
        for (int r = 0; r < 3; ++r)
            copy4(a.field + r * a.slot + static_cast<long long>(grow0 + wr0) * XP,
                  sm + r * sslot + wr0 * XP, (wr1 - wr0) * XP);
    if constexpr (GRAD) {
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kNZ; ++j) {
            if (j < nzr) {
                const long long o = static_cast<long long>(zb + rb0 + j) * XP + x;
                const float* gc = gcorr + (rb0 + j) * XP + x;
                if (vx0) a.grad[o] = g[j].x + gc[0];
                if (vx1) a.grad[o + 1] = g[j].y + gc[1];
            }
        }
    }
}

// query: report whether one such cluster can be resident instead of launching.
template <int R, bool GRAD>
cudaError_t launch_t(const Cluster2dArgs& a, cudaStream_t s, bool query) {
    auto kern = cluster2d_kernel<R, GRAD>;
    const size_t smem = cluster2d_smem_bytes(a.Pz, a.XP, R, a.nc, GRAD) +
                        static_cast<size_t>(a.inj_cap) * kCluster2dInjBytes +
                        static_cast<size_t>(a.smp_cap) * kCluster2dSmpBytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(a.nc);
    lc.blockDim = dim3(Shape<GRAD>::NT);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = a.nc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if (query) {
        int n = 0;
        e = cudaOccupancyMaxActiveClusters(&n, kern, &lc);
        return e != cudaSuccess ? e : (n > 0 ? cudaSuccess : cudaErrorInvalidConfiguration);
    }
    return cudaLaunchKernelEx(&lc, kern, a);
}

cudaError_t dispatch(const Cluster2dArgs& a, int R, bool grad, cudaStream_t s, bool query) {
#define SFDB_R_CASE(RR) \
    case RR:            \
        return grad ? launch_t<RR, true>(a, s, query) : launch_t<RR, false>(a, s, query);
    switch (R) {
        SFDB_R_CASE(1)
        SFDB_R_CASE(2)
        SFDB_R_CASE(3)
        SFDB_R_CASE(4)
        default:
            return cudaErrorInvalidValue;
    }
#undef SFDB_R_CASE
}

}  // namespace

size_t cluster2d_smem_bytes(int Pz, int XP, int R, int nc, bool grad) {
    const int nz = Pz - 2 * R, nbmax = (nz + nc - 1) / nc;
    return (3 * static_cast<size_t>(nbmax + 2 * R) + (grad ? nbmax : 0)) * XP * 4;
}

int cluster2d_ctas(int Pz, int Px, int XP, int R, bool grad) {
    if (R < 1 || R > kMaxR) return 0;
    const int nz = Pz - 2 * R;
    const int xa = R & ~1, npairs = (Px - R - xa + 1) / 2;
    for (int nc = 16; nc >= 2; --nc) {
        const int nbmax = (nz + nc - 1) / nc;
        if (nz / nc < R) continue;  // every band must cover the R rows it pushes
        const int NT = grad ? Shape<true>::NT : Shape<false>::NT;
        const int NZ = grad ? Shape<true>::NZ : Shape<false>::NZ;
        if (npairs * ((nbmax + NZ - 1) / NZ) > NT) continue;
        if (cluster2d_smem_bytes(Pz, XP, R, nc, grad) > kCluster2dSmemMax) continue;
        Cluster2dArgs q{};
        q.Pz = Pz;
        q.Px = Px;
        q.XP = XP;
        q.nc = nc;
        q.nbmax = nbmax;
        if (dispatch(q, R, grad, nullptr, true) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        return nc;
    }
    return 0;
}

cudaError_t launch_cluster2d(const Cluster2dArgs& a, int R, bool grad, cudaStream_t s) {
    return dispatch(a, R, grad, s, false);
}

}  // namespace sfdb200
