// Microbenchmark: cost per step of {__syncthreads; DSMEM edge push; cluster barrier}
// for a 16-CTA cluster (the 2-D cluster time loop's fixed per-step overhead).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void bench(int steps, int nfloat, long long* out) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) float sm[];
    const int c = cl.block_rank(), n = cl.num_blocks();
    float* up = c > 0 ? cl.map_shared_rank(sm, c - 1) : nullptr;
    float* dn = c < n - 1 ? cl.map_shared_rank(sm, c + 1) : nullptr;
    for (int i = threadIdx.x; i < 4 * nfloat; i += blockDim.x) sm[i] = 0.f;
    cl.sync();
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        __syncthreads();
        if (MODE >= 1) {
            const float4* src = reinterpret_cast<const float4*>(sm);
            if (up) for (int i = threadIdx.x; i < nfloat / 4; i += blockDim.x) reinterpret_cast<float4*>(up + 2 * nfloat)[i] = src[i];
            if (dn) for (int i = threadIdx.x; i < nfloat / 4; i += blockDim.x) reinterpret_cast<float4*>(dn + 3 * nfloat)[i] = src[i];
        }
        if (MODE == 2) {
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory");
        } else {
            asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[c] = t1 - t0;
}

int main() {
    long long* d;
    cudaMalloc(&d, 16 * sizeof(long long));
    for (int mode = 0; mode < 3; ++mode)
        for (int threads : {512, 1024}) {
            const int nfloat = 2 * 288;  // R = 2 rows of 288 floats
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(16);
            lc.blockDim = dim3(threads);
            lc.dynamicSmemBytes = 4 * nfloat * 4;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            lc.attrs = at; lc.numAttrs = 1;
            void (*k)(int, int, long long*) = mode == 0 ? bench<0> : (mode == 1 ? bench<1> : bench<2>);
            cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            const int steps = 10000;
            cudaLaunchKernelEx(&lc, k, steps, nfloat, d);
            cudaEventRecord(e0);
            cudaLaunchKernelEx(&lc, k, steps, nfloat, d);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            long long h[16]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            printf("mode %d (%s) threads %d: %.3f us/step, %lld cycles/step (CTA0), err=%s\n", mode,
                   mode == 0 ? "sync+barrier" : mode == 1 ? "sync+push+barrier(rel/acq)" : "sync+push+barrier(relaxed)",
                   threads, ms * 1e3 / steps, h[0] / steps, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
