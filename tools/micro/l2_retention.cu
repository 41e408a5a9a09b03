// How much of the most recently touched data does the B200 L2 still hold after
// a streaming pass over buffers much larger than L2?  Kernel 1 copies A -> B
// front to back (N MB each); kernel 2 re-reads the last M MB of A and of B.
// Time of kernel 2 vs M, for default cache policy and for evict_last hints on
// the tail of kernel 1 (evict_first on the rest).  Timing only.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_retention l2_retention.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 ld_hint(const float4* p, unsigned long long pol) {
    float4 v;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_hint(float4* p, float4 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

// mode 0: plain ld/st; 1: evict_last on the last `tail` float4s, evict_first before;
// 2: evict_last on the tail, plain before
__global__ void stream_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n,
                              size_t tail, int mode) {
    unsigned long long plast, pfirst, pnorm;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(plast));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pfirst));
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pnorm));
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (mode == 0) {
            float4 v = a[i];
            v.x += 1.0f;
            b[i] = v;
        } else {
            const unsigned long long pol = i >= n - tail ? plast : (mode == 1 ? pfirst : pnorm);
            float4 v = ld_hint(a + i, pol);
            v.x += 1.0f;
            st_hint(b + i, v, pol);
        }
    }
}

// re-reads the last m float4s of a and b, back to front; mode != 0: evict_first
__global__ void reread_kernel(const float4* __restrict__ a, const float4* __restrict__ b, size_t n,
                              size_t m, float* sink, int mode) {
    unsigned long long pfirst;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pfirst));
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    float acc = 0.0f;
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += stride) {
        const size_t i = n - 1 - k;
        float4 x, y;
        if (mode == 0) { x = a[i]; y = b[i]; }
        else { x = ld_hint(a + i, pfirst); y = ld_hint(b + i, pfirst); }
        acc += x.x + y.y;
    }
    if (acc == 12345.678f) *sink = acc;
}

int main(int argc, char** argv) {
    const size_t MB = 1 << 20;
    const size_t nbytes = (argc > 1 ? atol(argv[1]) : 400) * MB;  // per buffer
    const size_t n = nbytes / 16;
    float4 *a, *b;
    float* sink;
    cudaMalloc(&a, nbytes);
    cudaMalloc(&b, nbytes);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 0, nbytes);
    cudaMemset(b, 0, nbytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 148 * 8, block = 256;
    for (int mode = 0; mode < 3; ++mode)
        for (size_t mmb : {4, 8, 16, 24, 32, 48, 64, 96}) {
            const size_t m = mmb * MB / 16;  // per buffer
            float best = 1e9f, cold = 1e9f;
            for (int rep = 0; rep < 6; ++rep) {
                stream_kernel<<<grid, block>>>(a, b, n, m, mode);
                cudaEventRecord(e0);
                reread_kernel<<<grid, block>>>(a, b, n, m, sink, mode);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep) best = ms < best ? ms : best;
                // cold: re-read the FIRST m (long evicted) for comparison
                stream_kernel<<<grid, block>>>(a, b, n, m, mode);
                cudaEventRecord(e0);
                reread_kernel<<<grid, block>>>(a, b, m, m, sink, mode);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep) cold = ms < cold ? ms : cold;
            }
            printf("{\"mode\": %d, \"buffer_mb\": %zu, \"tail_mb_per_buffer\": %zu, \"reread_us\": %.2f, "
                   "\"reread_cold_us\": %.2f, \"hot_GBps\": %.0f, \"cold_GBps\": %.0f}\n",
                   mode, nbytes / MB, mmb, best * 1e3, cold * 1e3, 2.0 * mmb * MB / (best * 1e-3) / 1e9,
                   2.0 * mmb * MB / (cold * 1e-3) / 1e9);
        }
    return 0;
}
