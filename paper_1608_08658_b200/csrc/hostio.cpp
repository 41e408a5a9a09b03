// Host <-> device copies of the caller's buffers (the reference's argv arrays).
//
// Page-locked host memory goes straight to cudaMemcpyAsync.  Pageable memory
// -- what the reference's std::vector buffers are -- would make the driver
// stage it through its own small pinned buffers one piece at a time (measured
// on cfg2: 10.7 GB/s up, 21 GB/s down).  Here it is staged through two pinned
// chunks per plan: a few host threads fill (or drain) one chunk while the DMA
// of the other runs, so the copy runs near the PCIe rate instead.
#include <pthread.h>
#include <sched.h>
#include <unistd.h>

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "plan.hpp"

namespace sfdb200 {
namespace {

constexpr size_t kChunk = 32u << 20;  // bytes per pinned staging chunk

// memcpy split over a few host threads (one for small copies).
unsigned copy_threads() {
    static const unsigned t = [] {
        if (const char* e = std::getenv("SFDB200_COPY_THREADS")) return std::max(1, std::atoi(e));
        return static_cast<int>(std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2)));
    }();
    return t;
}

// Helper threads inherit the calling thread's CPU binding (an OpenMP runtime
// started with OMP_PROC_BIND pins the initial thread to one core, e.g. under
// bench.py or the reference's own OpenMP kernels), which would put every
// helper on that core.  They take instead the mask the process had when this
// library was loaded (before any such binding): a caller's taskset / numactl
// / per-rank NUMA binding stays in force.
struct ProcessMask {
    cpu_set_t* set = nullptr;
    size_t size = 0;
    ProcessMask() {
        const long n = std::max<long>(1024, sysconf(_SC_NPROCESSORS_CONF));
        set = CPU_ALLOC(n);
        size = CPU_ALLOC_SIZE(n);
        if (sched_getaffinity(0, size, set) != 0) {
            CPU_FREE(set);
            set = nullptr;
        }
    }
};
const ProcessMask g_process_mask;  // initialised when the library loads

void unbind_self() {
    if (g_process_mask.set)
        pthread_setaffinity_np(pthread_self(), g_process_mask.size, g_process_mask.set);
}

// f(begin, end) over [0, n) split across the copy threads (one for small n).
template <class F>
void par_range(size_t n, size_t bytes, F&& f) {
    const size_t t = std::min<size_t>(copy_threads(), std::max<size_t>(1, bytes >> 22));
    if (t <= 1) {
        f(size_t{0}, n);
        return;
    }
    std::vector<std::thread> th;
    const size_t per = (n + t - 1) / t;
    for (size_t i = 1; i < t; ++i) {
        const size_t o = i * per;
        if (o >= n) break;
        th.emplace_back([&, o] {
            unbind_self();
            f(o, std::min(n, o + per));
        });
    }
    f(size_t{0}, std::min(per, n));
    for (auto& x : th) x.join();
}

void par_memcpy(void* dst, const void* src, size_t n) {
    par_range(n, n, [&](size_t b, size_t e) {
        std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b);
    });
}

// The conversion loops, vectorised for the host's ISA (resolved at load).
// The destinations are written with non-temporal stores: they are not read
// again here, and plain stores would first read every line for ownership
// (on the measured box the pageable copies are host-memory-bound).
__attribute__((target("avx512f"))) bool narrow_avx512(float* __restrict__ dst,
                                                       const double* __restrict__ src, size_t n) {
    size_t i = 0;
    unsigned bad = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31); ++i) {
        const float f = static_cast<float>(src[i]);
        dst[i] = f;
        bad |= static_cast<double>(f) != src[i];
    }
    __mmask8 acc = 0;
    for (; i + 8 <= n; i += 8) {
        const __m512d v = _mm512_loadu_pd(src + i);
        const __m256 f = _mm512_cvtpd_ps(v);
        _mm256_stream_ps(dst + i, f);
        acc |= _mm512_cmp_pd_mask(_mm512_cvtps_pd(f), v, _CMP_NEQ_UQ);  // NaN included
    }
    for (; i < n; ++i) {
        const float f = static_cast<float>(src[i]);
        dst[i] = f;
        bad |= static_cast<double>(f) != src[i];
    }
    _mm_sfence();
    return bad != 0 || acc != 0;
}

__attribute__((target("avx512f"))) void widen_avx512(double* __restrict__ dst,
                                                      const float* __restrict__ src, size_t n) {
    size_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 63); ++i)
        dst[i] = static_cast<double>(src[i]);
    for (; i + 8 <= n; i += 8) _mm512_stream_pd(dst + i, _mm512_cvtps_pd(_mm256_loadu_ps(src + i)));
    for (; i < n; ++i) dst[i] = static_cast<double>(src[i]);
    _mm_sfence();
}

__attribute__((target("avx2"))) bool narrow_avx2(float* __restrict__ dst,
                                                  const double* __restrict__ src, size_t n) {
    size_t i = 0;
    unsigned bad = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 15); ++i) {
        const float f = static_cast<float>(src[i]);
        dst[i] = f;
        bad |= static_cast<double>(f) != src[i];
    }
    __m256d acc = _mm256_setzero_pd();
    for (; i + 4 <= n; i += 4) {
        const __m256d v = _mm256_loadu_pd(src + i);
        const __m128 f = _mm256_cvtpd_ps(v);
        _mm_stream_ps(dst + i, f);
        acc = _mm256_or_pd(acc, _mm256_cmp_pd(_mm256_cvtps_pd(f), v, _CMP_NEQ_UQ));
    }
    for (; i < n; ++i) {
        const float f = static_cast<float>(src[i]);
        dst[i] = f;
        bad |= static_cast<double>(f) != src[i];
    }
    _mm_sfence();
    return bad != 0 || _mm256_movemask_pd(acc) != 0;
}

__attribute__((target("avx2"))) void widen_avx2(double* __restrict__ dst,
                                                 const float* __restrict__ src, size_t n) {
    size_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31); ++i)
        dst[i] = static_cast<double>(src[i]);
    for (; i + 4 <= n; i += 4) _mm256_stream_pd(dst + i, _mm256_cvtps_pd(_mm_loadu_ps(src + i)));
    for (; i < n; ++i) dst[i] = static_cast<double>(src[i]);
    _mm_sfence();
}

bool narrow_scalar(float* __restrict__ dst, const double* __restrict__ src, size_t n) {
    unsigned bad = 0;
    for (size_t i = 0; i < n; ++i) {
        const float f = static_cast<float>(src[i]);
        dst[i] = f;
        bad |= static_cast<double>(f) != src[i];
    }
    return bad != 0;
}

void widen_scalar(double* __restrict__ dst, const float* __restrict__ src, size_t n) {
    for (size_t i = 0; i < n; ++i) dst[i] = static_cast<double>(src[i]);
}

int host_isa() {  // 2 = AVX-512F, 1 = AVX2, 0 = baseline
    static const int isa = __builtin_cpu_supports("avx512f") ? 2
                            : __builtin_cpu_supports("avx2") ? 1
                                                             : 0;
    return isa;
}

bool narrow_block(float* dst, const double* src, size_t n) {
    switch (host_isa()) {
        case 2: return narrow_avx512(dst, src, n);
        case 1: return narrow_avx2(dst, src, n);
        default: return narrow_scalar(dst, src, n);
    }
}

void widen_block(double* dst, const float* src, size_t n) {
    switch (host_isa()) {
        case 2: widen_avx512(dst, src, n); break;
        case 1: widen_avx2(dst, src, n); break;
        default: widen_scalar(dst, src, n);
    }
}

// fp64 -> fp32 (round to nearest); exact: report whether every value survives.
bool par_narrow(float* dst, const double* src, size_t n, bool exact) {
    std::atomic<bool> bad{false};
    par_range(n, n * 8, [&](size_t b, size_t e) {
        if (narrow_block(dst + b, src + b, e - b) && exact)
            bad.store(true, std::memory_order_relaxed);
    });
    return !bad.load();
}

void par_widen(double* dst, const float* src, size_t n) {
    par_range(n, n * 8, [&](size_t b, size_t e) { widen_block(dst + b, src + b, e - b); });
}

void ensure_pinned(sfdb200_plan& p) {
    if (p.pin[0]) return;
    for (int b = 0; b < 2; ++b) {
        ck(cudaHostAlloc(&p.pin[b], kChunk, cudaHostAllocDefault), "cudaHostAlloc");
        ck(cudaEventCreateWithFlags(&p.pin_ev[b], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventRecord(p.pin_ev[b], p.stream), "event");
    }
}

}  // namespace

bool host_pinned(const void* ptr) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void copy_h2d(sfdb200_plan& p, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    if (bytes < (1u << 20) || host_pinned(src)) {
        ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, p.stream), "H2D");
        return;
    }
    ensure_pinned(p);
    for (size_t o = 0, k = 0; o < bytes; o += kChunk, ++k) {
        const int b = static_cast<int>(k & 1);
        const size_t n = std::min(kChunk, bytes - o);
        ck(cudaEventSynchronize(p.pin_ev[b]), "H2D staging");  // its previous DMA is done
        par_memcpy(p.pin[b], static_cast<const char*>(src) + o, n);
        ck(cudaMemcpyAsync(static_cast<char*>(dst) + o, p.pin[b], n, cudaMemcpyHostToDevice,
                           p.stream),
           "H2D");
        ck(cudaEventRecord(p.pin_ev[b], p.stream), "event");
    }
}

void copy_d2h(sfdb200_plan& p, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    if (bytes < (1u << 20) || host_pinned(dst)) {
        ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, p.stream), "D2H");
        return;
    }
    ensure_pinned(p);
    const size_t chunks = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t k) {
        const int b = static_cast<int>(k & 1);
        const size_t o = k * kChunk, n = std::min(kChunk, bytes - o);
        ck(cudaMemcpyAsync(p.pin[b], static_cast<const char*>(src) + o, n,
                           cudaMemcpyDeviceToHost, p.stream),
           "D2H");
        ck(cudaEventRecord(p.pin_ev[b], p.stream), "event");
    };
    issue(0);
    if (chunks > 1) issue(1);
    for (size_t k = 0; k < chunks; ++k) {
        const int b = static_cast<int>(k & 1);
        const size_t o = k * kChunk, n = std::min(kChunk, bytes - o);
        ck(cudaEventSynchronize(p.pin_ev[b]), "D2H staging");
        par_memcpy(static_cast<char*>(dst) + o, p.pin[b], n);
        if (k + 2 < chunks) issue(k + 2);
    }
}

bool copy_h2d_narrow(sfdb200_plan& p, float* dst, const double* src, size_t count, bool exact) {
    if (count == 0) return true;
    ensure_pinned(p);
    constexpr size_t per = kChunk / sizeof(float);
    for (size_t o = 0, k = 0; o < count; o += per, ++k) {
        const int b = static_cast<int>(k & 1);
        const size_t n = std::min(per, count - o);
        ck(cudaEventSynchronize(p.pin_ev[b]), "H2D staging");  // its previous DMA is done
        if (!par_narrow(static_cast<float*>(p.pin[b]), src + o, n, exact)) return false;
        ck(cudaMemcpyAsync(dst + o, p.pin[b], n * sizeof(float), cudaMemcpyHostToDevice,
                           p.stream),
           "H2D");
        ck(cudaEventRecord(p.pin_ev[b], p.stream), "event");
    }
    return true;
}

void copy_d2h_widen(sfdb200_plan& p, double* dst, const float* src, size_t count) {
    if (count == 0) return;
    ensure_pinned(p);
    constexpr size_t per = kChunk / sizeof(float);
    const size_t chunks = (count + per - 1) / per;
    auto issue = [&](size_t k) {
        const int b = static_cast<int>(k & 1);
        const size_t o = k * per, n = std::min(per, count - o);
        ck(cudaMemcpyAsync(p.pin[b], src + o, n * sizeof(float), cudaMemcpyDeviceToHost,
                           p.stream),
           "D2H");
        ck(cudaEventRecord(p.pin_ev[b], p.stream), "event");
    };
    issue(0);
    if (chunks > 1) issue(1);
    for (size_t k = 0; k < chunks; ++k) {
        const int b = static_cast<int>(k & 1);
        const size_t o = k * per, n = std::min(per, count - o);
        ck(cudaEventSynchronize(p.pin_ev[b]), "D2H staging");
        par_widen(dst + o, static_cast<const float*>(p.pin[b]), n);
        if (k + 2 < chunks) issue(k + 2);
    }
}

// The reference's damping (build_damping, seismic.cpp:152-173) is
// max(dz[z], dy[y], dx[x]), zero in the interior.  Candidate profiles are the
// three lines through the smallest cells found from the grid centre (one
// argmin per axis); the whole field is then compared with max(A[z], B[y],
// C[x]) bit for bit, split over host threads, while the DMA of m runs.  When
// the identity holds the lines ARE the per-axis minima the device check
// extracts (a line through a cell where all three profiles are minimal is the
// min profile of a separable field), so only the lines are uploaded.  Any
// other field -- negative, NaN, perturbed cells, signed zeros on the lines, or
// separable with its minima away from the centre lines (the argmin search
// stops at ties) -- returns false and takes the device path.
bool host_sep_damp(const double* d, long long Pz, long long Py, long long Px,
                   std::vector<double>& prof) {
    if (Pz < 1 || Py < 1 || Px < 1) return false;
    auto at = [&](long long z, long long y, long long x) { return d[(z * Py + y) * Px + x]; };
    auto argmin = [](long long n, auto&& f) {
        long long k = 0;
        for (long long i = 1; i < n; ++i)
            if (f(i) < f(k)) k = i;
        return k;
    };
    long long yc = Py / 2, xc = Px / 2;
    const long long zc = argmin(Pz, [&](long long z) { return at(z, yc, xc); });
    yc = argmin(Py, [&](long long y) { return at(zc, y, xc); });
    xc = argmin(Px, [&](long long x) { return at(zc, yc, x); });
    prof.resize(static_cast<size_t>(Pz + Py + Px));
    double* A = prof.data();
    double* B = A + Pz;
    double* C = B + Py;
    for (long long z = 0; z < Pz; ++z) A[z] = at(z, yc, xc);
    for (long long y = 0; y < Py; ++y) B[y] = at(zc, y, xc);
    for (long long x = 0; x < Px; ++x) C[x] = at(zc, yc, x);
    for (const double v : prof)
        if (!(v >= 0.0) || std::signbit(v)) return false;

    const unsigned t = static_cast<unsigned>(
        std::min<long long>(Pz, std::max(1u, std::thread::hardware_concurrency())));
    std::atomic<bool> bad{false};
    auto check = [&](long long z0, long long z1) {
        for (long long z = z0; z < z1 && !bad.load(std::memory_order_relaxed); ++z)
            for (long long y = 0; y < Py; ++y) {
                const double rzy = std::max(A[z], B[y]);
                const double* row = d + (z * Py + y) * Px;
                bool ok = true;
                for (long long x = 0; x < Px; ++x) {
                    const double v = row[x];
                    ok &= (v == std::max(rzy, C[x])) & (v >= 0.0);
                }
                if (!ok) {
                    bad.store(true, std::memory_order_relaxed);
                    return;
                }
            }
    };
    std::vector<std::thread> th;
    const long long per = (Pz + t - 1) / t;
    for (unsigned i = 1; i < t; ++i) {
        const long long z0 = i * per;
        if (z0 >= Pz) break;
        th.emplace_back([=, &check] {
            unbind_self();
            check(z0, std::min(Pz, z0 + per));
        });
    }
    check(0, std::min(Pz, per));
    for (auto& x : th) x.join();
    return !bad.load();
}

namespace {
struct HostCopy {
    void* dst;
    const void* src;
    size_t n;
};
void CUDART_CB host_copy(void* arg) {  // a stream host function: no CUDA calls
    auto* j = static_cast<HostCopy*>(arg);
    par_memcpy(j->dst, j->src, j->n);
    delete j;
}
struct HostWiden {
    double* dst;
    const float* src;
    size_t n;
};
void CUDART_CB host_widen(void* arg) {
    auto* j = static_cast<HostWiden*>(arg);
    par_widen(j->dst, j->src, j->n);
    delete j;
}
}  // namespace

void copy_d2h_stream_widen(sfdb200_plan& p, double* dst, const float* src, size_t count,
                           cudaStream_t s) {
    for (int b = 0; b < 2; ++b)
        if (!p.xpin[b]) ck(cudaHostAlloc(&p.xpin[b], kChunk, cudaHostAllocDefault), "cudaHostAlloc");
    constexpr size_t per = kChunk / sizeof(float);
    for (size_t o = 0; o < count; o += per) {
        const int b = p.xpin_next;
        p.xpin_next ^= 1;
        const size_t n = std::min(per, count - o);
        // chunk b's previous host function precedes this copy in stream order
        ck(cudaMemcpyAsync(p.xpin[b], src + o, n * sizeof(float), cudaMemcpyDeviceToHost, s),
           "D2H");
        ck(cudaLaunchHostFunc(s, host_widen,
                              new HostWiden{dst + o, static_cast<const float*>(p.xpin[b]), n}),
           "cudaLaunchHostFunc");
    }
}

void copy_d2h_stream_pageable(sfdb200_plan& p, void* dst, const void* src, size_t bytes,
                              cudaStream_t s) {
    for (int b = 0; b < 2; ++b)
        if (!p.xpin[b]) ck(cudaHostAlloc(&p.xpin[b], kChunk, cudaHostAllocDefault), "cudaHostAlloc");
    for (size_t o = 0; o < bytes; o += kChunk) {
        const int b = p.xpin_next;
        p.xpin_next ^= 1;
        const size_t n = std::min(kChunk, bytes - o);
        // chunk b's previous host function precedes this copy in stream order
        ck(cudaMemcpyAsync(p.xpin[b], static_cast<const char*>(src) + o, n,
                           cudaMemcpyDeviceToHost, s),
           "D2H");
        ck(cudaLaunchHostFunc(s, host_copy, new HostCopy{static_cast<char*>(dst) + o, p.xpin[b], n}),
           "cudaLaunchHostFunc");
    }
}

void release_pinned(sfdb200_plan& p) {
    if (p.xstream && (p.xpin[0] || p.xpin[1])) cudaStreamSynchronize(p.xstream);
    for (int b = 0; b < 2; ++b) {
        if (p.xpin[b]) cudaFreeHost(p.xpin[b]);
        p.xpin[b] = nullptr;
    }
    for (int b = 0; b < 2; ++b) {
        if (p.pin_ev[b]) {
            cudaEventSynchronize(p.pin_ev[b]);
            cudaEventDestroy(p.pin_ev[b]);
        }
        if (p.pin[b]) cudaFreeHost(p.pin[b]);
        p.pin[b] = nullptr;
        p.pin_ev[b] = nullptr;
    }
}

}  // namespace sfdb200

int sfdb200_damp_separable(const double* damp, long Pz, long Py, long Px, double* prof) {
    if (!damp || !prof || Pz < 1 || Py < 1 || Px < 1) return SFDB200_EINVAL;
    std::vector<double> p;
    const bool sep = sfdb200::host_sep_damp(damp, Pz, Py, Px, p);
    if (sep) std::memcpy(prof, p.data(), p.size() * sizeof(double));
    return sep ? 1 : 0;
}
