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

#include <algorithm>
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

// Helper threads inherit the caller's CPU binding (an OpenMP runtime started
// with OMP_PROC_BIND pins the initial thread to one core, e.g. under bench.py
// or the reference's own OpenMP kernels), which would put every helper on that
// core; they widen their own mask to every CPU id (the kernel intersects it
// with the process's cpuset, whose ids need not start at 0).
void unbind_self() {
    const long n = std::max<long>(1024, sysconf(_SC_NPROCESSORS_CONF));
    cpu_set_t* set = CPU_ALLOC(n);
    const size_t sz = CPU_ALLOC_SIZE(n);
    CPU_ZERO_S(sz, set);
    for (long c = 0; c < n; ++c) CPU_SET_S(c, sz, set);
    pthread_setaffinity_np(pthread_self(), sz, set);
    CPU_FREE(set);
}

void par_memcpy(void* dst, const void* src, size_t n) {
    const size_t t = std::min<size_t>(copy_threads(), std::max<size_t>(1, n >> 22));
    if (t <= 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    const size_t per = (n + t - 1) / t;
    for (size_t i = 1; i < t; ++i) {
        const size_t o = i * per;
        if (o >= n) break;
        th.emplace_back([=] {
            unbind_self();
            std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                        std::min(per, n - o));
        });
    }
    std::memcpy(dst, src, std::min(per, n));
    for (auto& x : th) x.join();
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

void release_pinned(sfdb200_plan& p) {
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
