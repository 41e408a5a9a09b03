// Fused P2P ghost exchange between z-slab ranks over NVLink.
//
// The NCCL path (comm.cpp) sweeps the R planes next to each neighbour in their
// own launches, then sends them with ncclSend/ncclRecv while the interior
// runs.  Here a step is ONE sweep launch whose first items are those boundary
// tiles (sweep3d.cuh, SweepArgs::nbi): each boundary item, after its planes
// and injections, re-sends its values through a CUDA IPC mapping of the
// neighbour's field straight into the neighbour's ghost planes of the same
// row (SweepArgs::pdelta), and the last boundary item publishes the step into
// the neighbours' counters (st.release.sys) while the interior items of the
// same launch keep running.  Ordering between the processes:
//
//   exec_begin:  zero rows -> signal B (cuStreamWriteValue32) -> wait >= B
//   step i:      wait >= B + i (one-thread poll kernel, GEQ) -> fused launch,
//                whose boundary items publish B + i + 1 to the neighbours
//   exec_end:    wait >= B + steps        (their last stores into my ghosts)
//
// B advances by steps + 1 per execute on every rank, so counters never reset.
// A neighbour can be at most one step ahead, and then writes the ghost planes
// of a row this rank no longer reads (row t % 3 while this rank reads row
// (t - 2) % 3 ghosts), so there is no write-after-read hazard.
#include <cuda.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>

#include "plan.hpp"

namespace sfdb200 {
namespace {

struct Blob {  // SFDB200_IPC_BYTES, plain bytes exchanged by the caller
    cudaIpcMemHandle_t field;
    cudaIpcMemHandle_t flags;
    int device;
    int pz;             // local planes
    long long slot;     // elements per row
    long long plane;    // elements per plane (y, x extents and pitch)
    int radius;
    int rank, world;
};
static_assert(sizeof(Blob) <= SFDB200_IPC_BYTES, "IPC blob too large");

typedef CUresult (*PFN_write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <class F>
F driver_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
        fail(SFDB200_ECUDA, std::string(name) + " is unavailable");
    return reinterpret_cast<F>(p);
}

}  // namespace

long long p2p_delta(const sfdb200_plan& p, int side, long long row) {
    const FieldGeom& g = p.g;
    const int R = g.R;
    // lower: my planes [R, 2R) -> its planes [Pz' - R, Pz'); upper: my planes
    // [Pz - 2R, Pz - R) -> its planes [0, R)
    const long long dplanes = side == 0 ? p.peer_pz[0] - 2LL * R : -(g.Pz - 2LL * R);
    const auto mine = reinterpret_cast<std::uintptr_t>(p.field + row * g.slot);
    const auto theirs = reinterpret_cast<std::uintptr_t>(p.peer_field[side] + row * p.peer_slot[side]) +
                        static_cast<std::uintptr_t>(dplanes * g.pz * 4);
    return static_cast<long long>(theirs - mine);
}

int p2p_boundary_items(const sfdb200_plan& p) {
    if (!p.dist() || !p.p2p || p.g.ndim != 3) return 0;
    return p.cfg.tiles_x * p.cfg.tiles_y * ((p.rank > 0 ? 1 : 0) + (p.rank < p.world - 1 ? 1 : 0));
}

void p2p_export(const sfdb200_plan& p, void* out) {
    if (!p.dist() || p.g.ndim != 3) fail(SFDB200_EINVAL, "P2P exchange needs a 3-D z-slab plan");
    Blob b{};
    ck(cudaIpcGetMemHandle(&b.field, p.field), "cudaIpcGetMemHandle");
    ck(cudaIpcGetMemHandle(&b.flags, p.flags), "cudaIpcGetMemHandle");
    b.device = p.d.device;
    b.pz = p.g.Pz;
    b.slot = p.g.slot;
    b.plane = p.g.pz;
    b.radius = p.g.R;
    b.rank = p.rank;
    b.world = p.world;
    std::memset(out, 0, SFDB200_IPC_BYTES);
    std::memcpy(out, &b, sizeof b);
}

void p2p_import(sfdb200_plan& p, const void* lower, const void* upper) {
    if (!p.dist() || p.g.ndim != 3) fail(SFDB200_EINVAL, "P2P exchange needs a 3-D z-slab plan");
    const void* blobs[2] = {lower, upper};
    const int want[2] = {p.rank - 1, p.rank + 1};
    Blob b[2]{};
    for (int side = 0; side < 2; ++side) {
        const bool has = side == 0 ? p.rank > 0 : p.rank < p.world - 1;
        if (has != (blobs[side] != nullptr))
            fail(SFDB200_EINVAL, "P2P import: neighbour blob missing or unexpected");
        if (!has) continue;
        std::memcpy(&b[side], blobs[side], sizeof(Blob));
        if (b[side].rank != want[side] || b[side].world != p.world)
            fail(SFDB200_EINVAL, "P2P import: blob is not the neighbour's");
        if (b[side].plane != p.g.pz || b[side].radius != p.g.R)
            fail(SFDB200_EINVAL, "P2P import: the neighbour's plan is for another problem");
        int can = 0;
        ck(cudaDeviceCanAccessPeer(&can, p.d.device, b[side].device), "cudaDeviceCanAccessPeer");
        if (!can) fail(SFDB200_EINVAL, "P2P import: neighbour device is not peer-accessible");
    }
    p2p_release(p);
    for (int side = 0; side < 2; ++side) {
        if (!blobs[side]) continue;
        void* f = nullptr;
        void* fl = nullptr;
        ck(cudaIpcOpenMemHandle(&f, b[side].field, cudaIpcMemLazyEnablePeerAccess),
           "cudaIpcOpenMemHandle");
        ck(cudaIpcOpenMemHandle(&fl, b[side].flags, cudaIpcMemLazyEnablePeerAccess),
           "cudaIpcOpenMemHandle");
        p.peer_field[side] = static_cast<float*>(f);
        p.peer_flags[side] = static_cast<unsigned int*>(fl);
        p.peer_slot[side] = b[side].slot;
        p.peer_pz[side] = b[side].pz;
        p.peer_ipc[side] = true;
    }
    p.p2p = true;
    p.p2p_sync = true;
}

void p2p_release(sfdb200_plan& p) {
    for (int side = 0; side < 2; ++side) {
        if (p.peer_ipc[side]) {
            cudaIpcCloseMemHandle(p.peer_field[side]);
            cudaIpcCloseMemHandle(p.peer_flags[side]);
        }
        p.peer_ipc[side] = false;
        p.peer_field[side] = nullptr;
        p.peer_flags[side] = nullptr;
    }
    p.p2p = false;
    p.p2p_sync = false;
}

// I am the upper neighbour of side 0 (it reads its counter [1]) and the lower
// neighbour of side 1 (its counter [0]).
void p2p_signal(sfdb200_plan& p, unsigned int value, cudaStream_t s) {
    static PFN_write32 write32 = driver_fn<PFN_write32>("cuStreamWriteValue32");
    for (int side = 0; side < 2; ++side) {
        if (!p.peer_flags[side]) continue;
        unsigned int* dst = p.peer_flags[side] + (side == 0 ? 1 : 0);
        const CUresult r = write32(reinterpret_cast<CUstream>(s),
                                   reinterpret_cast<CUdeviceptr>(dst), value, 0);
        if (r != CUDA_SUCCESS)
            fail(SFDB200_ECUDA, "cuStreamWriteValue32 failed (" + std::to_string(r) + ")");
    }
}

// A one-thread kernel rather than cuStreamWaitValue32: a neighbour that never
// publishes (its process died, its mapping is wrong) marks the plan's exchange
// broken after SFDB200_P2P_TIMEOUT_MS (default 60 s) instead of hanging the
// GPU; the run then completes with invalid values and p2p_check reports it.
void p2p_wait(sfdb200_plan& p, unsigned int value, cudaStream_t s) {
    static const unsigned long long timeout_ns =
        1000000ull * static_cast<unsigned long long>(env_int("SFDB200_P2P_TIMEOUT_MS", 60000));
    const unsigned int* f0 = p.peer_flags[0] ? p.flags + 0 : nullptr;  // written by side 0
    const unsigned int* f1 = p.peer_flags[1] ? p.flags + 1 : nullptr;  // written by side 1
    if (!f0 && !f1) return;
    unsigned int* pb0 = p.peer_flags[0] ? p.peer_flags[0] + kBrokenFlag : nullptr;
    unsigned int* pb1 = p.peer_flags[1] ? p.peer_flags[1] + kBrokenFlag : nullptr;
    ck(launch_wait_flags(f0, f1, value, timeout_ns, p.flags + kBrokenFlag, pb0, pb1, s),
       "P2P wait");
}

void p2p_check(sfdb200_plan& p) {
    if (!p.flags || !p.p2p) return;
    unsigned int broken = 0;
    ck(cudaMemcpyAsync(&broken, p.flags + kBrokenFlag, sizeof broken, cudaMemcpyDeviceToHost,
                       p.stream),
       "D2H");
    ck(cudaStreamSynchronize(p.stream), "P2P check");
    if (broken)
        fail(SFDB200_ECUDA,
             "P2P exchange broken: a neighbour's step counter did not arrive in time (peer "
             "process gone, stalled or its plan not imported) or a rank aborted the exchange; "
             "this plan's results are invalid");
}

// Marks the exchange broken on this rank and both neighbours now, not in
// stream order: a wait kernel already polling on any of them returns, and
// every later sweep skips its peer stores.  A separate non-blocking stream,
// since the plan's stream may be parked in a wait.
void p2p_abort(sfdb200_plan& p) {
    if (!p.flags) fail(SFDB200_EINVAL, "abort: the plan has no P2P exchange");
    cudaStream_t s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    static const unsigned int one = 1;
    cudaError_t e = cudaSuccess;
    for (unsigned int* f : {p.flags, p.peer_flags[0], p.peer_flags[1]})
        if (f && e == cudaSuccess)
            e = cudaMemcpyAsync(f + kBrokenFlag, &one, sizeof one, cudaMemcpyHostToDevice, s);
    const cudaError_t e2 = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    ck(e, "abort");
    ck(e2, "abort");
}

void p2p_selftest(int device) {
    ck(cudaSetDevice(device), "cudaSetDevice");
    // Two bare plans on one device stand in for neighbouring ranks: A is the
    // lower neighbour of B (A writes B's counter [0], B writes A's [1]).
    sfdb200_plan a, b;
    a.flags = dalloc<unsigned int>(64);
    b.flags = dalloc<unsigned int>(64);
    a.peer_flags[1] = b.flags;
    b.peer_flags[0] = a.flags;
    a.p2p = b.p2p = true;
    cudaStream_t s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaMemsetAsync(a.flags, 0, 64 * sizeof(unsigned int), s), "memset");
    ck(cudaMemsetAsync(b.flags, 0, 64 * sizeof(unsigned int), s), "memset");
    for (unsigned int v = 1; v <= 3; ++v) {
        p2p_signal(a, v, s);
        p2p_signal(b, v, s);
        p2p_wait(a, v, s);
        p2p_wait(b, v, s);
    }
    // B stalls (alive, but never publishes step 4): A's wait gives up after
    // 2 ms, marks A broken and poisons B; B's next wait (60 s budget) then
    // returns at once instead of timing out in turn.
    const auto t0 = std::chrono::steady_clock::now();
    ck(launch_wait_flags(a.flags + 1, nullptr, 4, 2000000ull, a.flags + kBrokenFlag, nullptr,
                         b.flags + kBrokenFlag, s),
       "wait");
    ck(launch_wait_flags(b.flags, nullptr, 5, 60000000000ull, b.flags + kBrokenFlag,
                         a.flags + kBrokenFlag, nullptr, s),
       "wait");
    unsigned int ha[kBrokenFlag + 1] = {}, hb[kBrokenFlag + 1] = {};
    ck(cudaMemcpyAsync(ha, a.flags, sizeof ha, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaMemcpyAsync(hb, b.flags, sizeof hb, cudaMemcpyDeviceToHost, s), "D2H");
    const cudaError_t e = cudaStreamSynchronize(s);
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    cudaStreamDestroy(s);
    a.peer_flags[1] = b.peer_flags[0] = nullptr;
    ck(e, "stream counters");
    if (ha[1] != 3 || hb[0] != 3) fail(SFDB200_ECUDA, "stream counters: unexpected values");
    if (ha[kBrokenFlag] != 1) fail(SFDB200_ECUDA, "timed-out wait did not mark the exchange broken");
    if (hb[kBrokenFlag] != 1) fail(SFDB200_ECUDA, "the timed-out rank did not poison its neighbour");
    if (secs > 30.0) fail(SFDB200_ECUDA, "the poisoned neighbour's wait did not return at once");
    // p2p_check reports it on both sides.
    for (sfdb200_plan* q : {&a, &b}) {
        ck(cudaStreamCreateWithFlags(&q->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
        q->stream = q->own_stream;
        bool thrown = false;
        try {
            p2p_check(*q);
        } catch (const Error&) {
            thrown = true;
        }
        if (!thrown) fail(SFDB200_ECUDA, "p2p_check did not report the broken exchange");
    }
}

}  // namespace sfdb200
