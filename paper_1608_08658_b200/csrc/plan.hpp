// Internal host-side structures of the B200 backend (not installed).
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sfdb200.h"
#include "kernels.cuh"

namespace sfdb200 {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(e == cudaErrorMemoryAllocation ? SFDB200_ENOMEM : SFDB200_ECUDA,
             std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
T* dalloc(size_t n) {
    if (n == 0) return nullptr;
    void* p = nullptr;
    ck(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
    return static_cast<T*>(p);
}

int env_int(const char* name, int dflt);

// A flat list of (point, corner) entries for the inject kernel.
struct InjectList {
    long n = 0;
    long long* off = nullptr;
    float* coef = nullptr;
    int* pt = nullptr;
    unsigned char* gm = nullptr;
};

// A flat list of sampled points for the sample kernel.
struct SampleList {
    long n = 0;
    long long* off = nullptr;  // [n][corners]
    float* w = nullptr;        // [n][corners]
    int* pt = nullptr;         // receiver index
};

// One sparse set on the device.
struct SparseDev {
    long n = 0;                // points in the (global) set
    float* trace = nullptr;    // [nt][n]
    std::vector<void*> bufs;   // device buffers owned by the tables below
    unsigned long long key = 0;  // fingerprint of the inputs the tables were built from

    // Injection: entries of the interior sweep launch, CSR over its CTAs
    // (applied by the CTA that stores the corner, after its planes), and the
    // rest (boundary / halo planes, or every entry when the sweep is not
    // fused) as a flat list.
    // f_tab is a CSR over the launch's items of RUNS (the entries of one cell,
    // adjacent and in the reference's (p, c) order); run r covers the entries
    // [f_run[r], f_run[r + 1]).
    int* f_tab = nullptr;
    int* f_run = nullptr;
    long long* f_off = nullptr;
    float* f_coef = nullptr;
    int* f_pt = nullptr;
    unsigned char* f_gm = nullptr;
    InjectList inj_rest;
    // Sampling: every owned receiver (smp_all).  In the fused 3-D sweep the
    // previous row is sampled at the start of the next interior launch
    // (s_base = corner-0 offsets, weights and columns shared with smp_all);
    // otherwise after each step.  The last row always after the last step.
    long long* s_base = nullptr;
    SampleList smp_all;
    // 2-D cluster time loop (cluster2d.cu): entries grouped by the CTA whose
    // row band holds the corner (inject) or the receiver's base row (sample),
    // with offsets into that CTA's shared-memory slot.
    long k_n = 0;
    int k_max = 0;                 // most entries of one CTA
    int* k_begin = nullptr;        // [nc + 1]
    int* k_soff = nullptr;         // inject: [n]; sample: [n][4]
    long long* k_goff = nullptr;   // inject: element offset in a global row (u_t)
    float* k_coef = nullptr;       // inject: coefficient; sample: [n][4] weights
    int* k_pt = nullptr;
    unsigned char* k_gm = nullptr;

    template <class T>
    T* upload(const std::vector<T>& v, cudaStream_t st) {
        if (v.empty()) return nullptr;
        T* d = dalloc<T>(v.size());
        bufs.push_back(d);
        ck(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st),
           "H2D");
        return d;
    }
    void free_tables() {
        for (void* q : bufs) cudaFree(q);
        bufs.clear();
        key = 0;
        f_tab = nullptr; f_run = nullptr; f_off = nullptr; f_coef = nullptr; f_pt = nullptr; f_gm = nullptr;
        s_base = nullptr;
        inj_rest = InjectList{};
        smp_all = SampleList{};
        k_n = 0;
        k_max = 0;
        k_begin = nullptr; k_soff = nullptr; k_goff = nullptr; k_coef = nullptr; k_pt = nullptr;
        k_gm = nullptr;
    }
};

struct Comm;  // comm.cpp

// Local plane zl of a slab with Pl planes (R ghost / halo planes a side) is
// stored and updated by this rank: its updated planes, plus the global halo
// planes on the first / last rank (ghost planes belong to the neighbours).
inline bool owns_plane(long zl, int R, long Pl, int rank, int world) {
    if (zl < 0 || zl >= Pl) return false;
    if (zl >= R && zl < Pl - R) return true;
    return zl < R ? rank == 0 : rank == world - 1;
}

}  // namespace sfdb200

struct sfdb200_comm {
    sfdb200::Comm* impl = nullptr;
};

struct sfdb200_plan {
    sfdb200_desc gd{};  // the global problem
    sfdb200_desc d{};   // this rank's slab (padded[0] = local planes)
    sfdb200::FieldGeom g{};
    int corners = 0;
    long long rows = 3;
    long long hist_rows = 0;

    // z-slab decomposition: local plane zl <-> global plane zl + zoff.
    int world = 1, rank = 0;
    long zoff = 0;
    int zint_lo = 0, zint_hi = 0;  // interior sweep launch (local planes)
    int blen = 0;                  // planes per boundary item (plan.cu set_boundary)
    int ctas2d = 0;                // 2-D: cooperative time-loop grid
    int nc2d = 0;                  // 2-D: CTAs of the single-cluster time loop (0: cooperative)
    long long per_cta2d = 0;       // 2-D: updated points per CTA
    sfdb200::Comm* comm = nullptr;
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_b = nullptr, ev_x = nullptr;
    // Fused P2P ghost exchange (p2p.cpp): the boundary sweeps store into the
    // neighbours' ghost planes; side 0 = lower neighbour (rank - 1), 1 = upper.
    bool p2p = false;
    bool p2p_sync = false;              // step counters (separate processes); off in loopback
    float* peer_field[2] = {nullptr, nullptr};
    long long peer_slot[2] = {0, 0};    // elements per row of the neighbour's field
    int peer_pz[2] = {0, 0};            // the neighbour's local plane count
    bool peer_ipc[2] = {false, false};  // peer_field / peer_flags opened through IPC
    unsigned int* flags = nullptr;      // my inbound step counters [2] (written by the neighbours)
    unsigned int* peer_flags[2] = {nullptr, nullptr};
    unsigned int flag_base = 1;         // epoch base, advanced identically on every rank
    int tables_nbi = 0;                 // boundary items the sparse tables were built for

    float* field = nullptr;  // u (forward) / v (adjoint, gradient), `rows` rows
    float* c1 = nullptr;
    float* c2 = nullptr;
    float* eprof = nullptr;  // 3-D: damp/dt profiles ez[Pz], ey[Py], ex[Px] (SweepArgs::ez)
    unsigned long long* eprof_scratch = nullptr;
    std::vector<double> hprof;  // host-checked damp profiles (upload source)
    bool sep_damp = false;   // the uploaded damp field is max-separable
    bool sep_layout = true;  // the tiling uses the separable stage layout (cfg.sep)
    // Uniform checkpointing (forward plans, 3-D): every ck_interval steps the
    // two latest rows are copied to ck_store (pairs 0..ck_pairs-1; pair j-1
    // restarts segment j, see do_execute_checkpointed).
    long ck_interval = 0;
    float* ck_store = nullptr;
    long ck_pairs = 0;
    bool ck_valid = false;   // the last execute() filled the store
    // Gradient plans bound to a checkpointed forward plan: hist holds one
    // recomputed segment (ck_interval + 2 rows).
    sfdb200_plan* ck_fwd = nullptr;
    // Gradient plans bound to a saved Forward plan's rows (sfdb200_bind_history).
    const sfdb200_plan* hist_fwd = nullptr;
    // Forward plans: recorded on `stream` at the end of every execute(); bound
    // gradient plans wait for it before reading the history / checkpoints.
    cudaEvent_t ev_done = nullptr;
    float* hist = nullptr;   // gradient: u history
    bool own_hist = false;
    float* grad = nullptr;
    sfdb200::SparseDev src, rec;
    double* staging = nullptr;
    size_t staging_elems = 0;
    // hostio.cpp: two pinned chunks staging copies of pageable caller buffers
    void* pin[2] = {nullptr, nullptr};
    void* xpin[2] = {nullptr, nullptr};  // the same for the record streamed on xstream
    int xpin_next = 0;
    bool host_rec_pinned = false;
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    unsigned long long* counter = nullptr;
    unsigned int* flag = nullptr;
    unsigned int* dbg = nullptr;  // debug builds: first failed access check (kernels.cuh)
    unsigned long long* item_ctr = nullptr;  // dynamic persistent sweeps (SweepArgs::item_ctr)

    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    sfdb200::SweepConfig cfg;
    sfdb200::SweepMaps maps{};
    sfdb200::SweepArgs base{};
    bool maps_ready = false;
    std::vector<std::pair<float, sfdb200::SweepConfig>> cands;  // autotune timings, fastest first
    bool fused = true;
    bool tuned = false;

    // run(): completed receiver rows stream to the caller's host record during
    // the time loop (copy stream + its own staging), the rest at download.
    double* host_rec = nullptr;
    long flushed = 0;
    double* xstaging = nullptr;
    size_t xstaging_elems = 0;
    cudaStream_t xstream = nullptr;
    cudaEvent_t ev_flush = nullptr;

    bool timing = false;
    std::vector<cudaEvent_t> events;
    long timed_launches = 0;
    long launches = 0;
    long h2d = 0, d2h = 0;
    int sms = 148;

    ~sfdb200_plan();

    long steps() const { return d.nt > 2 ? d.nt - 2 : 0; }
    long long cells() const { return static_cast<long long>(g.Pz) * g.Py * g.Px; }
    long long plane_cells() const { return static_cast<long long>(g.Py) * g.Px; }
    bool grad_kind() const { return d.kind == SFDB200_GRADIENT; }
    bool dist() const { return world > 1; }
    // Planes this rank stores and updates: its updated slab, plus the global
    // halo planes on the first / last rank (ghost planes belong to neighbours).
    bool owns_plane(long zl) const { return sfdb200::owns_plane(zl, g.R, g.Pz, rank, world); }
    sfdb200::SparseDev& injected() { return d.kind == SFDB200_FORWARD ? src : rec; }
    sfdb200::SparseDev* sampled() {
        if (d.kind == SFDB200_FORWARD) return &rec;
        if (d.kind == SFDB200_ADJOINT) return &src;
        return nullptr;
    }
    void ensure_staging(size_t elems) {
        if (elems <= staging_elems) return;
        cudaFree(staging);
        staging = nullptr;
        staging = sfdb200::dalloc<double>(elems);
        staging_elems = elems;
    }
};

namespace sfdb200 {

// sparse.cpp: host-side sparse tables for one set (corner offsets in the
// local device layout, ownership by rank, fused per-CTA tables).
void upload_sparse(sfdb200_plan& p, SparseDev& s, const long* idx, const double* w,
                   const double* m_global, unsigned long long data_hash = 0);
// Hash of a set's indices, weights and m at its corners (computed on the host
// while the model's H2D copy is in flight).
unsigned long long sparse_data_hash(const sfdb200_plan& p, long n, const long* idx,
                                    const double* w, const double* m_global);

// hostio.cpp: copies of the caller's host buffers (pageable ones staged
// through pinned chunks filled / drained by host threads).  copy_h2d returns
// once src may be reused (the DMA may still run); copy_d2h returns with the
// data in dst when dst is pageable, asynchronously (on p.stream) when pinned.
bool host_pinned(const void* ptr);
void copy_h2d(sfdb200_plan& p, void* dst, const void* src, size_t bytes);
void copy_d2h(sfdb200_plan& p, void* dst, const void* src, size_t bytes);
void release_pinned(sfdb200_plan& p);
// Half-width transfers for pageable caller buffers: host threads narrow the
// fp64 values to fp32 into the pinned chunks (round to nearest, the device's
// own conversion), so PCIe carries 4 B per value instead of 8, and widen
// fp32 values back (exact) on the way down.  copy_h2d_narrow with exact =
// true returns false -- having copied nothing that matters -- as soon as a
// value is not exactly representable in fp32 (the caller then moves fp64).
bool copy_h2d_narrow(sfdb200_plan& p, float* dst, const double* src, size_t count, bool exact);
void copy_d2h_widen(sfdb200_plan& p, double* dst, const float* src, size_t count);
// The same on stream s, drained into dst by stream host functions.
void copy_d2h_stream_widen(sfdb200_plan& p, double* dst, const float* src, size_t count,
                           cudaStream_t s);
// Stream-ordered D2H into a pageable destination on stream s (the record
// streamed during a run): through the plan's two xpin chunks, each drained by
// a stream host function, so the caller's thread never blocks.
void copy_d2h_stream_pageable(sfdb200_plan& p, void* dst, const void* src, size_t bytes,
                              cudaStream_t s);
// hostio.cpp: the damp field [Pz][Py][Px] is max(A[z], B[y], C[x]) bit for
// bit (non-negative); prof = A, B, C (the per-axis minima).
bool host_sep_damp(const double* damp, long long Pz, long long Py, long long Px,
                   std::vector<double>& prof);

// p2p.cpp: fused P2P ghost exchange.
// Byte offset from my `row` to the neighbour's ghost copy of the planes I
// send it on `side` (0 lower, 1 upper).
long long p2p_delta(const sfdb200_plan& p, int side, long long row);
// Boundary tiles at the front of the fused interior launch (0 unless the plan
// uses the P2P exchange): tiles x (number of neighbours).
int p2p_boundary_items(const sfdb200_plan& p);
void p2p_export(const sfdb200_plan& p, void* out);
void p2p_import(sfdb200_plan& p, const void* lower, const void* upper);
void p2p_release(sfdb200_plan& p);
// Stream memory operations on the step counters.
void p2p_signal(sfdb200_plan& p, unsigned int value, cudaStream_t s);
void p2p_wait(sfdb200_plan& p, unsigned int value, cudaStream_t s);
void p2p_check(sfdb200_plan& p);  // syncs; fails if a P2P wait timed out
void p2p_abort(sfdb200_plan& p);  // marks this rank and its neighbours broken now
constexpr int kBrokenFlag = 24;    // index in flags[] of the sticky timed-out flag
void p2p_selftest(int device);

// comm.cpp: NCCL (loaded at run time) for the ghost-plane exchange.
Comm* comm_create(const void* id128, int world, int rank, int device);
// Emulated rank (one-GPU test harness): no NCCL; see sfdb200_execute_group.
Comm* comm_create_loopback(int world, int rank, int device);
bool comm_loopback(const Comm* c);
void comm_destroy(Comm* c);
void comm_unique_id(void* id128);
// Sends/receives R ghost planes of one field row with the z neighbours.
void comm_exchange(Comm* c, sfdb200_plan& p, float* row, cudaStream_t s);
int comm_world(const Comm* c);
int comm_rank(const Comm* c);
int comm_device(const Comm* c);

// Owned global updated planes [z_begin, z_end) of `rank` (even split).
void slab_of(long pz_global, int R, int world, int rank, long* z_begin, long* z_end);

}  // namespace sfdb200
