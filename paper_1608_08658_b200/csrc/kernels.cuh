// Internal interface between the plan/runtime layer (plan.cu) and the sm_100a
// kernels (kernels.cu).  No torch, no reference types: plain pointers.
#pragma once
#include <string>

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sfdb200 {

constexpr int kMaxRadius = 8;  // space order 16

// Device field layout: fp32, row-major
// [row][z][y][x] with x padded to a 128-byte pitch XP (XP % 32 == 0), y
// unpadded.  2-D problems use Py == 1 ([row][z][1][x]).
struct FieldGeom {
    int ndim;
    int R;                 // stencil radius = space_order / 2
    int Pz, Py, Px;        // padded extents (Py == 1 in 2-D)
    int XP;                // x pitch in elements
    long long py, pz;      // element strides of y rows and z planes
    long long slot;        // elements per time row (Pz * pz)
};

// Sweep of the solved damped update, written in the incremental form
//   out = u1 + c1 (u1 - u2) + c2 lap(u1),  c1 = (a-b)/(a+b), c2 = 1/(a+b),
//   a = m/dt^2, b = damp/(2 dt)
// (algebraically the reference's (2a u1 - (a-b) u2 + lap)/(a+b),
// tests/golden/forward_3d_full.c:44-49).  With GRAD the same pass accumulates
// the imaging condition grad += -(1/dt^2) u_t (v_t - 2 v_{t+1} + v_{t+2}).
// Debug builds (make debug -> libsfdb200_debug.so, -DSFDB200_DEBUG): the
// kernels check their global-memory accesses against the rows they address
// and, on a violation, record the first check's code in *dbg and skip the
// access (the host then fails the plan: download / sfdb200_plan_check).
// Release builds compile the checks away.
#ifdef SFDB200_DEBUG
#define SFDB_CHECK(flag, cond, code) \
    ((cond) || ((flag) ? (atomicCAS((flag), 0u, static_cast<unsigned int>(code)), false) : false))
#else
#define SFDB_CHECK(flag, cond, code) true
#endif
enum DebugCheck : unsigned int {
    kDbgStore = 1,      // sweep store outside the output row
    kDbgGradStore = 2,  // gradient store outside the gradient row
    kDbgPeerStore = 3,  // P2P store outside the neighbour's row
    kDbgSample = 4,     // receiver corner outside the sampled row
    kDbgInject = 5,     // injection corner outside the written row
    kDbgTmaPlane = 6,   // TMA plane coordinate outside the field
    kDbgQueue = 7,      // z-queue prologue load outside the field
    kDbg2d = 8,         // 2-D loop: sparse offset outside the row
    kDbgInjectOwner = 9 // fused injection into a cell the injecting item did not store
};

struct SweepArgs {
    float* out;             // output row base
    const float* u1;        // row read at stencil offsets
    const float* u2;        // row read at the centre
    const float* c1;
    const float* c2;
    // Separable damping: when damp(z,y,x) == max(dz[z], dy[y],
    // dx[x]) exactly, as the reference's build_damping makes it, the 3-D sweep
    // forms c1 = 1 - e c2 with e = damp/dt = max(ez[z], ey[y], ex[x]) instead
    // of streaming the c1 field (16 instead of 20 B per updated point).
    // nullptr: stream c1.
    const float* ez;
    const float* ey;
    const float* ex;
    const float* ut;        // GRAD: u history row t
    float* grad;            // GRAD
    int row_out, row_u1, row_u2, row_ut;  // row coordinates for the tensor maps
    int zlo, zhi, zchunk;   // updated z range and planes per CTA
    // Bit k set: z chunk k streams downward (pair kernel; sweep3d.cuh
    // zdown_mask), so that chunks sharing a boundary read its planes at the
    // same time and the queue prologue hits L2.
    unsigned long long zdown;
    // Pair kernel, one CTA per item, more tiles than resident slots: items are
    // ordered in groups of `group` tiles (= the resident slots), all z chunks
    // of a group in turn, chunk-major within it, every chunk streaming up; the
    // slot a finished (tile, chunk k) frees is handed (in block order) to
    // (tile, chunk k + 1), whose first 2R planes are the ones just read, still
    // in L2.  0: tile-major order with zdown pairing.
    int group;
    float w[kMaxRadius + 1];  // w_k / h^2
    float neg2nd;           // -2 * ndim
    float nidt2;            // -1 / dt^2

    // Fused sparse operators (3-D sweep only; nullptr disables them), kept
    // out of the plane loop: they run once per CTA, before and after it.
    //
    // Sample the PREVIOUS step's row (= this launch's u1, complete once the
    // launch has passed griddepcontrol.wait) at the start of every CTA: the
    // receivers are split evenly over the CTAs of the launch, corner c of
    // receiver e at smp_base[e] + (c>>2) pz + ((c>>1)&1) py + (c&1), summed
    // c = 0..7 in the reference's order (codegen.cpp:450-458).
    const long long* smp_base;  // element offset of corner 0 in a row
    const float* smp_w;     // [entry][8]
    const int* smp_pt;      // receiver index (trace column)
    int smp_n;              // entries
    float* smp_row;         // trace row being sampled
    // Inject into this step's output once the CTA has stored all its planes
    // (codegen.cpp:436-449): the runs of item c are [inj_tab[c], inj_tab[c+1]),
    // one run per cell it stores; a run's entries (colliding corners) are
    // summed in the reference's (p, c) order and added once.
    const int* inj_tab;      // CSR over the items of runs (the entries of one cell)
    const int* inj_run;      // run r = entries [inj_run[r], inj_run[r + 1])
    const long long* inj_off;
    const float* inj_coef;
    const int* inj_pt;
    const unsigned char* inj_gm;  // GRAD: corner inside the updated region
    const float* inj_row;         // trace row of this step
    // Fused P2P ghost exchange (p2p.cpp), pair kernel: the first nbi items
    // of the launch are the boundary tiles (R planes next to a neighbour,
    // group g of `tiles` items on side bside[g]: planes [bz[side], bz[side] + R));
    // after its planes and injections each boundary item re-sends its values
    // to byte offset pdelta[side] (the neighbour's ghost copy, through its IPC
    // mapping).  The last boundary item to finish (done counter reaching
    // done_target) publishes sig_value to the neighbours' step counters
    // sig[0], sig[1] (system-scope release).  nbi = 0: no boundary items.
    int nbi;
    int blen;               // planes per boundary item (its first / last R are sent)
    int bside[2];
    int bz[2];
    long long pdelta[2];
    unsigned int* done;
    unsigned int done_target;
    unsigned int* sig[2];
    unsigned int sig_value;
    // This rank's sticky broken flag (P2P with step counters): once set, the
    // boundary items skip their peer stores and the step publication.
    const unsigned int* broken;
    // Pair kernel, dynamic persistent mode (SweepConfig::ctas == -2, separable
    // layout): the producer lane of each resident CTA takes the next item from
    // this counter and stages its index with the item's first plane; the CTA
    // taking the launch's last fetch resets it to 0 for the next launch.
    unsigned long long* item_ctr;
    // Debug checks (SFDB_CHECK): elements per row of this plan's fields and
    // of the neighbours' (P2P), the neighbours' rows written this step, the flag.
    long long slot;
    long long peer_slot[2];
    const float* peer_row[2];
    unsigned int* dbg;
};

struct SweepMaps {          // TMA descriptors (3-D only)
    CUtensorMap uh;         // u1 rows, halo box (BW, TY+2R, 1, 1)
    CUtensorMap uc;         // u1/u2 rows, centre box (32, TY, 1, 1)
    CUtensorMap c1, c2;     // coefficient fields, centre box
    CUtensorMap ut;         // GRAD: history rows, centre box
    CUtensorMap gr;         // GRAD: the gradient field, centre box
};

struct SweepConfig {        // 3-D tiling, chosen by choose_config()
    int by = 4;             // warps per CTA (each warp: 32 x-columns)
    int ny = 2;             // y rows per thread in each tile half (tile is 2*by*ny rows);
                            // pair mapping: rows per thread (two row groups per warp)
    int stages = 4;         // TMA pipeline depth
    int rot = 1;            // z unroll: 1 = by 2R+1 (queue rotates by renaming), 0 = none,
                            // k >= 2 = by k (pair mapping; sweep3d.cuh z_unroll)
    int zchunks = 1;        // CTAs along z per (x, y) tile
    int zlen = 1;           // planes per z chunk
    int pdl = 1;            // programmatic dependent launch (overlap launch + CTA setup)
    int pair = 0;           // thread owns column pairs x, x+1 (sweep3d_pair_kernel)
    int sep = 1;            // pair mapping: separable-damping stage layout (no c1 box);
                            // must match SweepArgs::ez != nullptr
    int ctas = 0;           // pair mapping: 0 = one CTA per (tile, z chunk) item, > 0 = that
                            // many persistent CTAs, -1 = one per resident slot (items
                            // round robin), -2 = one per resident slot taking items from
                            // a counter (SweepArgs::item_ctr; separable layout)
    int group = 1;          // pair mapping: grouped item order when tiles exceed the
                            // resident slots (SweepArgs::group); SFDB200_GROUP=0 disables
    int tiles_x = 0, tiles_y = 0;
    size_t smem_bytes = 0;
    int ty() const { return 2 * by * ny; }
    int bw(int R) const { return 32 + 2 * ((R + 3) & ~3); }
};

size_t sweep3d_smem_bytes(int R, const SweepConfig& cfg, bool grad);

cudaError_t launch_sweep3d(const FieldGeom& g, const SweepConfig& cfg, const SweepMaps& maps,
                           const SweepArgs& a, bool grad, cudaStream_t s);
// Per-radius instantiations (sweep3d_r<R>.cu); occ != nullptr queries the
// resident CTAs per SM instead of launching.
#define SFDB_DECL_R(RR)                                                                  \
    cudaError_t sweep3d_r##RR(const FieldGeom& g, const SweepConfig& cfg,                \
                              const SweepMaps& m, const SweepArgs& a, bool grad,          \
                              cudaStream_t s, int* occ);
SFDB_DECL_R(1)
SFDB_DECL_R(2)
SFDB_DECL_R(3)
SFDB_DECL_R(4)
SFDB_DECL_R(5)
SFDB_DECL_R(6)
SFDB_DECL_R(7)
SFDB_DECL_R(8)
#undef SFDB_DECL_R

namespace detail {
// sweep3d_instantiation(): when set, a launcher writes the kernel template it
// would launch (ncu's naming) here and returns without launching.
inline thread_local std::string* g_describe = nullptr;
}  // namespace detail
// The kernel template (with arguments) the variant cfg launches, e.g.
// "sweep3d_pair_kernel<4, 4, 2, 4, 0, 4, 9, 1>"; empty if cfg has none.
std::string sweep3d_instantiation(const FieldGeom& g, const SweepConfig& cfg, bool grad);
// Resident CTAs per SM of the variant cfg selects (registers + shared memory).
cudaError_t sweep3d_occupancy(const FieldGeom& g, const SweepConfig& cfg, bool grad,
                              int* blocks_per_sm);
cudaError_t launch_sweep2d(const FieldGeom& g, const SweepArgs& a, bool grad, cudaStream_t s);

// 2-D: the whole time loop in one cooperative launch (see kernels.cu).
struct Loop2dArgs {
    float* field;              // wavefield rows
    long long slot, pz;        // elements per row, per z line
    const float* c1;
    const float* c2;
    const float* hist;         // GRAD: u history rows
    float* grad;               // GRAD
    int kind, save;            // 0 forward, 1 adjoint, 2 gradient; forward history rows
    long nt;
    float w[kMaxRadius + 1];
    float neg2nd, nidt2;
    int Px;
    long long npts;            // updated points (Pz - 2R) * (Px - 2R)
    long long per_cta;         // updated points per CTA
    // injections owned by each CTA (CSR over CTAs), trace [nt][inj_n]
    const int* inj_begin;
    const long long* inj_off;
    const float* inj_coef;
    const int* inj_pt;
    const unsigned char* inj_gm;
    const float* inj_trace;
    long inj_n;
    // sampling: smp_cnt points [n][4] spread over the CTAs, trace [nt][smp_n]
    const long long* smp_off;
    const float* smp_w;
    const int* smp_pt;
    long smp_cnt, smp_per_cta;
    float* smp_trace;
    long smp_n;
    unsigned int* dbg;         // debug builds (SFDB_CHECK)
};
cudaError_t launch_loop2d(const Loop2dArgs& a, int R, bool grad, int ctas, cudaStream_t s);

// 2-D: the whole time loop in ONE thread-block cluster (cluster2d.cu).  The
// wavefield lives in the cluster's shared memory: CTA c owns a band of
// updated rows (cluster2d_band) plus R halo rows a side in three time slots;
// halo rows move between CTAs through distributed shared memory and the
// steps are separated by cluster barriers instead of grid-wide ones.
struct Cluster2dArgs {
    float* field;              // global rows (non-save: the 3 slots at the end)
    float* hist;               // forward save: history rows written every step
    const float* ut;           // GRAD: u history rows (read)
    float* grad;               // GRAD
    const float* c1;
    const float* c2;
    long long slot;            // elements per row
    int kind, save;
    long nt;
    float w[kMaxRadius + 1];
    float neg2nd, nidt2;
    int Pz, Px, XP, nc, nbmax;
    // injection / sampling tables (SparseDev::k_*), traces [nt][n]
    const int* inj_begin;
    const int* inj_soff;
    const long long* inj_goff;
    const float* inj_coef;
    const int* inj_pt;
    const unsigned char* inj_gm;
    const float* inj_trace;
    long inj_n;
    const int* smp_begin;
    const int* smp_soff;
    const float* smp_w;
    const int* smp_pt;
    float* smp_trace;
    long smp_n;
    // Entries per CTA staged in shared memory (an L1 line does not survive the
    // acquire of a cluster barrier); the rest are read from global memory.
    int inj_cap, smp_cap;
};
// Rows [zb, ze) of CTA c (updated rows R .. Pz-R split evenly).
__host__ __device__ inline void cluster2d_band(int Pz, int R, int nc, int c, int* zb, int* ze) {
    const int nz = Pz - 2 * R, base = nz / nc, rem = nz % nc;
    *zb = R + c * base + (c < rem ? c : rem);
    *ze = *zb + base + (c < rem ? 1 : 0);
}
// 0 when the problem does not fit one cluster (caller keeps loop2d).
int cluster2d_ctas(int Pz, int Px, int XP, int R, bool grad);
size_t cluster2d_smem_bytes(int Pz, int XP, int R, int nc, bool grad);
constexpr size_t kCluster2dSmemMax = 227 * 1024;
constexpr int kCluster2dInjBytes = 16, kCluster2dSmpBytes = 36;  // staged bytes per entry
cudaError_t launch_cluster2d(const Cluster2dArgs& a, int R, bool grad, cudaStream_t s);
int loop2d_blocks_per_sm(int R, bool grad);

// Sparse operators over flat entry lists: off = element offset of a corner
// inside one row, coef = w dt^2 / m[corner] (inject), pt = the entry's point
// (trace column).
// GRAD: the imaging condition of the row just finalised also sees the
// injected increment, grad[c] += -(1/dt^2) u_t[c] delta, for corners inside
// the updated region (gmask[p][c] != 0).
cudaError_t launch_inject(float* field, const long long* off, const float* coef, const int* pt,
                          const float* row, long n, float* grad, const float* ut,
                          const unsigned char* gmask, float nidt2, cudaStream_t s);
// grad += v2 u2 idt2 over the updated region (SFDB200_F_GRAD_NO_ROW2).
cudaError_t launch_grad_row2(float* grad, const float* v2, const float* u2, float idt2,
                             const FieldGeom& g, cudaStream_t s);
// Waits (one thread, on the stream) until the P2P step counters f0, f1 (either
// may be null) reach `value`; after timeout_ns, or once *broken is set, it
// sets *broken and the neighbours' flags peer_broken0/1 (either may be null;
// sticky: later waits return at once, later sweeps skip their peer stores)
// and returns.
cudaError_t launch_wait_flags(const unsigned int* f0, const unsigned int* f1, unsigned int value,
                              unsigned long long timeout_ns, unsigned int* broken,
                              unsigned int* peer_broken0, unsigned int* peer_broken1,
                              cudaStream_t s);
// pt (optional): output index of each sampled point (a subset of the set).
cudaError_t launch_sample(const float* field, const long long* off, const float* w,
                          const int* pt, float* row, long npoints, int corners, cudaStream_t s);

// Format conversion between the reference's dense fp64 layout and the device
// fp32 pitched layout.
cudaError_t launch_coeffs(const FieldGeom& g, const double* m, const double* damp, double dt,
                          float* c1, float* c2, cudaStream_t s);
// 3-D, separable damping checked on the host: prof = the fp64 per-axis
// profiles pz[Pz], py[Py], px[Px] (device memory); also writes e* as below.
cudaError_t launch_coeffs_sep(const FieldGeom& g, const double* m, const double* prof, double dt,
                              float* c1, float* c2, float* ez, float* ey, float* ex,
                              cudaStream_t s);
// Splits a dense fp64 damp field [Pz][Py][Px] into per-axis profiles
// e*[i] = fp32(min-profile / dt) and sets *mismatch != 0 unless
// damp == max(dz[z], dy[y], dx[x]) holds bit-exactly for every cell.
// scratch: Pz + Py + Px 64-bit words.
cudaError_t launch_damp_profiles(const double* damp, int Pz, int Py, int Px, double dt,
                                 unsigned long long* scratch, float* ez, float* ey, float* ex,
                                 unsigned int* mismatch, cudaStream_t s);
cudaError_t launch_to_f32(const FieldGeom& g, const double* src, float* dst, long long rows,
                          cudaStream_t s);
cudaError_t launch_to_f64(const FieldGeom& g, const float* src, double* dst, long long rows,
                          cudaStream_t s);
cudaError_t launch_dense_to_f32(const double* src, float* dst, long long n, cudaStream_t s);
// fp32 rows: dense [rows][Px] <-> pitched [rows][XP] (host-narrowed uploads,
// downloads widened on the host, hostio.cpp)
cudaError_t launch_pitch_f32(const FieldGeom& g, const float* src, float* dst, long long rows,
                             cudaStream_t s);
cudaError_t launch_unpitch_f32(const FieldGeom& g, const float* src, float* dst, long long rows,
                               cudaStream_t s);
// m narrowed on the host (only when exact): the same coefficients
cudaError_t launch_coeffs(const FieldGeom& g, const float* m, const double* damp, double dt,
                          float* c1, float* c2, cudaStream_t s);
cudaError_t launch_coeffs_sep(const FieldGeom& g, const float* m, const double* prof, double dt,
                              float* c1, float* c2, float* ez, float* ey, float* ex,
                              cudaStream_t s);
cudaError_t launch_dense_to_f64(const float* src, double* dst, long long n, cudaStream_t s);
// Counts non-finite values (the reference's check_finite, seismic.cpp:39-44).
cudaError_t launch_count_nonfinite(const float* a, long long n, unsigned long long* counter,
                                   cudaStream_t s);

}  // namespace sfdb200
