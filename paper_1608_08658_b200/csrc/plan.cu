// Host runtime of the B200 backend: plans (device buffers, tensor maps,
// streams), the device-resident time loop and the C ABI of include/sfdb200.h.
//
// Reference counterparts:
//   sfdb200_call / sfdb200_run   int <Name>_call(void **argv), codegen.cpp:598-607,
//                                invoked by runtime::run, runtime.cpp:335-353
//   argv layout                  codegen::signature, codegen.cpp:247-265
//   time loop + sparse section   codegen.cpp:494-547 (forward t in [2,nt),
//                                backward t = nt-1 .. 2, lowering.hpp:78-80)
//   first touch                  codegen.cpp:464-492
//   gradient row-2 host term     seismic.cpp:468-490 (folded into the t = 2 step
//                                by the summation-by-parts form)
//   check_finite                 seismic.cpp:39-44
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sfdb200.h"
#include "kernels.cuh"

using namespace sfdb200;

namespace {

thread_local std::string g_error;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Error(code, msg); }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(e == cudaErrorMemoryAllocation ? SFDB200_ENOMEM : SFDB200_ECUDA,
             std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SFDB200_OK;
    } catch (const Error& e) {
        g_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_error = e.what();
        return SFDB200_EINVAL;
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            fail(SFDB200_ECUDA, "cuTensorMapEncodeTiled is unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// 4-D fp32 tensor map over [rows][z][y][x] (x pitched), zero OOB fill.
CUtensorMap make_map(const float* base, const FieldGeom& g, long long rows, unsigned box_x,
                     unsigned box_y) {
    CUtensorMap m;
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.Px), static_cast<cuuint64_t>(g.Py),
                                static_cast<cuuint64_t>(g.Pz), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(g.py) * 4,
                                   static_cast<cuuint64_t>(g.pz) * 4,
                                   static_cast<cuuint64_t>(g.slot) * 4};
    const cuuint32_t box[4] = {box_x, box_y, 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                                   const_cast<float*>(base), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(SFDB200_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return m;
}

template <class T>
T* dalloc(size_t n) {
    if (n == 0) return nullptr;
    void* p = nullptr;
    ck(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
    return static_cast<T*>(p);
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

// One sparse set on the device: per (point, corner) row offsets and weights.
struct SparseDev {
    long n = 0;
    long long* off = nullptr;
    float* coef = nullptr;       // w * dt^2 / m[corner]  (inject)
    float* w = nullptr;          // w                     (sample)
    unsigned char* gmask = nullptr;  // corner inside the updated region
    float* trace = nullptr;      // [nt][n]
    // 3-D fused operators: device buffers owned by this set, freed together.
    std::vector<void*> fused_bufs;
    // Inject entries per (sweep CTA, plane): table + entry arrays.
    int* f_tab = nullptr;
    int2* f_rng = nullptr;
    long long* f_off = nullptr;
    float* f_coef = nullptr;
    int* f_pt = nullptr;
    unsigned char* f_gm = nullptr;
    // Sample entries per (sweep CTA, base plane), read from the staged plane.
    int* s_tab = nullptr;
    int2* s_rng = nullptr;
    int* s_hidx = nullptr;
    float* s_w = nullptr;
    int* s_pt = nullptr;
    float* s_acc = nullptr;
    // Receivers no sweep CTA can sample (corner planes split across z chunks,
    // or halo cells): sampled by sample_kernel after the sweep.
    long fb_n = 0;
    long long* fb_off = nullptr;
    float* fb_w = nullptr;
    int* fb_pt = nullptr;
    void free_fused() {
        for (void* q : fused_bufs) cudaFree(q);
        fused_bufs.clear();
        f_tab = nullptr; f_rng = nullptr; f_off = nullptr; f_coef = nullptr; f_pt = nullptr; f_gm = nullptr;
        s_tab = nullptr; s_rng = nullptr; s_hidx = nullptr; s_w = nullptr; s_pt = nullptr; s_acc = nullptr;
        fb_n = 0; fb_off = nullptr; fb_w = nullptr; fb_pt = nullptr;
    }
    template <class T>
    T* upload(const std::vector<T>& v, cudaStream_t st);
};

}  // namespace

struct sfdb200_plan {
    sfdb200_desc d{};
    FieldGeom g{};
    int corners = 0;
    long long rows = 3;
    long long hist_rows = 0;

    float* field = nullptr;  // u (forward) / v (adjoint, gradient)
    float* c1 = nullptr;
    float* c2 = nullptr;
    float* hist = nullptr;   // gradient: u history
    bool own_hist = false;
    float* grad = nullptr;
    SparseDev src, rec;
    double* staging = nullptr;
    size_t staging_elems = 0;
    unsigned long long* counter = nullptr;

    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    SweepConfig cfg;
    SweepMaps maps{};
    SweepArgs base{};
    bool maps_ready = false;

    bool timing = false;
    std::vector<cudaEvent_t> events;
    long timed_launches = 0;
    long h2d = 0, d2h = 0;
    int sms = 148;

    ~sfdb200_plan() {
        cudaFree(field);
        cudaFree(c1);
        cudaFree(c2);
        if (own_hist) cudaFree(hist);
        cudaFree(grad);
        for (SparseDev* s : {&src, &rec}) {
            cudaFree(s->off);
            cudaFree(s->coef);
            cudaFree(s->w);
            cudaFree(s->gmask);
            cudaFree(s->trace);
            s->free_fused();
        }
        cudaFree(staging);
        cudaFree(counter);
        for (cudaEvent_t e : events) cudaEventDestroy(e);
        if (own_stream) cudaStreamDestroy(own_stream);
    }

    long steps() const { return d.nt > 2 ? d.nt - 2 : 0; }
    long long cells() const { return static_cast<long long>(g.Pz) * g.Py * g.Px; }
    bool grad_kind() const { return d.kind == SFDB200_GRADIENT; }

    // The set injected into the wavefield and the set sampled from it.
    SparseDev& injected() { return d.kind == SFDB200_FORWARD ? src : rec; }
    SparseDev* sampled() {
        if (d.kind == SFDB200_FORWARD) return &rec;
        if (d.kind == SFDB200_ADJOINT) return &src;
        return nullptr;
    }

    void ensure_staging(size_t elems) {
        if (elems <= staging_elems) return;
        cudaFree(staging);
        staging = nullptr;
        staging = dalloc<double>(elems);
        staging_elems = elems;
    }
};

namespace {

void validate(const sfdb200_desc& d) {
    if (d.kind < SFDB200_FORWARD || d.kind > SFDB200_GRADIENT) fail(SFDB200_EINVAL, "unknown operator kind");
    if (d.ndim != 2 && d.ndim != 3) fail(SFDB200_EINVAL, "ndim must be 2 or 3");
    if (d.space_order < 2 || d.space_order % 2 || d.space_order > 2 * kMaxRadius)
        fail(SFDB200_EINVAL, "space order must be an even number in [2, 16]");
    const int R = d.space_order / 2;
    for (int k = 0; k < d.ndim; ++k)
        if (d.padded[k] < 2 * R + 1 || d.padded[k] > (1L << 20))
            fail(SFDB200_EINVAL, "padded extent out of range");
    if (d.nt < 0) fail(SFDB200_EINVAL, "nt must be non-negative");
    if (!(d.dt > 0) || !(d.h > 0)) fail(SFDB200_EINVAL, "dt and h must be positive");
    if (d.nsrc < 0 || d.nrec < 0) fail(SFDB200_EINVAL, "negative sparse-set size");
}

void choose_config(sfdb200_plan& p) {
    SweepConfig& c = p.cfg;
    const int R = p.g.R;
    if (const char* t = std::getenv("SFDB200_TILE")) {
        std::sscanf(t, "%d,%d,%d,%d", &c.by, &c.ny, &c.stages, &c.rot);
    }
    c.tiles_x = static_cast<int>((p.g.Px - R + 31) / 32);  // tiles start at x = 0 (TMA alignment)
    c.tiles_y = static_cast<int>((p.g.Py - 2 * R + c.ty() - 1) / c.ty());
    c.smem_bytes = sweep3d_smem_bytes(R, c, p.grad_kind());
    const int by_smem = static_cast<int>((227 * 1024) / (c.smem_bytes + 1024));
    const int by_threads = 2048 / (32 * c.by);
    const int per_sm = std::max(1, std::min({by_smem, by_threads, 32}));
    const long long slots = static_cast<long long>(p.sms) * per_sm;
    const long long tiles = static_cast<long long>(c.tiles_x) * c.tiles_y;
    const int zupd = p.g.Pz - 2 * R;
    int zc = static_cast<int>(std::max<long long>(1, slots / std::max<long long>(1, tiles)));
    zc = std::min(zc, std::max(1, zupd / (4 * R + 8)));
    c.zchunks = env_int("SFDB200_ZCHUNKS", zc);
    c.zchunks = std::max(1, std::min(c.zchunks, zupd));
    c.zlen = (zupd + c.zchunks - 1) / c.zchunks;
    c.zchunks = (zupd + c.zlen - 1) / c.zlen;  // no empty chunks
}

void build_maps(sfdb200_plan& p) {
    if (p.g.ndim != 3) return;
    const int R = p.g.R;
    const unsigned TY = static_cast<unsigned>(p.cfg.ty());
    p.maps.uh = make_map(p.field, p.g, p.rows, static_cast<unsigned>(p.cfg.bw(R)), TY + 2 * R);
    p.maps.uc = make_map(p.field, p.g, p.rows, 32, TY);
    p.maps.c1 = make_map(p.c1, p.g, 1, 32, TY);
    p.maps.c2 = make_map(p.c2, p.g, 1, 32, TY);
    if (p.grad_kind() && p.hist) p.maps.ut = make_map(p.hist, p.g, p.hist_rows, 32, TY);
    else p.maps.ut = p.maps.uc;
    p.maps_ready = true;
}

void create(const sfdb200_desc& d, sfdb200_plan& p) {
    validate(d);
    p.d = d;
    ck(cudaSetDevice(d.device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, d.device), "cudaGetDeviceProperties");
    if (prop.major != 10) fail(SFDB200_ECUDA, "sfdb200 is built for sm_100a (B200); found sm_" +
                                              std::to_string(prop.major * 10 + prop.minor));
    p.sms = prop.multiProcessorCount;

    FieldGeom& g = p.g;
    g.ndim = d.ndim;
    g.R = d.space_order / 2;
    g.Pz = static_cast<int>(d.padded[0]);
    g.Py = d.ndim == 3 ? static_cast<int>(d.padded[1]) : 1;
    g.Px = static_cast<int>(d.padded[d.ndim - 1]);
    g.XP = (g.Px + 31) & ~31;
    g.py = g.XP;
    g.pz = static_cast<long long>(g.Py) * g.XP;
    g.slot = static_cast<long long>(g.Pz) * g.pz;
    p.corners = 1 << d.ndim;
    p.rows = (d.kind == SFDB200_FORWARD && d.save) ? d.nt + 1 : 3;

    const int R = g.R;
    const double h2 = d.h * d.h;
    double w[2 * kMaxRadius + 1];
    if (sfdb200_fd2(d.space_order, w) != 0) fail(SFDB200_EINVAL, "bad space order");
    for (int k = 0; k <= R; ++k) p.base.w[k] = static_cast<float>(w[R + k] / h2);
    p.base.neg2nd = static_cast<float>(-2.0 * d.ndim);
    p.base.nidt2 = static_cast<float>(-1.0 / (d.dt * d.dt));
    p.base.zlo = R;
    p.base.zhi = g.Pz - R;

    ck(cudaStreamCreateWithFlags(&p.own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    p.stream = p.own_stream;


    p.field = dalloc<float>(static_cast<size_t>(p.rows * g.slot));
    p.c1 = dalloc<float>(static_cast<size_t>(g.slot));
    p.c2 = dalloc<float>(static_cast<size_t>(g.slot));
    if (p.grad_kind()) p.grad = dalloc<float>(static_cast<size_t>(g.slot));
    p.counter = dalloc<unsigned long long>(1);
    // Pitch padding columns and halo cells must read as zero for the TMA boxes.
    ck(cudaMemsetAsync(p.c1, 0, g.slot * 4, p.stream), "memset");
    ck(cudaMemsetAsync(p.c2, 0, g.slot * 4, p.stream), "memset");
    p.src.n = d.kind == SFDB200_GRADIENT ? 0 : d.nsrc;
    p.rec.n = d.nrec;
    for (SparseDev* s : {&p.src, &p.rec}) {
        const size_t nc = static_cast<size_t>(s->n) * p.corners;
        s->off = dalloc<long long>(nc);
        s->coef = dalloc<float>(nc);
        s->w = dalloc<float>(nc);
        s->gmask = dalloc<unsigned char>(nc);
        s->trace = dalloc<float>(static_cast<size_t>(d.nt * s->n));
    }
    if (g.ndim == 3) choose_config(p);
    if (!p.grad_kind()) build_maps(p);
    ck(cudaStreamSynchronize(p.stream), "plan setup");
}

template <class T>
T* SparseDev::upload(const std::vector<T>& v, cudaStream_t st) {
    if (v.empty()) return nullptr;
    T* d = dalloc<T>(v.size());
    fused_bufs.push_back(d);
    ck(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
    return d;
}

// Sweep CTA (static grid: x tiles fastest, then y tiles, then z chunks) and
// its local plane index for a point of the updated region.
struct Owner {
    int cta, plane;
};

Owner owner_of(const sfdb200_plan& p, long z, long y, long x) {
    const SweepConfig& c = p.cfg;
    const int R = p.g.R;
    const int bx = static_cast<int>(x / 32), by = static_cast<int>((y - R) / c.ty()),
              bz = static_cast<int>((z - R) / c.zlen);
    return {bx + c.tiles_x * (by + c.tiles_y * bz), static_cast<int>(z - R - bz * c.zlen)};
}

// Per CTA, the plane range [lo, hi + extra) holding entries (extra = 1 for
// samples, whose second half comes one plane later); empty ranges are (0, 0).
std::vector<int2> plane_ranges(const sfdb200_plan& p, const std::vector<int>& tab, int extra) {
    const int ctas = p.cfg.tiles_x * p.cfg.tiles_y * p.cfg.zchunks, L = p.cfg.zlen + 1;
    std::vector<int2> r(static_cast<size_t>(ctas), make_int2(0, 0));
    for (int c = 0; c < ctas; ++c) {
        const int* t = tab.data() + static_cast<size_t>(c) * L;
        int lo = -1, hi = -1;
        for (int i = 0; i + 1 < L; ++i)
            if (t[i + 1] > t[i]) {
                if (lo < 0) lo = i;
                hi = i;
            }
        if (lo >= 0) r[static_cast<size_t>(c)] = make_int2(lo, std::min(hi + 1 + extra, L - 1));
    }
    return r;
}

// Per-CTA plane table over entries sorted by (cta, plane).
std::vector<int> plane_table(const sfdb200_plan& p, const std::vector<Owner>& keys) {
    const int ctas = p.cfg.tiles_x * p.cfg.tiles_y * p.cfg.zchunks, L = p.cfg.zlen + 1;
    std::vector<int> tab(static_cast<size_t>(ctas) * L, 0);
    size_t e = 0;
    for (int c = 0; c < ctas; ++c)
        for (int i = 0; i < L; ++i) {
            while (e < keys.size() &&
                   (keys[e].cta < c || (keys[e].cta == c && keys[e].plane < i)))
                ++e;
            tab[static_cast<size_t>(c) * L + i] = static_cast<int>(e);
        }
    return tab;
}

// Injection entries grouped by the sweep CTA that stores their corner, in
// (plane, point, corner) order so each plane's injections follow the
// reference's (p, c) order.  Corners the sweep never writes (halo cells) go to
// CTA 0's first plane.
void build_inject(sfdb200_plan& p, SparseDev& s, const long* idx,
                  const std::vector<long long>& off, const std::vector<float>& coef,
                  const std::vector<unsigned char>& mask) {
    const int R = p.g.R, C = p.corners;
    struct E { Owner o; size_t i; };
    std::vector<E> es;
    for (long q = 0; q < s.n; ++q)
        for (int k = 0; k < C; ++k) {
            const long z = idx[q * 3] + ((k >> 2) & 1), y = idx[q * 3 + 1] + ((k >> 1) & 1),
                       x = idx[q * 3 + 2] + (k & 1);
            const bool inside = z >= R && z < p.g.Pz - R && y >= R && y < p.g.Py - R &&
                                x >= R && x < p.g.Px - R;
            es.push_back({inside ? owner_of(p, z, y, x) : Owner{0, 0},
                          static_cast<size_t>(q) * C + k});
        }
    std::stable_sort(es.begin(), es.end(), [](const E& a, const E& b) {
        return a.o.cta != b.o.cta ? a.o.cta < b.o.cta : a.o.plane < b.o.plane;
    });
    std::vector<Owner> keys;
    std::vector<long long> eoff;
    std::vector<float> ecoef;
    std::vector<int> ept;
    std::vector<unsigned char> egm;
    for (const E& e : es) {
        keys.push_back(e.o);
        eoff.push_back(off[e.i]);
        ecoef.push_back(coef[e.i]);
        ept.push_back(static_cast<int>(e.i / C));
        egm.push_back(mask[e.i]);
    }
    cudaStream_t st = p.stream;
    const std::vector<int> tab = plane_table(p, keys);
    s.f_tab = s.upload(tab, st);
    s.f_rng = s.upload(plane_ranges(p, tab, 0), st);
    s.f_off = s.upload(eoff, st);
    s.f_coef = s.upload(ecoef, st);
    s.f_pt = s.upload(ept, st);
    s.f_gm = s.upload(egm, st);
}

// Sample entries: a receiver whose base corner (z0, y, x) lies in a sweep
// CTA's tile with both planes z0, z0+1 in that CTA's z chunk is read from the
// staged halo plane (all its x/y corners are inside tile + halo).
void build_sample(sfdb200_plan& p, SparseDev& s, const long* idx,
                  const std::vector<long long>& off, const std::vector<float>& w32) {
    const int R = p.g.R, RA = (R + 3) & ~3, BW = p.cfg.bw(R), C = p.corners;
    struct E { Owner o; int hidx; long q; };
    std::vector<E> es;
    std::vector<long long> fb_off;
    std::vector<float> fb_w;
    std::vector<int> fb_pt;
    for (long q = 0; q < s.n; ++q) {
        const long z = idx[q * 3], y = idx[q * 3 + 1], x = idx[q * 3 + 2];
        bool ok = z >= R && z + 1 < p.g.Pz - R && y >= R && y < p.g.Py - R && x >= 0 &&
                  x < 32L * p.cfg.tiles_x;
        Owner o{0, 0};
        if (ok) {
            o = owner_of(p, z, y, x);
            ok = o.plane + 1 < p.cfg.zlen && z + 1 < p.g.Pz - R;  // z0 + 1 in the same chunk
        }
        if (ok) {
            const int y0 = R + ((static_cast<int>(y) - R) / p.cfg.ty()) * p.cfg.ty();
            const int x0 = (static_cast<int>(x) / 32) * 32;
            es.push_back({o, (static_cast<int>(y) - y0 + R) * BW + (static_cast<int>(x) - x0 + RA), q});
        } else {
            for (int k = 0; k < C; ++k) {
                fb_off.push_back(off[static_cast<size_t>(q) * C + k]);
                fb_w.push_back(w32[static_cast<size_t>(q) * C + k]);
            }
            fb_pt.push_back(static_cast<int>(q));
        }
    }
    std::stable_sort(es.begin(), es.end(), [](const E& a, const E& b) {
        return a.o.cta != b.o.cta ? a.o.cta < b.o.cta : a.o.plane < b.o.plane;
    });
    std::vector<Owner> keys;
    std::vector<int> hidx, pt;
    std::vector<float> w8;
    for (const E& e : es) {
        keys.push_back(e.o);
        hidx.push_back(e.hidx);
        pt.push_back(static_cast<int>(e.q));
        for (int k = 0; k < C; ++k) w8.push_back(w32[static_cast<size_t>(e.q) * C + k]);
    }
    cudaStream_t st = p.stream;
    const std::vector<int> tab = plane_table(p, keys);
    s.s_tab = s.upload(tab, st);
    s.s_rng = s.upload(plane_ranges(p, tab, 1), st);
    s.s_hidx = s.upload(hidx, st);
    s.s_w = s.upload(w8, st);
    s.s_pt = s.upload(pt, st);
    s.s_acc = s.upload(std::vector<float>(es.size(), 0.0f), st);
    s.fb_n = static_cast<long>(fb_pt.size());
    s.fb_off = s.upload(fb_off, st);
    s.fb_w = s.upload(fb_w, st);
    s.fb_pt = s.upload(fb_pt, st);
}

// Host-side sparse tables: corner offsets in the device layout, inject
// coefficients w*dt^2/m[corner] (the reference's v = w; v *= scale; v *= data;
// v /= m, interpreter.cpp:144-147, with the data factor applied on device),
// sample weights, and the updated-region mask used by the gradient.
void upload_sparse(sfdb200_plan& p, SparseDev& s, const long* idx, const double* w,
                   const double* m) {
    if (s.n == 0) return;
    const sfdb200_desc& d = p.d;
    const FieldGeom& g = p.g;
    const int nd = d.ndim, C = p.corners, R = g.R;
    std::vector<long long> off(static_cast<size_t>(s.n) * C);
    std::vector<float> coef(off.size()), w32(off.size());
    std::vector<unsigned char> mask(off.size());
    for (long q = 0; q < s.n; ++q)
        for (int c = 0; c < C; ++c) {
            long pos[3] = {0, 0, 0};
            bool inside = true;
            for (int k = 0; k < nd; ++k) {
                pos[k] = idx[q * nd + k] + ((c >> (nd - 1 - k)) & 1);
                if (pos[k] < 0 || pos[k] >= d.padded[k])
                    fail(SFDB200_EINVAL, "sparse point corner lies outside the padded grid");
                inside = inside && pos[k] >= R && pos[k] < d.padded[k] - R;
            }
            long long dense = 0;
            for (int k = 0; k < nd; ++k) dense = dense * d.padded[k] + pos[k];
            const long long o = nd == 3 ? pos[0] * g.pz + pos[1] * g.py + pos[2]
                                        : pos[0] * g.pz + pos[1];
            const size_t i = static_cast<size_t>(q) * C + c;
            off[i] = o;
            w32[i] = static_cast<float>(w[i]);
            coef[i] = static_cast<float>(w[i] * (d.dt * d.dt) / m[dense]);
            mask[i] = inside ? 1 : 0;
        }
    ck(cudaMemcpyAsync(s.off, off.data(), off.size() * 8, cudaMemcpyHostToDevice, p.stream), "H2D");
    ck(cudaMemcpyAsync(s.coef, coef.data(), coef.size() * 4, cudaMemcpyHostToDevice, p.stream), "H2D");
    ck(cudaMemcpyAsync(s.w, w32.data(), w32.size() * 4, cudaMemcpyHostToDevice, p.stream), "H2D");
    ck(cudaMemcpyAsync(s.gmask, mask.data(), mask.size(), cudaMemcpyHostToDevice, p.stream), "H2D");
    if (nd == 3) {
        s.free_fused();
        if (&s == &p.injected()) build_inject(p, s, idx, off, coef, mask);
        if (&s == p.sampled()) build_sample(p, s, idx, off, w32);
    }
    ck(cudaStreamSynchronize(p.stream), "sparse upload");
    p.h2d += static_cast<long>(s.n) * (nd * 8 + C * 8);
}

void upload_trace(sfdb200_plan& p, SparseDev& s, const double* data) {
    const long long n = p.d.nt * s.n;
    if (n == 0) return;
    p.ensure_staging(static_cast<size_t>(n));
    ck(cudaMemcpyAsync(p.staging, data, n * 8, cudaMemcpyHostToDevice, p.stream), "H2D");
    ck(launch_dense_to_f32(p.staging, s.trace, n, p.stream), "convert");
    p.h2d += n * 8;
}

void download_trace(sfdb200_plan& p, SparseDev& s, double* out) {
    const long long n = p.d.nt * s.n;
    if (n == 0) return;
    p.ensure_staging(static_cast<size_t>(n));
    ck(launch_dense_to_f64(s.trace, p.staging, n, p.stream), "convert");
    ck(cudaMemcpyAsync(out, p.staging, n * 8, cudaMemcpyDeviceToHost, p.stream), "D2H");
    p.d2h += n * 8;
}

// rows of a padded fp64 field <-> device fp32 rows, chunked through staging.
void upload_rows(sfdb200_plan& p, const double* src, float* dst, long long rows) {
    const long long cells = p.cells();
    const long long chunk = std::max<long long>(1, std::min<long long>(rows, 2));
    p.ensure_staging(static_cast<size_t>(chunk * cells));
    for (long long r = 0; r < rows; r += chunk) {
        const long long nr = std::min(chunk, rows - r);
        ck(cudaMemcpyAsync(p.staging, src + r * cells, nr * cells * 8, cudaMemcpyHostToDevice,
                           p.stream), "H2D");
        ck(launch_to_f32(p.g, p.staging, dst + r * p.g.slot, nr, p.stream), "convert");
        p.h2d += nr * cells * 8;
    }
}

void download_rows(sfdb200_plan& p, const float* src, double* dst, long long rows) {
    const long long cells = p.cells();
    const long long chunk = std::max<long long>(1, std::min<long long>(rows, 3));
    p.ensure_staging(static_cast<size_t>(chunk * cells));
    for (long long r = 0; r < rows; r += chunk) {
        const long long nr = std::min(chunk, rows - r);
        ck(launch_to_f64(p.g, src + r * p.g.slot, p.staging, nr, p.stream), "convert");
        ck(cudaMemcpyAsync(dst + r * cells, p.staging, nr * cells * 8, cudaMemcpyDeviceToHost,
                           p.stream), "D2H");
        ck(cudaStreamSynchronize(p.stream), "D2H");
        p.d2h += nr * cells * 8;
    }
}

void do_upload(sfdb200_plan& p, void** argv) {
    const sfdb200_desc& d = p.d;
    const bool grad = p.grad_kind();
    const int im = grad ? 2 : 1;  // index of m in argv
    const double* m = static_cast<const double*>(argv[im]);
    const double* damp = static_cast<const double*>(argv[im + 1]);
    if (!m || !damp) fail(SFDB200_EINVAL, "null model buffer");
    const long long cells = p.cells();
    p.h2d = 0;
    p.ensure_staging(static_cast<size_t>(2 * cells));
    ck(cudaMemcpyAsync(p.staging, m, cells * 8, cudaMemcpyHostToDevice, p.stream), "H2D m");
    ck(cudaMemcpyAsync(p.staging + cells, damp, cells * 8, cudaMemcpyHostToDevice, p.stream),
       "H2D damp");
    ck(launch_coeffs(p.g, p.staging, p.staging + cells, d.dt, p.c1, p.c2, p.stream), "coeffs");
    ck(cudaStreamSynchronize(p.stream), "coeffs");
    p.h2d += 2 * cells * 8;

    if (grad) {
        upload_sparse(p, p.rec, static_cast<const long*>(argv[5]),
                      static_cast<const double*>(argv[6]), m);
        upload_trace(p, p.rec, static_cast<const double*>(argv[7]));
        if (!p.hist || p.own_hist) {
            if (!p.hist) {
                p.hist_rows = d.nt + 1;
                p.hist = dalloc<float>(static_cast<size_t>(p.hist_rows * p.g.slot));
                p.own_hist = true;
                ck(cudaMemsetAsync(p.hist, 0, p.hist_rows * p.g.slot * 4, p.stream), "memset");
            }
            upload_rows(p, static_cast<const double*>(argv[1]), p.hist, p.hist_rows);
        }
        build_maps(p);
    } else {
        upload_sparse(p, p.src, static_cast<const long*>(argv[3]),
                      static_cast<const double*>(argv[4]), m);
        upload_sparse(p, p.rec, static_cast<const long*>(argv[6]),
                      static_cast<const double*>(argv[7]), m);
        if (d.kind == SFDB200_FORWARD) upload_trace(p, p.src, static_cast<const double*>(argv[5]));
        else upload_trace(p, p.rec, static_cast<const double*>(argv[8]));
    }
    ck(cudaStreamSynchronize(p.stream), "upload");
}

void sweep(sfdb200_plan& p, SweepArgs a) {
    if (p.g.ndim == 3) ck(launch_sweep3d(p.g, p.cfg, p.maps, a, p.grad_kind(), p.stream), "sweep3d");
    else ck(launch_sweep2d(p.g, a, p.grad_kind(), p.stream), "sweep2d");
}

void do_execute(sfdb200_plan& p) {
    const sfdb200_desc& d = p.d;
    const FieldGeom& g = p.g;
    if (p.g.ndim == 3 && !p.maps_ready) fail(SFDB200_EINVAL, "execute before upload");
    cudaStream_t s = p.stream;
    // First touch (codegen.cpp:464-492) and zeroed trace outputs.
    ck(cudaMemsetAsync(p.field, 0, p.rows * g.slot * 4, s), "memset");
    if (SparseDev* out = p.sampled())
        ck(cudaMemsetAsync(out->trace, 0, d.nt * out->n * 4, s), "memset");
    if (p.grad) ck(cudaMemsetAsync(p.grad, 0, g.slot * 4, s), "memset");

    const long nsteps = p.steps();
    if (p.timing) {
        const size_t need = static_cast<size_t>(2 * nsteps);
        while (p.events.size() < need) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "cudaEventCreate");
            p.events.push_back(e);
        }
    }
    p.timed_launches = 0;

    SparseDev& inj = p.injected();
    SparseDev* smp = p.sampled();
    if (smp && smp->n == 0) smp = nullptr;
    const bool fwd = d.kind == SFDB200_FORWARD;
    const bool save = fwd && d.save;
    // 3-D: the sparse operators ride inside the sweep launches;
    // SFDB200_UNFUSED=1 runs them as their own kernels (A/B measurements).
    const bool fused = g.ndim == 3 && !env_int("SFDB200_UNFUSED", 0);
    long prev_srow = -1;
    const float* prev_out = nullptr;
    for (long i = 0; i < nsteps; ++i) {
        const long t = fwd ? 2 + i : d.nt - 1 - i;
        long r0, r1, r2;
        if (save) {
            r0 = t; r1 = t - 1; r2 = t - 2;
        } else if (fwd) {
            r0 = t % 3; r1 = (t - 1) % 3; r2 = (t - 2) % 3;
        } else {
            r0 = t % 3; r1 = (t + 1) % 3; r2 = (t + 2) % 3;
        }
        SweepArgs a = p.base;
        a.out = p.field + r0 * g.slot;
        a.u1 = p.field + r1 * g.slot;
        a.u2 = p.field + r2 * g.slot;
        a.c1 = p.c1;
        a.c2 = p.c2;
        a.row_out = static_cast<int>(r0);
        a.row_u1 = static_cast<int>(r1);
        a.row_u2 = static_cast<int>(r2);
        if (p.grad_kind()) {
            a.ut = p.hist + t * g.slot;
            a.grad = p.grad;
            a.row_ut = static_cast<int>(t);
        }
        a.zchunk = p.cfg.zlen;

        // Sparse section in list order, inject then sample (codegen.cpp:426-462):
        // inject trace row t-1 (forward, trace_offset -1) or t (adjoint, gradient);
        // sample rec row t (forward) or src row t-1 (adjoint).
        const long irow = fwd ? t - 1 : t;
        const long srow = fwd ? t : t - 1;
        if (fused && inj.n) {
            a.inj_tab = inj.f_tab;
            a.inj_rng = inj.f_rng;
            a.inj_off = inj.f_off;
            a.inj_coef = inj.f_coef;
            a.inj_pt = inj.f_pt;
            a.inj_gm = inj.f_gm;
            a.inj_row = inj.trace + irow * inj.n;
        }
        if (fused && smp && prev_srow >= 0 && smp->s_tab) {  // previous row == this u1
            a.smp_tab = smp->s_tab;
            a.smp_rng = smp->s_rng;
            a.smp_hidx = smp->s_hidx;
            a.smp_w = smp->s_w;
            a.smp_pt = smp->s_pt;
            a.smp_acc = smp->s_acc;
            a.smp_row = smp->trace + prev_srow * smp->n;
        }
        if (p.timing) ck(cudaEventRecord(p.events[2 * i], s), "event");
        sweep(p, a);
        if (p.timing) ck(cudaEventRecord(p.events[2 * i + 1], s), "event");
        ++p.timed_launches;
        if (!fused) {
            if (inj.n)
                ck(launch_inject(a.out, inj.off, inj.coef, inj.trace + irow * inj.n, inj.n,
                                 p.corners, p.grad, p.grad_kind() ? a.ut : nullptr, inj.gmask,
                                 p.base.nidt2, s),
                   "inject");
            if (smp)
                ck(launch_sample(a.out, smp->off, smp->w, nullptr, smp->trace + srow * smp->n,
                                 smp->n, p.corners, s),
                   "sample");
        } else if (smp && smp->fb_n) {  // receivers no sweep CTA can sample
            ck(launch_sample(a.out, smp->fb_off, smp->fb_w, smp->fb_pt,
                             smp->trace + srow * smp->n, smp->fb_n, p.corners, s),
               "sample");
        }
        prev_srow = srow;
        prev_out = a.out;
    }
    // The last step's row has no following sweep to be sampled in.
    if (fused && smp && prev_out && smp->s_tab)
        ck(launch_sample(prev_out, smp->off, smp->w, nullptr, smp->trace + prev_srow * smp->n,
                         smp->n, p.corners, s),
           "sample");
    ck(cudaGetLastError(), "execute");
}

void check_finite(sfdb200_plan& p, const float* a, long long n, const char* what) {
    ck(cudaMemsetAsync(p.counter, 0, 8, p.stream), "memset");
    ck(launch_count_nonfinite(a, n, p.counter, p.stream), "check_finite");
    unsigned long long bad = 0;
    ck(cudaMemcpyAsync(&bad, p.counter, 8, cudaMemcpyDeviceToHost, p.stream), "D2H");
    ck(cudaStreamSynchronize(p.stream), "check_finite");
    if (bad)
        fail(SFDB200_ENONFINITE,
             std::string("non-finite value in ") + what + " after the run (unstable step?)");
}

void do_download(sfdb200_plan& p, void** argv) {
    const sfdb200_desc& d = p.d;
    p.d2h = 0;
    ck(cudaStreamSynchronize(p.stream), "execute");
    check_finite(p, p.field, p.rows * p.g.slot, d.kind == SFDB200_FORWARD ? "the wavefield" : "the adjoint field");
    if (p.grad) check_finite(p, p.grad, p.g.slot, "the gradient");
    if (SparseDev* s = p.sampled())
        check_finite(p, s->trace, d.nt * s->n,
                     d.kind == SFDB200_FORWARD ? "the receiver record" : "the source samples");
    if (argv[0]) download_rows(p, p.field, static_cast<double*>(argv[0]), p.rows);
    if (d.kind == SFDB200_FORWARD && argv[8]) download_trace(p, p.rec, static_cast<double*>(argv[8]));
    if (d.kind == SFDB200_ADJOINT && argv[5]) download_trace(p, p.src, static_cast<double*>(argv[5]));
    if (d.kind == SFDB200_GRADIENT && argv[4]) download_rows(p, p.grad, static_cast<double*>(argv[4]), 1);
    ck(cudaStreamSynchronize(p.stream), "download");
}

std::mutex g_cache_mu;
std::map<std::string, std::unique_ptr<sfdb200_plan>>& plan_cache() {
    static std::map<std::string, std::unique_ptr<sfdb200_plan>> m;
    return m;
}

std::string desc_key(const sfdb200_desc& d) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "%d|%d|%ld,%ld,%ld|%d|%ld|%a|%a|%ld|%ld|%d|%d", d.kind, d.ndim,
                  d.padded[0], d.padded[1], d.padded[2], d.space_order, d.nt, d.dt, d.h, d.nsrc,
                  d.nrec, d.save, d.device);
    return buf;
}

}  // namespace

extern "C" {

const char* sfdb200_last_error(void) { return g_error.c_str(); }
const char* sfdb200_version(void) { return "sfdb200 0.1 (sm_100a)"; }

int sfdb200_plan_create(const sfdb200_desc* desc, sfdb200_plan** out) {
    return guarded([&] {
        if (!desc || !out) fail(SFDB200_EINVAL, "null argument");
        auto p = std::make_unique<sfdb200_plan>();
        create(*desc, *p);
        *out = p.release();
    });
}

int sfdb200_plan_destroy(sfdb200_plan* plan) {
    return guarded([&] {
        if (plan) {
            cudaSetDevice(plan->d.device);
            cudaStreamSynchronize(plan->stream);
            delete plan;
        }
    });
}

int sfdb200_upload(sfdb200_plan* p, void** argv) {
    return guarded([&] {
        if (!p || !argv) fail(SFDB200_EINVAL, "null argument");
        ck(cudaSetDevice(p->d.device), "cudaSetDevice");
        do_upload(*p, argv);
    });
}

int sfdb200_execute(sfdb200_plan* p) {
    return guarded([&] {
        if (!p) fail(SFDB200_EINVAL, "null plan");
        ck(cudaSetDevice(p->d.device), "cudaSetDevice");
        do_execute(*p);
    });
}

int sfdb200_download(sfdb200_plan* p, void** argv) {
    return guarded([&] {
        if (!p || !argv) fail(SFDB200_EINVAL, "null argument");
        ck(cudaSetDevice(p->d.device), "cudaSetDevice");
        do_download(*p, argv);
    });
}

int sfdb200_run(sfdb200_plan* p, void** argv) {
    return guarded([&] {
        if (!p || !argv) fail(SFDB200_EINVAL, "null argument");
        ck(cudaSetDevice(p->d.device), "cudaSetDevice");
        do_upload(*p, argv);
        do_execute(*p);
        do_download(*p, argv);
    });
}

int sfdb200_call(const sfdb200_desc* desc, void** argv) {
    return guarded([&] {
        if (!desc || !argv) fail(SFDB200_EINVAL, "null argument");
        std::lock_guard<std::mutex> lock(g_cache_mu);
        auto& slot = plan_cache()[desc_key(*desc)];
        if (!slot) {
            auto p = std::make_unique<sfdb200_plan>();
            create(*desc, *p);
            slot = std::move(p);
        }
        sfdb200_plan& p = *slot;
        ck(cudaSetDevice(p.d.device), "cudaSetDevice");
        do_upload(p, argv);
        do_execute(p);
        do_download(p, argv);
    });
}

int sfdb200_bind_history(sfdb200_plan* gp, const sfdb200_plan* fp) {
    return guarded([&] {
        if (!gp || !fp) fail(SFDB200_EINVAL, "null plan");
        if (gp->d.kind != SFDB200_GRADIENT || fp->d.kind != SFDB200_FORWARD || !fp->d.save)
            fail(SFDB200_EINVAL, "bind_history needs a Gradient plan and a saved Forward plan");
        if (gp->d.nt != fp->d.nt || gp->d.ndim != fp->d.ndim || gp->d.device != fp->d.device ||
            gp->d.space_order != fp->d.space_order ||
            std::memcmp(gp->d.padded, fp->d.padded, sizeof gp->d.padded) != 0)
            fail(SFDB200_EINVAL, "history comes from a different problem");
        if (gp->own_hist) cudaFree(gp->hist);
        gp->hist = fp->field;
        gp->hist_rows = fp->rows;
        gp->own_hist = false;
        gp->maps_ready = false;
    });
}

int sfdb200_set_stream(sfdb200_plan* p, void* stream) {
    return guarded([&] {
        if (!p) fail(SFDB200_EINVAL, "null plan");
        p->stream = stream ? static_cast<cudaStream_t>(stream) : p->own_stream;
    });
}

int sfdb200_set_timing(sfdb200_plan* p, int on) {
    return guarded([&] {
        if (!p) fail(SFDB200_EINVAL, "null plan");
        p->timing = on != 0;
    });
}

int sfdb200_stencil_time(sfdb200_plan* p, double* total_ms, long* launches) {
    return guarded([&] {
        if (!p || !total_ms) fail(SFDB200_EINVAL, "null argument");
        if (!p->timing) fail(SFDB200_EINVAL, "timing is off");
        double tot = 0;
        if (p->timed_launches > 0) {
            ck(cudaEventSynchronize(p->events[2 * p->timed_launches - 1]), "event sync");
            for (long i = 0; i < p->timed_launches; ++i) {
                float ms = 0;
                ck(cudaEventElapsedTime(&ms, p->events[2 * i], p->events[2 * i + 1]), "elapsed");
                tot += ms;
            }
        }
        *total_ms = tot;
        if (launches) *launches = p->timed_launches;
    });
}

long sfdb200_launches_per_execute(const sfdb200_plan* p) {
    if (!p) return -1;
    const SparseDev& inj = p->d.kind == SFDB200_FORWARD ? p->src : p->rec;
    const SparseDev* smp = p->d.kind == SFDB200_FORWARD ? &p->rec
                           : p->d.kind == SFDB200_ADJOINT ? &p->src : nullptr;
    const bool has_smp = smp && smp->n;
    if (p->g.ndim == 3)  // sparse ops fused into the sweeps (+ fallback and final sample)
        return p->steps() * (1 + (has_smp && smp->fb_n ? 1 : 0)) +
               (has_smp && p->steps() ? 1 : 0);
    return (1 + (inj.n ? 1 : 0) + (has_smp ? 1 : 0)) * p->steps();
}

long sfdb200_points_per_step(const sfdb200_plan* p) {
    if (!p) return -1;
    long n = 1;
    const int R = p->d.space_order / 2;
    for (int k = 0; k < p->d.ndim; ++k) n *= p->d.padded[k] - 2 * R;
    return n;
}

long sfdb200_steps(const sfdb200_plan* p) { return p ? p->steps() : -1; }
long sfdb200_h2d_bytes(const sfdb200_plan* p) { return p ? p->h2d : -1; }
long sfdb200_d2h_bytes(const sfdb200_plan* p) { return p ? p->d2h : -1; }

}  // extern "C"
