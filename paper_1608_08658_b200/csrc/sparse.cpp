// Host-side preparation of the sparse operators (source injection, receiver
// sampling) for one plan: corner offsets in the device layout, ownership by
// z-slab rank, and the per-CTA tables that let the 3-D sweep apply them inside
// its own launch (injections after the CTA's planes, samples of the previous
// row at the CTA's start), including the P2P boundary items.
//
// Reference semantics: codegen.cpp:419-462 (corner bit order: bit ndim-1-d of
// c -> +1 along dim d; inject w * scale * data / m[corner]; sample
// sum_c w_c u[corner_c] in order c = 0..2^d-1), interpreter.cpp:118-160.
#include <algorithm>
#include <cstring>
#include <vector>

#include "plan.hpp"

namespace sfdb200 {
namespace {

struct Owner {
    int cta, plane;
};

// Item of the interior launch (x tiles fastest, then y tiles, then z chunks)
// holding a point, and its local plane index.  With the fused P2P exchange the
// launch starts with p2p_boundary_items(p) boundary tiles (R planes next to a
// neighbour, lower side first), which own the points of those planes.
Owner owner_of(const sfdb200_plan& p, long zl, long y, long x) {
    const SweepConfig& c = p.cfg;
    const int R = p.g.R;
    const int bx = static_cast<int>(x / 32), by = static_cast<int>((y - R) / c.ty());
    const int tile = bx + c.tiles_x * by, tiles = c.tiles_x * c.tiles_y;
    const int nbi = p2p_boundary_items(p);
    if (nbi) {
        const int hb = p.g.Pz - R - p.blen;  // first plane of the upper boundary items
        const bool lo = p.rank > 0 && zl >= R && zl < R + p.blen;
        const bool hi = p.rank < p.world - 1 && zl >= hb && zl < p.g.Pz - R;
        if (lo) return {tile, static_cast<int>(zl - R)};
        if (hi) return {(p.rank > 0 ? tiles : 0) + tile, static_cast<int>(zl - hb)};
    }
    const long zr = zl - p.zint_lo;
    const int bz = static_cast<int>(zr / c.zlen);
    return {nbi + tile + tiles * bz, static_cast<int>(zr - bz * c.zlen)};
}

// Swept by the interior launch (including its P2P boundary items).
bool in_interior(const sfdb200_plan& p, long zl, long y, long x) {
    const int R = p.g.R;
    const bool in_xy = y >= R && y < p.g.Py - R && x >= R && x < p.g.Px - R;
    if (!in_xy) return false;
    if (zl >= p.zint_lo && zl < p.zint_hi) return true;
    if (!p2p_boundary_items(p)) return false;
    return (p.rank > 0 && zl >= R && zl < R + p.blen) ||
           (p.rank < p.world - 1 && zl >= p.g.Pz - R - p.blen && zl < p.g.Pz - R);
}

int ctas_of(const sfdb200_plan& p) {
    return p.cfg.tiles_x * p.cfg.tiles_y * p.cfg.zchunks + p2p_boundary_items(p);
}

// 2-D cluster time loop: the CTA whose shared-memory rows hold row z (its
// band; the global halo rows belong to the first / last CTA) and the first
// global row of its shared-memory slot.
int band_owner(const sfdb200_plan& p, long z, int* row0) {
    const int R = p.g.R, nc = p.nc2d;
    int c = 0;
    for (int k = 0; k < nc; ++k) {
        int zb, ze;
        cluster2d_band(p.g.Pz, R, nc, k, &zb, &ze);
        if (z >= zb) c = k;
    }
    int zb, ze;
    cluster2d_band(p.g.Pz, R, nc, c, &zb, &ze);
    *row0 = zb - R;
    return c;
}

// CSR begin offsets [nc + 1] from per-entry owners (entries sorted by owner).
std::vector<int> csr_begin(const std::vector<int>& owner, int n, int* most) {
    std::vector<int> b(static_cast<size_t>(n) + 1, 0);
    for (int o : owner) ++b[static_cast<size_t>(o) + 1];
    *most = 0;
    for (int c = 0; c < n; ++c) *most = std::max(*most, b[static_cast<size_t>(c) + 1]);
    for (int c = 0; c < n; ++c) b[static_cast<size_t>(c) + 1] += b[static_cast<size_t>(c)];
    return b;
}

struct Corner {
    long long off;     // element offset in one local row
    long zl, y, x;     // local position
    long long dense;   // global dense index (for m)
    bool owned;        // this rank stores and updates the cell
    bool updated;      // inside the updated region (the gradient accumulates there)
};

}  // namespace

namespace {

unsigned long long mix64(unsigned long long h, unsigned long long v) {
    h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
    return h * 0xff51afd7ed558ccdULL;
}

// Fingerprint of the tables' inputs: the data hash (sparse_data_hash) and
// the sweep tiling the fused tables depend on.
unsigned long long fingerprint(const sfdb200_plan& p, unsigned long long data) {
    if (!data) return 0;
    unsigned long long h = mix64(data, static_cast<unsigned long long>(p.cfg.ty()) << 32 ^
                                           static_cast<unsigned>(p.cfg.zlen));
    h = mix64(h, static_cast<unsigned long long>(p.cfg.zchunks) << 32 ^
                     static_cast<unsigned>(p.cfg.tiles_x));
    h = mix64(h, static_cast<unsigned long long>(p2p_boundary_items(p)));
    return h | 1ULL;
}

}  // namespace

// Hash of indices, weights and m at the corners (the inject coefficients);
// 0 when a corner lies outside the grid (the table builder reports it).
unsigned long long sparse_data_hash(const sfdb200_plan& p, long n, const long* idx,
                                    const double* w, const double* m) {
    const sfdb200_desc& gd = p.gd;
    const int nd = gd.ndim, C = 1 << nd;
    unsigned long long h = 0x9e3779b97f4a7c15ULL;
    auto bits = [](double d) {
        unsigned long long u;
        std::memcpy(&u, &d, 8);
        return u;
    };
    h = mix64(h, static_cast<unsigned long long>(n));
    h = mix64(h, bits(gd.dt));
    for (long i = 0; i < n * nd; ++i) h = mix64(h, static_cast<unsigned long long>(idx[i]));
    for (long i = 0; i < n * C; ++i) h = mix64(h, bits(w[i]));
    for (long q = 0; q < n; ++q)
        for (int c = 0; c < C; ++c) {
            long long dense = 0;
            for (int k = 0; k < nd; ++k) {
                const long pos = idx[q * nd + k] + ((c >> (nd - 1 - k)) & 1);
                if (pos < 0 || pos >= gd.padded[k]) return 0;
                dense = dense * gd.padded[k] + pos;
            }
            h = mix64(h, bits(m[dense]));
        }
    return h | 1ULL;
}

void upload_sparse(sfdb200_plan& p, SparseDev& s, const long* idx, const double* w,
                   const double* m, unsigned long long data_hash) {
    if (s.n == 0) {
        s.free_tables();
        return;
    }
    // Re-running a plan on the same points (repeated shots, FWI iterations)
    // reuses the device tables.
    const unsigned long long key =
        fingerprint(p, data_hash ? data_hash : sparse_data_hash(p, s.n, idx, w, m));
    if (key && key == s.key) return;
    s.free_tables();
    const sfdb200_desc& gd = p.gd;
    const FieldGeom& g = p.g;
    const int nd = gd.ndim, C = p.corners, R = g.R;
    const cudaStream_t st = p.stream;
    const bool is_inj = &s == &p.injected();
    const bool is_smp = &s == p.sampled();
    const bool fused3d = nd == 3 && p.fused;

    std::vector<Corner> cs(static_cast<size_t>(s.n) * C);
    for (long q = 0; q < s.n; ++q)
        for (int c = 0; c < C; ++c) {
            long pos[3] = {0, 0, 0};
            long long dense = 0;
            for (int k = 0; k < nd; ++k) {
                pos[k] = idx[q * nd + k] + ((c >> (nd - 1 - k)) & 1);
                if (pos[k] < 0 || pos[k] >= gd.padded[k])
                    fail(SFDB200_EINVAL, "sparse point corner lies outside the padded grid");
                dense = dense * gd.padded[k] + pos[k];
            }
            Corner& k = cs[static_cast<size_t>(q) * C + c];
            k.zl = pos[0] - p.zoff;
            k.y = nd == 3 ? pos[1] : 0;
            k.x = pos[nd - 1];
            k.dense = dense;
            k.owned = p.owns_plane(k.zl);
            // every corner a table addresses lies in this rank's rows
            if (k.owned && (k.zl < 0 || k.zl >= g.Pz))
                fail(SFDB200_ECUDA, "internal: an owned sparse corner lies outside the slab");
            k.off = k.zl * g.pz + k.y * g.py + k.x;
            k.updated = k.zl >= R && k.zl < g.Pz - R && k.x >= R && k.x < g.Px - R &&
                        (nd == 2 || (k.y >= R && k.y < g.Py - R));
        }

    if (is_inj && nd == 2) {
        // 2-D time loop: entries grouped by the CTA owning the corner's point
        // (CSR in f_tab), reference (p, c) order within a CTA; halo corners
        // (never swept) go to CTA 0.
        const long nx = g.Px - 2L * R;
        struct E { int cta; size_t i; };
        std::vector<E> es;
        for (size_t i = 0; i < cs.size(); ++i) {
            const Corner& k = cs[i];
            int cta = 0;
            if (k.updated) cta = static_cast<int>(((k.zl - R) * nx + (k.x - R)) / p.per_cta2d);
            es.push_back({cta, i});
        }
        std::stable_sort(es.begin(), es.end(), [](const E& a, const E& b) { return a.cta < b.cta; });
        std::vector<int> begin(static_cast<size_t>(p.ctas2d) + 1, 0), ept;
        std::vector<long long> eoff;
        std::vector<float> ecoef;
        std::vector<unsigned char> egm;
        for (const E& e : es) {
            const Corner& k = cs[e.i];
            ++begin[static_cast<size_t>(e.cta) + 1];
            eoff.push_back(k.off);
            ecoef.push_back(static_cast<float>(w[e.i] * (gd.dt * gd.dt) / m[k.dense]));
            ept.push_back(static_cast<int>(e.i / C));
            egm.push_back(k.updated ? 1 : 0);
        }
        for (int c = 0; c < p.ctas2d; ++c) begin[static_cast<size_t>(c) + 1] += begin[static_cast<size_t>(c)];
        s.f_tab = s.upload(begin, st);
        s.f_off = s.upload(eoff, st);
        s.f_coef = s.upload(ecoef, st);
        s.f_pt = s.upload(ept, st);
        s.f_gm = s.upload(egm, st);
        if (p.nc2d) {  // cluster loop: by row band, shared-memory offsets, (p, c) order
            struct K { int cta; int soff; size_t i; };
            std::vector<K> ks;
            for (size_t i = 0; i < cs.size(); ++i) {
                const Corner& k = cs[i];
                int row0 = 0;
                const int cta = band_owner(p, k.zl, &row0);
                ks.push_back({cta, static_cast<int>((k.zl - row0) * g.XP + k.x), i});
            }
            std::stable_sort(ks.begin(), ks.end(), [](const K& a, const K& b) { return a.cta < b.cta; });
            std::vector<int> owner, soff, kpt;
            std::vector<long long> goff;
            std::vector<float> coef;
            std::vector<unsigned char> gm;
            for (const K& k : ks) {
                const Corner& c = cs[k.i];
                owner.push_back(k.cta);
                soff.push_back(k.soff);
                goff.push_back(c.off);
                coef.push_back(static_cast<float>(w[k.i] * (gd.dt * gd.dt) / m[c.dense]));
                kpt.push_back(static_cast<int>(k.i / C));
                gm.push_back(c.updated ? 1 : 0);
            }
            s.k_n = static_cast<long>(ks.size());
            s.k_begin = s.upload(csr_begin(owner, p.nc2d, &s.k_max), st);
            s.k_soff = s.upload(soff, st);
            s.k_goff = s.upload(goff, st);
            s.k_coef = s.upload(coef, st);
            s.k_pt = s.upload(kpt, st);
            s.k_gm = s.upload(gm, st);
        }
    } else if (is_inj) {
        // coef = w * dt^2 / m[corner]: the reference's v = w; v *= scale;
        // v /= m with the data factor applied on the device (interpreter.cpp:144-147).
        struct E { Owner o; size_t i; };
        std::vector<E> fused;
        std::vector<long long> r_off;
        std::vector<float> r_coef;
        std::vector<int> r_pt;
        std::vector<unsigned char> r_gm;
        for (size_t i = 0; i < cs.size(); ++i) {
            const Corner& k = cs[i];
            if (!k.owned) continue;
            if (fused3d && in_interior(p, k.zl, k.y, k.x)) {
                fused.push_back({owner_of(p, k.zl, k.y, k.x), i});
                continue;
            }
            r_off.push_back(k.off);
            r_coef.push_back(static_cast<float>(w[i] * (gd.dt * gd.dt) / m[k.dense]));
            r_pt.push_back(static_cast<int>(i / C));
            r_gm.push_back(k.updated ? 1 : 0);
        }
        s.inj_rest.n = static_cast<long>(r_off.size());
        s.inj_rest.off = s.upload(r_off, st);
        s.inj_rest.coef = s.upload(r_coef, st);
        s.inj_rest.pt = s.upload(r_pt, st);
        s.inj_rest.gm = s.upload(r_gm, st);
        if (!fused.empty()) {
            // CSR over the CTAs; within a CTA by cell, the reference's (p, c)
            // order among the entries of one cell (colliding corners): the
            // kernel sums each cell's run in that order and adds it once, so
            // the result does not depend on the order atomics land in.
            std::stable_sort(fused.begin(), fused.end(), [&](const E& a, const E& b) {
                return a.o.cta != b.o.cta ? a.o.cta < b.o.cta : cs[a.i].off < cs[b.i].off;
            });
            std::vector<int> owner, ept;
            std::vector<long long> eoff;
            std::vector<float> ecoef;
            std::vector<unsigned char> egm;
            for (const E& e : fused) {
                const Corner& k = cs[e.i];
                owner.push_back(e.o.cta);
                eoff.push_back(k.off);
                ecoef.push_back(static_cast<float>(w[e.i] * (gd.dt * gd.dt) / m[k.dense]));
                ept.push_back(static_cast<int>(e.i / C));
                egm.push_back(1);
            }
            // Runs: maximal groups of adjacent entries with the same item and
            // cell.  The kernel walks an item's runs, one thread per run.
            std::vector<int> run, run_owner;
            for (size_t i = 0; i < eoff.size();) {
                size_t j = i + 1;
                while (j < eoff.size() && owner[j] == owner[i] && eoff[j] == eoff[i]) ++j;
                run.push_back(static_cast<int>(i));
                run_owner.push_back(owner[i]);
                i = j;
            }
            run.push_back(static_cast<int>(eoff.size()));
            int most = 0;
            s.f_tab = s.upload(csr_begin(run_owner, ctas_of(p), &most), st);
            s.f_run = s.upload(run, st);
            s.f_off = s.upload(eoff, st);
            s.f_coef = s.upload(ecoef, st);
            s.f_pt = s.upload(ept, st);
            s.f_gm = s.upload(egm, st);
        }
    }

    if (is_smp) {
        // A receiver belongs to the rank owning its base plane z0 (z0 + 1 may
        // be a ghost plane, exchanged before the next step).
        std::vector<long long> a_off, a_base;
        std::vector<float> a_w;
        std::vector<int> a_pt;
        for (long q = 0; q < s.n; ++q) {
            const Corner& b = cs[static_cast<size_t>(q) * C];  // corner 0: the base
            if (!b.owned) continue;
            for (int c = 0; c < C; ++c) {
                a_off.push_back(cs[static_cast<size_t>(q) * C + c].off);
                a_w.push_back(static_cast<float>(w[static_cast<size_t>(q) * C + c]));
            }
            a_base.push_back(b.off);
            a_pt.push_back(static_cast<int>(q));
        }
#ifdef SFDB200_DEBUG
        // Fault injection for the access-check test (debug builds only): the
        // first receiver's base moves one row past the end of the field row.
        if (env_int("SFDB200_DEBUG_FAULT", 0) == 1 && !a_base.empty()) a_base[0] += g.slot;
#endif
        if (nd == 2 && p.nc2d) {  // cluster loop: by the band of the base row
            struct K { int cta; long q; };
            std::vector<K> ks;
            for (long q = 0; q < s.n; ++q) {
                int row0 = 0;
                ks.push_back({band_owner(p, cs[static_cast<size_t>(q) * C].zl, &row0), q});
            }
            std::stable_sort(ks.begin(), ks.end(), [](const K& a, const K& b) { return a.cta < b.cta; });
            std::vector<int> owner, soff, kpt;
            std::vector<float> kw;
            for (const K& k : ks) {
                int row0 = 0;
                band_owner(p, cs[static_cast<size_t>(k.q) * C].zl, &row0);
                owner.push_back(k.cta);
                kpt.push_back(static_cast<int>(k.q));
                for (int c = 0; c < C; ++c) {
                    const Corner& cc = cs[static_cast<size_t>(k.q) * C + c];
                    soff.push_back(static_cast<int>((cc.zl - row0) * g.XP + cc.x));
                    kw.push_back(static_cast<float>(w[static_cast<size_t>(k.q) * C + c]));
                }
            }
            s.k_n = s.n;
            s.k_begin = s.upload(csr_begin(owner, p.nc2d, &s.k_max), st);
            s.k_soff = s.upload(soff, st);
            s.k_coef = s.upload(kw, st);
            s.k_pt = s.upload(kpt, st);
        }
        s.smp_all.n = static_cast<long>(a_pt.size());
        s.smp_all.off = s.upload(a_off, st);
        s.smp_all.w = s.upload(a_w, st);
        s.smp_all.pt = s.upload(a_pt, st);
        if (fused3d) s.s_base = s.upload(a_base, st);
    }
    ck(cudaStreamSynchronize(st), "sparse upload");
    s.key = key;
    p.h2d += static_cast<long>(s.n) * (nd * 8 + C * 8);
}

}  // namespace sfdb200
