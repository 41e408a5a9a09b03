// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference library (stencilfd, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// Python tests, the golden-fixture generator and bench.py's reference arm
// call the reference's own operator API:
//   sfd::seismic::make_model        proj/src/seismic.cpp:100-142
//   sfd::seismic::locate_points     proj/src/seismic.cpp:195-230
//   sfd::seismic::ricker            proj/src/seismic.cpp:175-185
//   sfd::seismic::critical_dt       proj/src/seismic.cpp:187-193
//   sfd::seismic::forward           proj/src/seismic.cpp:333-380
//   sfd::seismic::adjoint           proj/src/seismic.cpp:382-426
//   sfd::seismic::gradient          proj/src/seismic.cpp:428-496
//   sfd::seismic::build_*_ir + codegen::generate (seismic.cpp:241-331,
//                                   codegen.cpp:579-629): the kernel source
//   sfd::seismic::save/load_model, save/load_record (seismic.cpp:557-614),
//   sfd::runtime::dump_grid (runtime.cpp:425-440): the file formats
// Every entry returns 0 on success and 1 on a thrown exception; the message
// is kept in a thread-local buffer (sfdref_last_error).

#include <algorithm>
#include <cstring>
#include <locale>
#include <memory>
#include <exception>
#include <string>
#include <vector>

#include "stencilfd/codegen.hpp"
#include "stencilfd/fd.hpp"
#include "stencilfd/runtime.hpp"
#include "stencilfd/seismic.hpp"

using namespace sfd;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        // Hosts such as CPython switch LC_CTYPE to the user's locale; the
        // reference's std::regex (grid_function.cpp) is run under "C".
        std::locale::global(std::locale::classic());
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

seismic::VelocityModel model_of(int ndim, const long* interior, double h, long nbpml, int so,
                                const double* m_interior) {
    std::vector<long> shape(interior, interior + ndim);
    long n = 1;
    for (long e : shape) n *= e;
    return seismic::make_model(shape, h, nbpml, so, std::vector<double>(m_interior, m_interior + n));
}

std::vector<std::vector<double>> coords_of(long npts, int ndim, const double* c) {
    std::vector<std::vector<double>> out;
    for (long p = 0; p < npts; ++p) out.emplace_back(c + p * ndim, c + (p + 1) * ndim);
    return out;
}

seismic::RunConfig config_of(int portable) {
    seismic::RunConfig cfg;
    if (portable) cfg.preset = runtime::preset_portable();
    return cfg;
}

}  // namespace

extern "C" {

const char* sfdref_last_error() { return g_err.c_str(); }

/// m_out/damp_out: padded cells; padded_out: ndim extents.
int sfdref_model(int ndim, const long* interior, double h, long nbpml, int so,
                 const double* m_interior, long* padded_out, double* m_out, double* damp_out) {
    return guarded([&] {
        const seismic::VelocityModel m = model_of(ndim, interior, h, nbpml, so, m_interior);
        for (int d = 0; d < ndim; ++d) padded_out[d] = m.padded[d];
        if (m_out) std::memcpy(m_out, m.m.data(), m.m.size() * sizeof(double));
        if (damp_out) std::memcpy(damp_out, m.damp.data(), m.damp.size() * sizeof(double));
    });
}

int sfdref_locate(int ndim, const long* interior, double h, long nbpml, int so,
                  const double* m_interior, long npts, const double* coords, long* idx_out,
                  double* w_out) {
    return guarded([&] {
        const seismic::VelocityModel m = model_of(ndim, interior, h, nbpml, so, m_interior);
        const seismic::SparsePoints p = seismic::locate_points(m, coords_of(npts, ndim, coords));
        std::memcpy(idx_out, p.idx.data(), p.idx.size() * sizeof(long));
        std::memcpy(w_out, p.w.data(), p.w.size() * sizeof(double));
    });
}

int sfdref_critical_dt(int ndim, const long* interior, double h, long nbpml, int so,
                       const double* m_interior, double* out) {
    return guarded([&] {
        *out = seismic::critical_dt(model_of(ndim, interior, h, nbpml, so, m_interior));
    });
}

int sfdref_ricker(double f0, double t0, long nt, double dt, double* out) {
    return guarded([&] {
        const std::vector<double> r = seismic::ricker(f0, t0, nt, dt);
        std::memcpy(out, r.data(), r.size() * sizeof(double));
    });
}

/// Second-derivative taps of fd_coefficients(2, so), offsets -so/2..so/2.
int sfdref_fd2(int so, double* out) {
    return guarded([&] {
        for (const StencilTap& t : fd_coefficients(2, so))
            out[t.offset + so / 2] = t.weight.to_double();
    });
}

/// u_out: (save ? nt+1 : 3) * cells; rec_out: nt * nrec.
int sfdref_forward(int ndim, const long* interior, double h, long nbpml, int so,
                   const double* m_interior, long nsrc, const double* src_coords,
                   const double* src_trace, long nrec, const double* rec_coords, long nt,
                   double dt, int save, int portable, double* u_out, double* rec_out,
                   double* seconds) {
    return guarded([&] {
        const seismic::VelocityModel m = model_of(ndim, interior, h, nbpml, so, m_interior);
        const seismic::SparsePoints src =
            seismic::locate_points(m, coords_of(nsrc, ndim, src_coords));
        const seismic::SparsePoints rec =
            seismic::locate_points(m, coords_of(nrec, ndim, rec_coords));
        const seismic::ForwardResult f = seismic::forward(
            m, src, std::vector<double>(src_trace, src_trace + nt * nsrc), rec, nt, dt,
            save != 0, config_of(portable));
        if (u_out) std::memcpy(u_out, f.u.data(), f.u.size() * sizeof(double));
        if (rec_out)
            std::memcpy(rec_out, f.record.data.data(), f.record.data.size() * sizeof(double));
        if (seconds) *seconds = f.stats.seconds;
    });
}

/// A model and its sparse sets built once (make_model, locate_points) and run
/// many times: the reference arm of bench.py times seismic::forward on cfg5
/// (1120^3), whose model construction alone takes seconds per call.
struct RefProblem {
    seismic::VelocityModel model;
    seismic::SparsePoints src, rec;
};

void* sfdref_problem_create(int ndim, const long* interior, double h, long nbpml, int so,
                            const double* m_interior, long nsrc, const double* src_coords,
                            long nrec, const double* rec_coords) {
    RefProblem* p = nullptr;
    const int rc = guarded([&] {
        auto q = std::make_unique<RefProblem>();
        q->model = model_of(ndim, interior, h, nbpml, so, m_interior);
        q->src = seismic::locate_points(q->model, coords_of(nsrc, ndim, src_coords));
        q->rec = seismic::locate_points(q->model, coords_of(nrec, ndim, rec_coords));
        p = q.release();
    });
    return rc == 0 ? p : nullptr;
}

void sfdref_problem_free(void* p) { delete static_cast<RefProblem*>(p); }

/// seismic::forward on a created problem; rec_out / seconds may be null.
int sfdref_problem_forward(void* prob, const double* src_trace, long nt, double dt,
                           double* rec_out, double* seconds) {
    return guarded([&] {
        RefProblem& q = *static_cast<RefProblem*>(prob);
        const seismic::ForwardResult f = seismic::forward(
            q.model, q.src, std::vector<double>(src_trace, src_trace + nt * q.src.npoints), q.rec,
            nt, dt, false, config_of(0));
        if (rec_out)
            std::memcpy(rec_out, f.record.data.data(), f.record.data.size() * sizeof(double));
        if (seconds) *seconds = f.stats.seconds;
    });
}

/// v_out: 3 * cells; src_out: nt * nsrc.
int sfdref_adjoint(int ndim, const long* interior, double h, long nbpml, int so,
                   const double* m_interior, long nrec, const double* rec_coords,
                   const double* residual, long nsrc, const double* src_coords, long nt,
                   double dt, int portable, double* v_out, double* src_out, double* seconds) {
    return guarded([&] {
        const seismic::VelocityModel m = model_of(ndim, interior, h, nbpml, so, m_interior);
        const seismic::SparsePoints rec =
            seismic::locate_points(m, coords_of(nrec, ndim, rec_coords));
        const seismic::SparsePoints src =
            seismic::locate_points(m, coords_of(nsrc, ndim, src_coords));
        seismic::ShotRecord r = seismic::zero_record(nt, dt, nrec);
        r.data.assign(residual, residual + nt * nrec);
        const seismic::AdjointResult a =
            seismic::adjoint(m, rec, r, src, nt, dt, config_of(portable));
        if (v_out) std::memcpy(v_out, a.v.data(), a.v.size() * sizeof(double));
        if (src_out)
            std::memcpy(src_out, a.src_samples.data.data(),
                        a.src_samples.data.size() * sizeof(double));
        if (seconds) *seconds = a.stats.seconds;
    });
}

/// u_history: (nt+1) * cells; grad_out: cells.
int sfdref_gradient(int ndim, const long* interior, double h, long nbpml, int so,
                    const double* m_interior, long nrec, const double* rec_coords,
                    const double* residual, const double* u_history, long nt, double dt,
                    int portable, double* grad_out, double* seconds) {
    return guarded([&] {
        const seismic::VelocityModel m = model_of(ndim, interior, h, nbpml, so, m_interior);
        const seismic::SparsePoints rec =
            seismic::locate_points(m, coords_of(nrec, ndim, rec_coords));
        seismic::ShotRecord r = seismic::zero_record(nt, dt, nrec);
        r.data.assign(residual, residual + nt * nrec);
        const std::vector<double> hist(u_history, u_history + (nt + 1) * m.cells());
        const seismic::GradientResult g =
            seismic::gradient(m, rec, r, hist, nt, dt, config_of(portable));
        std::memcpy(grad_out, g.grad.data(), g.grad.size() * sizeof(double));
        if (seconds) *seconds = g.stats.seconds;
    });
}

/// The C source codegen::generate emits for build_{forward,adjoint,gradient}_ir
/// (kind 0 / 1 / 2) on this model; plan 0 = default CodegenPlan, 1 = all_off,
/// 2 = fixed blocks of 4, 3 = blocking off.  Writes at most len bytes
/// (NUL-terminated) and the full length to *need.
int sfdref_generate(int kind, int ndim, const long* interior, double h, long nbpml, int so,
                    const double* m_interior, long nsrc, long nrec, long nt, double dt, int save,
                    int plan, char* out, long len, long* need) {
    return guarded([&] {
        const seismic::VelocityModel m = model_of(ndim, interior, h, nbpml, so, m_interior);
        const lower::KernelIR ir = kind == 0 ? seismic::build_forward_ir(m, nsrc, nrec, nt, dt, save)
                                   : kind == 1 ? seismic::build_adjoint_ir(m, nsrc, nrec, nt, dt)
                                               : seismic::build_gradient_ir(m, nrec, nt, dt);
        codegen::CodegenPlan p = plan == 1 ? codegen::CodegenPlan::all_off() : codegen::CodegenPlan{};
        if (plan == 2) {
            p.blocking = codegen::CodegenPlan::Blocking::Fixed;
            p.fixed_blocks.assign(static_cast<size_t>(codegen::blocked_dims(ndim)), 4);
        } else if (plan == 3) {
            p.blocking = codegen::CodegenPlan::Blocking::Off;
        }
        const std::string src = codegen::generate(ir, p).source;
        *need = static_cast<long>(src.size()) + 1;
        if (out && len > 0) {
            const size_t n = std::min(src.size(), static_cast<size_t>(len - 1));
            std::memcpy(out, src.data(), n);
            out[n] = 0;
        }
    });
}

/// seismic::objective on two records of n samples (npoints = n, nt = 1).
int sfdref_objective(const double* syn, const double* obs, long n, double* residual, double* phi) {
    return guarded([&] {
        seismic::ShotRecord a = seismic::zero_record(1, 1.0, n), b = a, r;
        a.data.assign(syn, syn + n);
        b.data.assign(obs, obs + n);
        *phi = seismic::objective(a, b, residual ? &r : nullptr);
        if (residual) std::memcpy(residual, r.data.data(), static_cast<size_t>(n) * sizeof(double));
    });
}

/// save_model of make_model(interior, h, nbpml, so, m_interior).
int sfdref_save_model(int ndim, const long* interior, double h, long nbpml, int so,
                      const double* m_interior, const char* prefix) {
    return guarded([&] {
        seismic::save_model(model_of(ndim, interior, h, nbpml, so, m_interior), prefix);
    });
}

/// load_model(prefix, so): ndim, interior, h, nbpml and the padded m / damp
/// (pass null m_out to query the shape first).
int sfdref_load_model(const char* prefix, int so, int* ndim, long* interior, double* h,
                      long* nbpml, long* padded, double* m_out, double* damp_out) {
    return guarded([&] {
        const seismic::VelocityModel m = seismic::load_model(prefix, so);
        *ndim = m.ndim();
        for (int d = 0; d < m.ndim(); ++d) {
            interior[d] = m.interior[static_cast<size_t>(d)];
            padded[d] = m.padded[static_cast<size_t>(d)];
        }
        *h = m.h;
        *nbpml = m.nbpml;
        if (m_out) std::memcpy(m_out, m.m.data(), m.m.size() * sizeof(double));
        if (damp_out) std::memcpy(damp_out, m.damp.data(), m.damp.size() * sizeof(double));
    });
}

int sfdref_save_record(long nt, double dt, long npts, int ndim, const double* coords,
                       const double* data, const char* prefix) {
    return guarded([&] {
        seismic::ShotRecord r = seismic::zero_record(nt, dt, npts);
        r.data.assign(data, data + nt * npts);
        seismic::save_record(r, coords_of(npts, ndim, coords), prefix);
    });
}

/// load_record: nt, dt, npoints, coordinate width; data / coords when non-null.
int sfdref_load_record(const char* prefix, long* nt, double* dt, long* npts, int* ndim,
                       double* coords, double* data) {
    return guarded([&] {
        std::vector<std::vector<double>> c;
        const seismic::ShotRecord r = seismic::load_record(prefix, &c);
        *nt = r.nt;
        *dt = r.dt;
        *npts = r.npoints;
        *ndim = c.empty() ? 0 : static_cast<int>(c[0].size());
        if (coords)
            for (size_t p = 0; p < c.size(); ++p)
                std::memcpy(coords + p * c[p].size(), c[p].data(), c[p].size() * sizeof(double));
        if (data) std::memcpy(data, r.data.data(), r.data.size() * sizeof(double));
    });
}

int sfdref_dump_grid(const double* data, int nshape, const long* shape, long halo, long time_slots,
                     const char* prefix) {
    return guarded([&] {
        runtime::dump_grid(data, std::vector<long>(shape, shape + nshape), halo, time_slots, prefix);
    });
}

}  // extern "C"
