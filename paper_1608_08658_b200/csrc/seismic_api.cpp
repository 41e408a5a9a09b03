// C++ operator API (include/sfdb200/seismic.hpp) over the C ABI: the drop-in
// for sfd::seismic (proj/src/seismic.cpp) with the kernels on the B200.
#include "../../include/sfdb200/seismic.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <numeric>

namespace sfdb200::seismic {
namespace {

long product(const std::vector<long>& v) {
    long p = 1;
    for (long e : v) p *= e;
    return p;
}

void check(int rc) {
    if (rc == SFDB200_OK) return;
    if (rc == SFDB200_EINVAL) throw std::invalid_argument(sfdb200_last_error());
    throw RuntimeError(sfdb200_last_error());
}

// seismic.cpp:31-37
void check_dt(const VelocityModel& model, double dt) {
    if (dt <= 0) throw std::invalid_argument("dt must be positive");
    const double limit = critical_dt(model);
    if (dt > limit)
        throw std::invalid_argument("dt " + std::to_string(dt) +
                                    " exceeds the stable CFL limit " + std::to_string(limit));
}

sfdb200_desc desc_of(int kind, const VelocityModel& m, long nt, double dt, long nsrc, long nrec,
                     bool save, const RunConfig& cfg) {
    sfdb200_desc d{};
    d.kind = kind;
    d.ndim = m.ndim();
    for (int k = 0; k < d.ndim; ++k) d.padded[k] = m.padded[static_cast<size_t>(k)];
    d.space_order = m.space_order;
    d.nt = nt;
    d.dt = dt;
    d.h = m.h;
    d.nsrc = nsrc;
    d.nrec = nrec;
    d.save = save ? 1 : 0;
    d.device = cfg.device;
    return d;
}

// One plan for the call: upload, device loop, download (runtime::run's single
// timed kernel call, runtime.cpp:335-353).
RunStats run(const sfdb200_desc& d, std::vector<void*> argv) {
    sfdb200_plan* plan = nullptr;
    check(sfdb200_plan_create(&d, &plan));
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = sfdb200_run(plan, argv.data());
    const auto t1 = std::chrono::steady_clock::now();
    const long pts = sfdb200_points_per_step(plan) * sfdb200_steps(plan);
    sfdb200_plan_destroy(plan);
    check(rc);
    RunStats st;
    st.seconds = std::chrono::duration<double>(t1 - t0).count();
    st.gpts = st.seconds > 0 ? static_cast<double>(pts) / st.seconds / 1e9 : 0;
    return st;
}

void* ptr(const void* p) { return const_cast<void*>(p); }

}  // namespace

long VelocityModel::cells() const { return product(padded); }
double VelocityModel::m_min() const { return *std::min_element(m.begin(), m.end()); }

VelocityModel make_model(std::vector<long> interior, double h, long nbpml, int space_order,
                         const std::vector<double>& m_interior) {
    if (interior.empty()) throw std::invalid_argument("model needs at least one dimension");
    for (long e : interior)
        if (e < 3) throw std::invalid_argument("model interior extents must be at least 3");
    if (h <= 0) throw std::invalid_argument("grid spacing must be positive");
    if (nbpml < 0) throw std::invalid_argument("absorbing-layer width must be non-negative");
    if (space_order < 2 || space_order % 2 != 0)
        throw std::invalid_argument("space order must be a positive even number");
    if (static_cast<long>(m_interior.size()) != product(interior))
        throw std::invalid_argument("squared-slowness field does not match the interior shape");
    for (double v : m_interior)
        if (!(v > 0)) throw std::invalid_argument("squared slowness must be positive");
    VelocityModel model;
    model.interior = std::move(interior);
    model.h = h;
    model.nbpml = nbpml;
    model.space_order = space_order;
    model.padded.resize(model.interior.size());
    long cells = 1;
    for (size_t d = 0; d < model.interior.size(); ++d)
        cells *= model.interior[d] + 2 * model.pad();
    model.m.resize(static_cast<size_t>(cells));
    model.damp.resize(static_cast<size_t>(cells));
    check(sfdb200_make_model(model.ndim(), model.interior.data(), h, nbpml, space_order,
                             m_interior.data(), model.padded.data(), model.m.data(),
                             model.damp.data()));
    return model;
}

VelocityModel make_constant_model(std::vector<long> interior, double h, long nbpml,
                                  int space_order, double velocity) {
    if (velocity <= 0) throw std::invalid_argument("velocity must be positive");
    const std::vector<double> m(static_cast<size_t>(product(interior)),
                                1.0 / (velocity * velocity));
    return make_model(std::move(interior), h, nbpml, space_order, m);
}

std::vector<double> build_damping(const std::vector<long>& padded, long nbpml, long halo,
                                  double h) {
    std::vector<double> out(static_cast<size_t>(product(padded)));
    check(sfdb200_build_damping(static_cast<int>(padded.size()), padded.data(), nbpml, halo, h,
                                out.data()));
    return out;
}

std::vector<double> ricker(double f0, double t0, long nt, double dt) {
    if (f0 <= 0) throw std::invalid_argument("peak frequency must be positive");
    if (nt < 0) throw std::invalid_argument("sample count must be non-negative");
    std::vector<double> out(static_cast<size_t>(nt));
    check(sfdb200_ricker(f0, t0, nt, dt, out.data()));
    return out;
}

double critical_dt(const VelocityModel& model) {
    return sfdb200_critical_dt(model.ndim(), model.h, model.space_order, model.m_min());
}

SparsePoints locate_points(const VelocityModel& model,
                           const std::vector<std::vector<double>>& coords) {
    const int nd = model.ndim();
    SparsePoints pts;
    pts.npoints = static_cast<long>(coords.size());
    pts.ndim = nd;
    std::vector<double> flat;
    for (const std::vector<double>& c : coords) {
        if (static_cast<int>(c.size()) != nd)
            throw std::invalid_argument("coordinate dimensionality does not match the model");
        for (int d = 0; d < nd; ++d) {
            const double span = static_cast<double>(model.interior[static_cast<size_t>(d)] - 1) * model.h;
            if (c[static_cast<size_t>(d)] < 0.0 || c[static_cast<size_t>(d)] > span)
                throw std::invalid_argument("point coordinate " + std::to_string(c[static_cast<size_t>(d)]) +
                                            " lies outside the physical interior [0, " +
                                            std::to_string(span) + "]");
        }
        flat.insert(flat.end(), c.begin(), c.end());
    }
    pts.idx.resize(static_cast<size_t>(pts.npoints * nd));
    pts.w.resize(static_cast<size_t>(pts.npoints << nd));
    check(sfdb200_locate_points(nd, model.interior.data(), model.h, model.nbpml,
                                model.space_order, pts.npoints, flat.data(), pts.idx.data(),
                                pts.w.data()));
    return pts;
}

ShotRecord zero_record(long nt, double dt, long npoints) {
    ShotRecord r;
    r.nt = nt;
    r.dt = dt;
    r.npoints = npoints;
    r.data.assign(static_cast<size_t>(nt * npoints), 0.0);
    return r;
}

ForwardResult forward(const VelocityModel& model, const SparsePoints& src,
                      const std::vector<double>& src_trace, const SparsePoints& rec, long nt,
                      double dt, bool save, const RunConfig& cfg) {
    check_dt(model, dt);
    if (static_cast<long>(src_trace.size()) != nt * src.npoints)
        throw std::invalid_argument("source trace must hold nt samples per source point");
    ForwardResult out;
    out.saved = save;
    out.u.assign(static_cast<size_t>((save ? history_rows(nt) : 3) * model.cells()), 0.0);
    out.record = zero_record(nt, dt, rec.npoints);
    const sfdb200_desc d = desc_of(SFDB200_FORWARD, model, nt, dt, src.npoints, rec.npoints, save, cfg);
    out.stats = run(d, {out.u.data(), ptr(model.m.data()), ptr(model.damp.data()),
                        ptr(src.idx.data()), ptr(src.w.data()), ptr(src_trace.data()),
                        ptr(rec.idx.data()), ptr(rec.w.data()), out.record.data.data()});
    return out;
}

AdjointResult adjoint(const VelocityModel& model, const SparsePoints& rec,
                      const ShotRecord& residual, const SparsePoints& src, long nt, double dt,
                      const RunConfig& cfg) {
    check_dt(model, dt);
    if (residual.nt != nt || residual.npoints != rec.npoints ||
        static_cast<long>(residual.data.size()) != nt * rec.npoints)
        throw std::invalid_argument("residual record does not match nt and the receiver set");
    AdjointResult out;
    out.v.assign(static_cast<size_t>(3 * model.cells()), 0.0);
    out.src_samples = zero_record(nt, dt, src.npoints);
    const sfdb200_desc d = desc_of(SFDB200_ADJOINT, model, nt, dt, src.npoints, rec.npoints, false, cfg);
    out.stats = run(d, {out.v.data(), ptr(model.m.data()), ptr(model.damp.data()),
                        ptr(src.idx.data()), ptr(src.w.data()), out.src_samples.data.data(),
                        ptr(rec.idx.data()), ptr(rec.w.data()), ptr(residual.data.data())});
    return out;
}

GradientResult gradient(const VelocityModel& model, const SparsePoints& rec,
                        const ShotRecord& residual, const std::vector<double>& u_history,
                        long nt, double dt, const RunConfig& cfg) {
    check_dt(model, dt);
    if (residual.nt != nt || residual.npoints != rec.npoints ||
        static_cast<long>(residual.data.size()) != nt * rec.npoints)
        throw std::invalid_argument("residual record does not match nt and the receiver set");
    if (static_cast<long>(u_history.size()) != history_rows(nt) * model.cells())
        throw std::invalid_argument("wavefield history must come from a saved forward run");
    GradientResult out;
    out.grad.assign(static_cast<size_t>(model.cells()), 0.0);
    std::vector<double> v(static_cast<size_t>(3 * model.cells()));
    const sfdb200_desc d = desc_of(SFDB200_GRADIENT, model, nt, dt, 0, rec.npoints, false, cfg);
    out.stats = run(d, {v.data(), ptr(u_history.data()), ptr(model.m.data()),
                        ptr(model.damp.data()), out.grad.data(), ptr(rec.idx.data()),
                        ptr(rec.w.data()), ptr(residual.data.data())});
    return out;
}

double objective(const ShotRecord& synthetic, const ShotRecord& observed, ShotRecord* residual) {
    if (synthetic.nt != observed.nt || synthetic.npoints != observed.npoints ||
        synthetic.data.size() != observed.data.size())
        throw std::invalid_argument("records disagree in shape");
    double phi = 0.0;
    if (residual) *residual = zero_record(synthetic.nt, synthetic.dt, synthetic.npoints);
    for (size_t i = 0; i < synthetic.data.size(); ++i) {
        const double dlt = synthetic.data[i] - observed.data[i];
        phi += dlt * dlt;
        if (residual) residual->data[i] = dlt;
    }
    return 0.5 * phi;
}

std::vector<double> restrict_interior(const VelocityModel& model,
                                      const std::vector<double>& padded_field) {
    if (static_cast<long>(padded_field.size()) != model.cells())
        throw std::invalid_argument("field does not match the padded shape");
    const int nd = model.ndim();
    std::vector<double> out(static_cast<size_t>(product(model.interior)));
    std::vector<long> pos(static_cast<size_t>(nd), 0);
    for (size_t i = 0; i < out.size(); ++i) {
        long cell = 0;
        for (int d = 0; d < nd; ++d)
            cell = cell * model.padded[static_cast<size_t>(d)] + pos[static_cast<size_t>(d)] + model.pad();
        out[i] = padded_field[static_cast<size_t>(cell)];
        for (int d = nd - 1; d >= 0; --d) {
            if (++pos[static_cast<size_t>(d)] < model.interior[static_cast<size_t>(d)]) break;
            pos[static_cast<size_t>(d)] = 0;
        }
    }
    return out;
}

void add_interior(const VelocityModel& model, const std::vector<double>& interior_field,
                  double scale, std::vector<double>& padded_field) {
    if (static_cast<long>(interior_field.size()) != product(model.interior) ||
        static_cast<long>(padded_field.size()) != model.cells())
        throw std::invalid_argument("field shapes do not match the model");
    const int nd = model.ndim();
    std::vector<long> pos(static_cast<size_t>(nd), 0);
    for (size_t i = 0; i < interior_field.size(); ++i) {
        long cell = 0;
        for (int d = 0; d < nd; ++d)
            cell = cell * model.padded[static_cast<size_t>(d)] + pos[static_cast<size_t>(d)] + model.pad();
        padded_field[static_cast<size_t>(cell)] += scale * interior_field[i];
        for (int d = nd - 1; d >= 0; --d) {
            if (++pos[static_cast<size_t>(d)] < model.interior[static_cast<size_t>(d)]) break;
            pos[static_cast<size_t>(d)] = 0;
        }
    }
}

}  // namespace sfdb200::seismic
