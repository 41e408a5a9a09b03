// C++ operator API of the B200 backend, mirroring sfd::seismic
// (/root/reference/proj/include/stencilfd/seismic.hpp:15-170): same type and
// function names, argument meaning and exceptions (std::invalid_argument for
// bad input, RuntimeError for failures after launch), so reference callers
// switch by changing the namespace.  Every operator runs on the B200 through
// libsfdb200.so; there is no CPU path.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "../sfdb200.h"

#pragma GCC visibility push(default)
namespace sfdb200::seismic {

struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// seismic.hpp:20-34
struct VelocityModel {
    std::vector<long> interior;
    double h = 10.0;
    long nbpml = 10;
    int space_order = 2;
    std::vector<long> padded;
    std::vector<double> m;
    std::vector<double> damp;

    int ndim() const { return static_cast<int>(interior.size()); }
    long halo() const { return space_order / 2; }
    long pad() const { return nbpml + halo(); }
    long cells() const;
    double m_min() const;
};

VelocityModel make_model(std::vector<long> interior, double h, long nbpml, int space_order,
                         const std::vector<double>& m_interior);
VelocityModel make_constant_model(std::vector<long> interior, double h, long nbpml,
                                  int space_order, double velocity);
std::vector<double> build_damping(const std::vector<long>& padded, long nbpml, long halo,
                                  double h);
std::vector<double> ricker(double f0, double t0, long nt, double dt);
double critical_dt(const VelocityModel& model);

/// seismic.hpp:61-71
struct SparsePoints {
    long npoints = 0;
    int ndim = 0;
    std::vector<long> idx;  // npoints x ndim
    std::vector<double> w;  // npoints x 2^ndim
};
SparsePoints locate_points(const VelocityModel& model,
                           const std::vector<std::vector<double>>& coords);

/// seismic.hpp:74-81
struct ShotRecord {
    long nt = 0;
    double dt = 0;
    long npoints = 0;
    std::vector<double> data;
};
ShotRecord zero_record(long nt, double dt, long npoints);

/// seismic.hpp:85-89 (the CPU compiler preset / blocks become the device).
struct RunConfig {
    int device = 0;
};

struct RunStats {
    double seconds = 0;  ///< wall time of upload + device run + download
    double gpts = 0;     ///< updated points x steps / seconds / 1e9
};

inline long history_rows(long nt) { return nt + 1; }

struct ForwardResult {
    ShotRecord record;
    std::vector<double> u;  // 3 rolling slots, or history_rows(nt) rows when saved
    bool saved = false;
    RunStats stats;
};
ForwardResult forward(const VelocityModel& model, const SparsePoints& src,
                      const std::vector<double>& src_trace, const SparsePoints& rec, long nt,
                      double dt, bool save, const RunConfig& cfg = {});

struct AdjointResult {
    ShotRecord src_samples;
    std::vector<double> v;  // 3 rolling slots
    RunStats stats;
};
AdjointResult adjoint(const VelocityModel& model, const SparsePoints& rec,
                      const ShotRecord& residual, const SparsePoints& src, long nt, double dt,
                      const RunConfig& cfg = {});

struct GradientResult {
    std::vector<double> grad;  // padded cells
    RunStats stats;
};
GradientResult gradient(const VelocityModel& model, const SparsePoints& rec,
                        const ShotRecord& residual, const std::vector<double>& u_history,
                        long nt, double dt, const RunConfig& cfg = {});

double objective(const ShotRecord& synthetic, const ShotRecord& observed,
                 ShotRecord* residual = nullptr);
std::vector<double> restrict_interior(const VelocityModel& model,
                                      const std::vector<double>& padded_field);
void add_interior(const VelocityModel& model, const std::vector<double>& interior_field,
                  double scale, std::vector<double>& padded_field);

}  // namespace sfdb200::seismic
#pragma GCC visibility pop
