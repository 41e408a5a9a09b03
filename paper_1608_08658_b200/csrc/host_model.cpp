// Host-side helpers of the operator API, mirroring sfd::seismic so that the
// values handed to the kernels are bit-identical to the reference's.  Built
// with -ffp-contract=off like the reference library (proj/CMakeLists.txt:10-12).
//
//   sfdb200_fd2            fd_coefficients(2, so)         proj/src/fd.cpp:8-60
//   sfdb200_make_model     make_model + build_damping     proj/src/seismic.cpp:100-173
//   sfdb200_locate_points  locate_points                  proj/src/seismic.cpp:195-230
//   sfdb200_ricker         ricker                         proj/src/seismic.cpp:175-185
//   sfdb200_critical_dt    critical_dt                    proj/src/seismic.cpp:187-193
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numbers>
#include <vector>

#include "../../include/sfdb200.h"

namespace {

using i128 = __int128;

i128 gcd(i128 a, i128 b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b != 0) {
        const i128 t = a % b;
        a = b;
        b = t;
    }
    return a;
}

struct Frac {
    i128 num, den;
    void reduce() {
        const i128 g = gcd(num, den);
        num /= g;
        den /= g;
    }
    double value() const { return static_cast<double>(num) / static_cast<double>(den); }
};

// Damping profile along one axis (seismic.cpp:47-62).
std::vector<double> axis_profile(long extent, long nbpml, long halo, double h) {
    std::vector<double> out(static_cast<size_t>(extent), 0.0);
    if (nbpml <= 0) return out;
    const double c = 1.5 * std::log(1000.0) / (static_cast<double>(nbpml) * h);
    for (long i = 0; i < extent; ++i) {
        const long edge = std::min(i, extent - 1 - i);
        const double depth = std::max(static_cast<double>(edge - halo), 0.0);
        const double xi = std::clamp((static_cast<double>(nbpml) - depth) / nbpml, 0.0, 1.0);
        out[static_cast<size_t>(i)] =
            c * (xi - std::sin(2.0 * std::numbers::pi * xi) / (2.0 * std::numbers::pi));
    }
    return out;
}

}  // namespace

extern "C" {

// Closed form of the central second-derivative weights, exact in rationals:
//   w_{+-k} = 2 (-1)^{k+1} (r!)^2 / (k^2 (r-k)! (r+k)!),  w_0 = -2 sum_{k<=r} 1/k^2
// (the values Fornberg's recursion yields), rounded as num/den like
// Rational::to_double (rational.hpp:35-37).
int sfdb200_fd2(int so, double* w) {
    if (so < 2 || so % 2 != 0 || so > 24 || !w) return SFDB200_EINVAL;
    const int r = so / 2;
    i128 fact[25];
    fact[0] = 1;
    for (int i = 1; i <= 2 * r; ++i) fact[i] = fact[i - 1] * i;
    Frac centre{0, 1};
    for (int k = 1; k <= r; ++k) {
        Frac wk{2 * fact[r] * fact[r], static_cast<i128>(k) * k * fact[r - k] * fact[r + k]};
        wk.reduce();
        if (k % 2 == 0) wk.num = -wk.num;
        w[r - k] = w[r + k] = wk.value();
        centre = Frac{centre.num * k * k - 2 * centre.den, centre.den * k * k};
        centre.reduce();
    }
    w[r] = centre.value();
    return SFDB200_OK;
}

int sfdb200_build_damping(int ndim, const long* padded, long nbpml, long halo, double h,
                          double* out) {
    if (ndim < 1 || ndim > 3 || !padded || !out || !(h > 0)) return SFDB200_EINVAL;
    std::vector<std::vector<double>> axis;
    long cells = 1;
    for (int d = 0; d < ndim; ++d) {
        axis.push_back(axis_profile(padded[d], nbpml, halo, h));
        cells *= padded[d];
    }
    long pos[3] = {0, 0, 0};
    for (long cell = 0; cell < cells; ++cell) {
        double v = 0.0;
        for (int d = 0; d < ndim; ++d) v = std::max(v, axis[d][static_cast<size_t>(pos[d])]);
        out[cell] = v;
        for (int d = ndim - 1; d >= 0; --d) {
            if (++pos[d] < padded[d]) break;
            pos[d] = 0;
        }
    }
    return SFDB200_OK;
}

int sfdb200_make_model(int ndim, const long* interior, double h, long nbpml, int so,
                       const double* m_interior, long* padded, double* m, double* damp) {
    if (ndim < 1 || ndim > 3 || !interior || !m_interior || !padded || !m || !damp)
        return SFDB200_EINVAL;
    if (!(h > 0) || nbpml < 0 || so < 2 || so % 2 != 0) return SFDB200_EINVAL;
    const long pad = nbpml + so / 2;
    long cells = 1, icells = 1;
    for (int d = 0; d < ndim; ++d) {
        if (interior[d] < 3) return SFDB200_EINVAL;
        padded[d] = interior[d] + 2 * pad;
        cells *= padded[d];
        icells *= interior[d];
    }
    for (long i = 0; i < icells; ++i)
        if (!(m_interior[i] > 0)) return SFDB200_EINVAL;
    std::vector<std::vector<double>> axis;
    for (int d = 0; d < ndim; ++d) axis.push_back(axis_profile(padded[d], nbpml, so / 2, h));
    long pos[3] = {0, 0, 0};
    for (long cell = 0; cell < cells; ++cell) {
        long src = 0;
        double dv = 0.0;
        for (int d = 0; d < ndim; ++d) {
            src = src * interior[d] + std::clamp(pos[d] - pad, 0L, interior[d] - 1);
            dv = std::max(dv, axis[d][static_cast<size_t>(pos[d])]);
        }
        m[cell] = m_interior[src];
        damp[cell] = dv;
        for (int d = ndim - 1; d >= 0; --d) {
            if (++pos[d] < padded[d]) break;
            pos[d] = 0;
        }
    }
    return SFDB200_OK;
}

int sfdb200_locate_points(int ndim, const long* interior, double h, long nbpml, int so,
                          long npoints, const double* coords, long* idx, double* w) {
    if (ndim < 1 || ndim > 3 || npoints < 0 || !(h > 0)) return SFDB200_EINVAL;
    const long pad = nbpml + so / 2;
    const int corners = 1 << ndim;
    for (long p = 0; p < npoints; ++p) {
        double alpha[3];
        for (int d = 0; d < ndim; ++d) {
            const double span = static_cast<double>(interior[d] - 1) * h;
            const double x = coords[p * ndim + d];
            if (x < 0.0 || x > span) return SFDB200_EINVAL;
            const double base = std::floor(x / h);
            alpha[d] = x / h - base;
            idx[p * ndim + d] = static_cast<long>(base) + pad;
        }
        for (int k = 0; k < corners; ++k) {
            double v = 1.0;
            for (int d = 0; d < ndim; ++d)
                v *= ((k >> (ndim - 1 - d)) & 1) ? alpha[d] : 1.0 - alpha[d];
            w[p * corners + k] = v;
        }
    }
    return SFDB200_OK;
}

int sfdb200_ricker(double f0, double t0, long nt, double dt, double* out) {
    if (!(f0 > 0) || nt < 0) return SFDB200_EINVAL;
    for (long k = 0; k < nt; ++k) {
        const double tau = static_cast<double>(k) * dt - t0;
        const double a = std::numbers::pi * std::numbers::pi * f0 * f0 * tau * tau;
        out[k] = (1.0 - 2.0 * a) * std::exp(-a);
    }
    return SFDB200_OK;
}

double sfdb200_critical_dt(int ndim, double h, int so, double m_min) {
    double w[25];
    if (sfdb200_fd2(so, w) != SFDB200_OK) return -1.0;
    double tap_sum = 0.0;
    for (int i = 0; i <= so; ++i) tap_sum += std::abs(w[i]);
    return 0.9 * 2.0 * h * std::sqrt(m_min / (static_cast<double>(ndim) * tap_sum));
}

// objective (seismic.cpp:498-510): Phi = 1/2 sum (syn - obs)^2, summed in
// element order like the reference (compiled without contraction, so the
// bits agree); residual (optional) = syn - obs.
int sfdb200_objective(const double* syn, const double* obs, long n, double* residual, double* phi) {
    if (n < 0 || !phi || (n > 0 && (!syn || !obs))) return SFDB200_EINVAL;
    double acc = 0.0;
    for (long i = 0; i < n; ++i) {
        const double d = syn[i] - obs[i];
        acc += d * d;
        if (residual) residual[i] = d;
    }
    *phi = 0.5 * acc;
    return SFDB200_OK;
}

}  // extern "C"
