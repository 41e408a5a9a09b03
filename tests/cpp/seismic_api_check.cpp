// Exercises the C++ operator mirror (include/sfdb200/seismic.hpp) the way a
// reference caller would (cf. proj/tests/test_seismic.cpp:308-360): forward
// with save, objective, gradient, adjoint; writes inputs and outputs as raw
// float64 for tests/test_gpu_cpp_api.py to check against the oracle.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "sfdb200/seismic.hpp"

namespace S = sfdb200::seismic;

static void dump(const std::string& path, const std::vector<double>& v) {
    std::ofstream(path, std::ios::binary)
        .write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
}

int main(int argc, char** argv) {
    const std::string out = argc > 1 ? argv[1] : ".";
    const long n = 24;
    std::vector<double> mi(static_cast<size_t>(n * n * n));
    for (long i = 0; i < n; ++i)
        for (long j = 0; j < n; ++j)
            for (long k = 0; k < n; ++k) {
                const double r2 = (i - 12.0) * (i - 12.0) + (j - 10.0) * (j - 10.0) + (k - 13.0) * (k - 13.0);
                const double v = 2000.0 + 500.0 * std::exp(-r2 / 20.0) + 10.0 * i;
                mi[static_cast<size_t>((i * n + j) * n + k)] = static_cast<float>(1.0 / (v * v));
            }
    const S::VelocityModel model = S::make_model({n, n, n}, 10.0, 8, 8, mi);
    const double dt = 0.8 * S::critical_dt(model);
    const long nt = 120;
    const S::SparsePoints src = S::locate_points(model, {{35.0, 115.5, 117.25}});
    std::vector<std::vector<double>> rc;
    for (int a = 0; a < 6; ++a)
        for (int b = 0; b < 6; ++b) rc.push_back({20.0, 10.0 + 40.0 * a + 0.3, 7.5 + 41.0 * b});
    const S::SparsePoints rec = S::locate_points(model, rc);
    std::vector<double> wav = S::ricker(25.0, 0.04, nt, dt);
    for (double& x : wav) x = static_cast<float>(x);

    const S::ForwardResult f = S::forward(model, src, wav, rec, nt, dt, true);
    S::ShotRecord observed = S::zero_record(nt, dt, rec.npoints);
    for (size_t i = 0; i < observed.data.size(); ++i)
        observed.data[i] = static_cast<float>(0.7 * f.record.data[i]);
    S::ShotRecord resid;
    const double phi = S::objective(f.record, observed, &resid);
    const S::GradientResult g = S::gradient(model, rec, resid, f.u, nt, dt);
    const S::AdjointResult a = S::adjoint(model, rec, resid, src, nt, dt);

    bool refused = false;
    try {
        S::forward(model, src, wav, rec, nt, 1.01 * S::critical_dt(model), false);
    } catch (const std::invalid_argument&) {
        refused = true;
    }
    dump(out + "/m_interior.bin", mi);
    dump(out + "/wavelet.bin", wav);
    dump(out + "/record.bin", f.record.data);
    dump(out + "/u_hist.bin", f.u);
    dump(out + "/grad.bin", g.grad);
    dump(out + "/adj_src.bin", a.src_samples.data);
    dump(out + "/residual.bin", resid.data);
    std::vector<double> rcf;
    for (auto& c : rc) rcf.insert(rcf.end(), c.begin(), c.end());
    dump(out + "/rec_coords.bin", rcf);
    std::printf("{\"dt\": %.17g, \"nt\": %ld, \"phi\": %.17g, \"refused\": %d, \"gpts\": %.3f}\n",
                dt, nt, phi, refused ? 1 : 0, f.stats.gpts);
    return 0;
}
