/* TEST INFRASTRUCTURE ONLY — CPU oracle (see sfd_oracle.h for the rules and
 * how this restatement is pinned to the reference).  fp64 throughout, built
 * with -ffp-contract=off like the reference library (proj/CMakeLists.txt:10-12).
 */
#include "sfd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

static i128 gcd128(i128 a, i128 b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        i128 t = a % b;
        a = b;
        b = t;
    }
    return a;
}

/* Central second-derivative weights in closed form (the values Fornberg's
 * recursion in proj/src/fd.cpp:8-60 produces exactly):
 *   w_{+-k} = 2 (-1)^{k+1} (r!)^2 / (k^2 (r-k)! (r+k)!),  w_0 = -2 sum_k 1/k^2.
 * Converted to double as Rational::to_double does (num / den, rational.hpp:35-37). */
int sfdo_fd2(int so, double* w) {
    if (so < 2 || so % 2 || so > 24) return 1;
    const int r = so / 2;
    i128 fact[2 * 12 + 1];
    fact[0] = 1;
    for (int i = 1; i <= 2 * r; ++i) fact[i] = fact[i - 1] * i;
    i128 c_num = 0, c_den = 1; /* running -2 sum 1/k^2 */
    for (int k = 1; k <= r; ++k) {
        i128 num = 2 * fact[r] * fact[r];
        i128 den = (i128)k * k * fact[r - k] * fact[r + k];
        i128 g = gcd128(num, den);
        num /= g;
        den /= g;
        if (k % 2 == 0) num = -num;
        w[r + k] = w[r - k] = (double)num / (double)den;
        /* c += -2 / k^2 */
        i128 n2 = c_num * k * k - 2 * c_den;
        i128 d2 = c_den * k * k;
        g = gcd128(n2, d2);
        c_num = n2 / g;
        c_den = d2 / g;
    }
    w[r] = (double)c_num / (double)c_den;
    return 0;
}

/* seismic.cpp:47-62 */
static void axis_damping(long extent, long nbpml, long halo, double h, double* out) {
    for (long i = 0; i < extent; ++i) out[i] = 0.0;
    if (nbpml <= 0) return;
    const double c = 1.5 * log(1000.0) / ((double)nbpml * h);
    const double two_pi = 2.0 * 3.141592653589793238462643383279502884;
    for (long i = 0; i < extent; ++i) {
        long edge = i < extent - 1 - i ? i : extent - 1 - i;
        double depth = (double)(edge - halo);
        if (depth < 0.0) depth = 0.0;
        double xi = ((double)nbpml - depth) / (double)nbpml;
        if (xi < 0.0) xi = 0.0;
        if (xi > 1.0) xi = 1.0;
        out[i] = c * (xi - sin(two_pi * xi) / two_pi);
    }
}

/* seismic.cpp:152-173: per-cell maximum over the axis profiles. */
void sfdo_damping(int ndim, const long* padded, long nbpml, long halo, double h, double* out) {
    double* axis[3];
    long cells = 1;
    for (int d = 0; d < ndim; ++d) {
        axis[d] = (double*)malloc(sizeof(double) * (size_t)padded[d]);
        axis_damping(padded[d], nbpml, halo, h, axis[d]);
        cells *= padded[d];
    }
    long pos[3] = {0, 0, 0};
    for (long cell = 0; cell < cells; ++cell) {
        double v = 0.0;
        for (int d = 0; d < ndim; ++d)
            if (axis[d][pos[d]] > v) v = axis[d][pos[d]];
        out[cell] = v;
        for (int d = ndim - 1; d >= 0; --d) {
            if (++pos[d] < padded[d]) break;
            pos[d] = 0;
        }
    }
    for (int d = 0; d < ndim; ++d) free(axis[d]);
}

/* seismic.cpp:100-142 */
int sfdo_make_model(int ndim, const long* interior, double h, long nbpml, int so,
                    const double* m_interior, long* padded, double* m, double* damp) {
    if (ndim < 1 || ndim > 3 || h <= 0 || nbpml < 0 || so < 2 || so % 2) return 1;
    const long pad = nbpml + so / 2;
    long cells = 1;
    for (int d = 0; d < ndim; ++d) {
        if (interior[d] < 3) return 1;
        padded[d] = interior[d] + 2 * pad;
        cells *= padded[d];
    }
    long pos[3] = {0, 0, 0};
    for (long cell = 0; cell < cells; ++cell) {
        long src = 0;
        for (int d = 0; d < ndim; ++d) {
            long c = pos[d] - pad;
            if (c < 0) c = 0;
            if (c > interior[d] - 1) c = interior[d] - 1;
            src = src * interior[d] + c;
        }
        if (!(m_interior[src] > 0)) return 1;
        m[cell] = m_interior[src];
        for (int d = ndim - 1; d >= 0; --d) {
            if (++pos[d] < padded[d]) break;
            pos[d] = 0;
        }
    }
    sfdo_damping(ndim, padded, nbpml, so / 2, h, damp);
    return 0;
}

/* seismic.cpp:195-230 */
int sfdo_locate(int ndim, const long* interior, double h, long nbpml, int so, long npts,
                const double* coords, long* idx, double* w) {
    const long pad = nbpml + so / 2;
    const int corners = 1 << ndim;
    for (long p = 0; p < npts; ++p) {
        double alpha[3];
        for (int d = 0; d < ndim; ++d) {
            const double span = (double)(interior[d] - 1) * h;
            const double x = coords[p * ndim + d];
            if (x < 0.0 || x > span) return 1;
            const double base = floor(x / h);
            alpha[d] = x / h - base;
            idx[p * ndim + d] = (long)base + pad;
        }
        for (int k = 0; k < corners; ++k) {
            double v = 1.0;
            for (int d = 0; d < ndim; ++d) {
                const int high = (k >> (ndim - 1 - d)) & 1;
                v *= high ? alpha[d] : 1.0 - alpha[d];
            }
            w[p * corners + k] = v;
        }
    }
    return 0;
}

/* seismic.cpp:175-185 */
void sfdo_ricker(double f0, double t0, long nt, double dt, double* out) {
    const double pi = 3.141592653589793238462643383279502884;
    for (long k = 0; k < nt; ++k) {
        const double tau = (double)k * dt - t0;
        const double a = pi * pi * f0 * f0 * tau * tau;
        out[k] = (1.0 - 2.0 * a) * exp(-a);
    }
}

/* seismic.cpp:187-193 */
double sfdo_critical_dt(int ndim, double h, int so, double m_min) {
    double w[25], sum = 0.0;
    if (sfdo_fd2(so, w)) return -1.0;
    for (int i = 0; i <= so; ++i) sum += fabs(w[i]);
    return 0.9 * 2.0 * h * sqrt(m_min / ((double)ndim * sum));
}

/* ---- operators -------------------------------------------------------- */

typedef struct {
    int nd, r;
    long P[3];
    long stride[3]; /* element strides of d0, d1, d2 in one slot */
    long cells;
    long lo[3], hi[3]; /* updated region [r, P-r) */
    double cw[13];     /* w_k / h^2, k = 0..r */
} geom;

static int make_geom(const sfdo_problem* p, geom* g) {
    if (p->ndim < 1 || p->ndim > 3) return 1;
    g->nd = p->ndim;
    g->r = p->space_order / 2;
    double w[25];
    if (sfdo_fd2(p->space_order, w)) return 1;
    const double h2 = p->h * p->h;
    for (int k = 0; k <= g->r; ++k) g->cw[k] = w[g->r + k] / h2;
    g->cells = 1;
    for (int d = 0; d < 3; ++d) {
        g->P[d] = d < g->nd ? p->padded[d] : 1;
        g->lo[d] = d < g->nd ? g->r : 0;
        g->hi[d] = d < g->nd ? g->P[d] - g->r : 1;
    }
    for (int d = 0; d < g->nd; ++d) g->cells *= g->P[d];
    long s = 1;
    for (int d = g->nd - 1; d >= 0; --d) {
        g->stride[d] = s;
        s *= g->P[d];
    }
    for (int d = g->nd; d < 3; ++d) g->stride[d] = 0;
    return 0;
}

/* One sweep of the solved damped update (seismic.cpp:247-248, golden
 * tests/golden/forward_3d_full.c:44-49):
 *   out = (2a u1 - (a - b) u2 + lap(u1)) / (a + b),  a = m/dt^2, b = damp/(2 dt).
 * The adjoint solves to the identical update with time reversed. */
static void sweep(const geom* g, double dt, double* out, const double* u1, const double* u2,
                  const double* m, const double* damp) {
    const double idt2 = 1.0 / (dt * dt), i2dt = 1.0 / (2.0 * dt);
#pragma omp parallel for collapse(2) schedule(static)
    for (long i0 = g->lo[0]; i0 < g->hi[0]; ++i0)
        for (long i1 = g->lo[1]; i1 < g->hi[1]; ++i1)
            for (long i2 = g->lo[2]; i2 < g->hi[2]; ++i2) {
                const long x = i0 * g->stride[0] + i1 * g->stride[1] + i2 * g->stride[2];
                double lap = 0.0;
                for (int d = 0; d < g->nd; ++d) {
                    const long s = g->stride[d];
                    lap += g->cw[0] * u1[x];
                    for (int k = 1; k <= g->r; ++k) lap += g->cw[k] * (u1[x - k * s] + u1[x + k * s]);
                }
                const double a = m[x] * idt2, b = damp[x] * i2dt;
                out[x] = (2.0 * a * u1[x] - (a - b) * u2[x] + lap) / (a + b);
            }
}

static long corner_offset(const geom* g, const long* idx, int c) {
    long a = 0;
    for (int d = 0; d < g->nd; ++d) a += (idx[d] + ((c >> (g->nd - 1 - d)) & 1)) * g->stride[d];
    return a;
}

/* codegen.cpp:436-449, interpreter.cpp:135-149: serial (p, c) order. */
static void inject(const geom* g, double* field, const double* m, long npts, const long* idx,
                   const double* w, const double* row, double scale) {
    const int corners = 1 << g->nd;
    for (long p = 0; p < npts; ++p)
        for (int c = 0; c < corners; ++c) {
            const long a = corner_offset(g, idx + p * g->nd, c);
            double v = w[p * corners + c];
            v *= scale;
            v *= row[p];
            v /= m[a];
            field[a] += v;
        }
}

/* codegen.cpp:450-458, interpreter.cpp:150-160 */
static void sample(const geom* g, const double* field, long npts, const long* idx,
                   const double* w, double* row) {
    const int corners = 1 << g->nd;
    for (long p = 0; p < npts; ++p) {
        double acc = 0.0;
        for (int c = 0; c < corners; ++c) {
            const double term = w[p * corners + c] * field[corner_offset(g, idx + p * g->nd, c)];
            acc = c == 0 ? term : acc + term;
        }
        row[p] = acc;
    }
}

/* seismic.cpp:333-380 with the kernel of build_forward_ir (seismic.cpp:241-267):
 * for t in [2, nt): sweep u[t]; inject src[t-1] * dt^2 / m; sample rec[t]. */
int sfdo_forward(const sfdo_problem* p, int save, double* u, const double* m, const double* damp,
                 const long* src_idx, const double* src_w, const double* src_data,
                 const long* rec_idx, const double* rec_w, double* rec_data) {
    geom g;
    if (make_geom(p, &g)) return 1;
    const long rows = save ? p->nt + 1 : 3;
    memset(u, 0, sizeof(double) * (size_t)(rows * g.cells));
    memset(rec_data, 0, sizeof(double) * (size_t)(p->nt * p->nrec));
    for (long t = 2; t < p->nt; ++t) {
        const long s0 = save ? t : t % 3, s1 = save ? t - 1 : (t - 1) % 3,
                   s2 = save ? t - 2 : (t - 2) % 3;
        double* out = u + s0 * g.cells;
        sweep(&g, p->dt, out, u + s1 * g.cells, u + s2 * g.cells, m, damp);
        inject(&g, out, m, p->nsrc, src_idx, src_w, src_data + (t - 1) * p->nsrc, p->dt * p->dt);
        sample(&g, out, p->nrec, rec_idx, rec_w, rec_data + t * p->nrec);
    }
    return 0;
}

/* seismic.cpp:382-426 with build_adjoint_ir (seismic.cpp:269-296):
 * for t = nt-1 .. 2: sweep v[t] from v[t+1], v[t+2]; inject rec[t]; sample src[t-1]. */
int sfdo_adjoint(const sfdo_problem* p, double* v, const double* m, const double* damp,
                 const long* src_idx, const double* src_w, double* src_data,
                 const long* rec_idx, const double* rec_w, const double* rec_data) {
    geom g;
    if (make_geom(p, &g)) return 1;
    memset(v, 0, sizeof(double) * (size_t)(3 * g.cells));
    memset(src_data, 0, sizeof(double) * (size_t)(p->nt * p->nsrc));
    for (long t = p->nt - 1; t >= 2; --t) {
        double* out = v + (t % 3) * g.cells;
        sweep(&g, p->dt, out, v + ((t + 1) % 3) * g.cells, v + ((t + 2) % 3) * g.cells, m, damp);
        inject(&g, out, m, p->nrec, rec_idx, rec_w, rec_data + t * p->nrec, p->dt * p->dt);
        sample(&g, out, p->nsrc, src_idx, src_w, src_data + (t - 1) * p->nsrc);
    }
    return 0;
}

/* seismic.cpp:428-496 with build_gradient_ir (seismic.cpp:298-331): the
 * adjoint sweep fused with grad += -(1/dt^2) v[t+1] (u[t+1] - 2u[t] + u[t-1]),
 * then the host row-2 term grad -= v[2] u[2] / dt^2 over the updated region. */
int sfdo_gradient(const sfdo_problem* p, double* v, const double* u, const double* m,
                  const double* damp, double* grad, const long* rec_idx, const double* rec_w,
                  const double* rec_data) {
    geom g;
    if (make_geom(p, &g)) return 1;
    memset(v, 0, sizeof(double) * (size_t)(3 * g.cells));
    memset(grad, 0, sizeof(double) * (size_t)g.cells);
    const double idt2 = 1.0 / (p->dt * p->dt);
    for (long t = p->nt - 1; t >= 2; --t) {
        double* out = v + (t % 3) * g.cells;
        const double* v1 = v + ((t + 1) % 3) * g.cells;
        sweep(&g, p->dt, out, v1, v + ((t + 2) % 3) * g.cells, m, damp);
        const double *up = u + (t + 1) * g.cells, *uc = u + t * g.cells, *um = u + (t - 1) * g.cells;
#pragma omp parallel for collapse(2) schedule(static)
        for (long i0 = g.lo[0]; i0 < g.hi[0]; ++i0)
            for (long i1 = g.lo[1]; i1 < g.hi[1]; ++i1)
                for (long i2 = g.lo[2]; i2 < g.hi[2]; ++i2) {
                    const long x = i0 * g.stride[0] + i1 * g.stride[1] + i2 * g.stride[2];
                    grad[x] += -idt2 * v1[x] * (up[x] - 2.0 * uc[x] + um[x]);
                }
        inject(&g, out, m, p->nrec, rec_idx, rec_w, rec_data + t * p->nrec, p->dt * p->dt);
    }
    const double* v2 = v + (2 % 3) * g.cells;
    const double* u2 = u + 2 * g.cells;
    for (long i0 = g.lo[0]; i0 < g.hi[0]; ++i0)
        for (long i1 = g.lo[1]; i1 < g.hi[1]; ++i1)
            for (long i2 = g.lo[2]; i2 < g.hi[2]; ++i2) {
                const long x = i0 * g.stride[0] + i1 * g.stride[1] + i2 * g.stride[2];
                grad[x] -= v2[x] * u2[x] / (p->dt * p->dt);
            }
    return 0;
}

/* Masked variants of inject / sample for the decomposition harness. */
static void inject_masked(const geom* g, double* field, const double* m, long npts,
                          const long* idx, const double* w, const double* row, double scale,
                          const unsigned char* cmask) {
    const int corners = 1 << g->nd;
    for (long p = 0; p < npts; ++p)
        for (int c = 0; c < corners; ++c) {
            if (cmask && !cmask[p * corners + c]) continue;
            const long a = corner_offset(g, idx + p * g->nd, c);
            double v = w[p * corners + c];
            v *= scale;
            v *= row[p];
            v /= m[a];
            field[a] += v;
        }
}

int sfdo_forward_steps(const sfdo_problem* p, double* u, const double* m, const double* damp,
                       const long* src_idx, const double* src_w, const double* src_data,
                       const unsigned char* src_cmask, const long* rec_idx, const double* rec_w,
                       double* rec_data, const unsigned char* rec_mask, long t_begin,
                       long t_end) {
    geom g;
    if (make_geom(p, &g)) return 1;
    const int corners = 1 << g.nd;
    for (long t = t_begin; t < t_end; ++t) {
        double* out = u + (t % 3) * g.cells;
        sweep(&g, p->dt, out, u + ((t - 1) % 3) * g.cells, u + ((t - 2) % 3) * g.cells, m, damp);
        inject_masked(&g, out, m, p->nsrc, src_idx, src_w, src_data + (t - 1) * p->nsrc,
                      p->dt * p->dt, src_cmask);
        if (!rec_data) continue;
        for (long q = 0; q < p->nrec; ++q) {
            if (rec_mask && !rec_mask[q]) continue;
            double acc = 0.0;
            for (int c = 0; c < corners; ++c) {
                const double term =
                    rec_w[q * corners + c] * out[corner_offset(&g, rec_idx + q * g.nd, c)];
                acc = c == 0 ? term : acc + term;
            }
            rec_data[t * p->nrec + q] = acc;
        }
    }
    return 0;
}

int sfdo_sample_row(const sfdo_problem* p, const double* u, long t, const long* rec_idx,
                    const double* rec_w, double* rec_data, const unsigned char* rec_mask) {
    geom g;
    if (make_geom(p, &g)) return 1;
    const int corners = 1 << g.nd;
    const double* f = u + (t % 3) * g.cells;
    for (long q = 0; q < p->nrec; ++q) {
        if (rec_mask && !rec_mask[q]) continue;
        double acc = 0.0;
        for (int c = 0; c < corners; ++c) {
            const double term = rec_w[q * corners + c] * f[corner_offset(&g, rec_idx + q * g.nd, c)];
            acc = c == 0 ? term : acc + term;
        }
        rec_data[t * p->nrec + q] = acc;
    }
    return 0;
}
