/* TEST INFRASTRUCTURE ONLY — the CPU oracle.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / reference legs may load it, and only as the
 * checker or the timed CPU baseline; the product library never links it.
 *
 * A plain-C, fp64 restatement of the reference's hot path (stencilfd,
 * /root/reference/proj).  Parity pinned against the reference itself: the
 * golden fixtures in tests/golden/ were produced by the unmodified reference
 * (oracle/_ref, tests/golden/make_golden.py) and tests/test_oracle.py checks
 * this restatement against them.
 *
 * Conventions (reference lowering.hpp:37-39, seismic.hpp:73-79): row-major,
 * last dimension fastest; time-major u[slot][d0][d1][d2]; sparse data[t][p];
 * idx[p][ndim] (padded frame); w[p][2^ndim] with corner bit (ndim-1-d) -> +1
 * along dim d (codegen.cpp:419-424, interpreter.cpp:118).
 */
#ifndef SFD_ORACLE_H
#define SFD_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Problem descriptor: what the reference bakes into its generated source. */
typedef struct {
    int ndim;          /* 2 or 3 (1 also works) */
    long padded[3];    /* padded extents, d0 slowest */
    int space_order;   /* even, >= 2 */
    long nt;           /* trace samples; loop spans written slots [2, nt) */
    double dt, h;
    long nsrc, nrec;
} sfdo_problem;

/* fd_coefficients(2, so) taps, w[0..so]; offset k-so/2 (fd.cpp:8-60). */
int sfdo_fd2(int so, double* w);
/* Damping field over the padded grid (seismic.cpp:47-62,152-173). */
void sfdo_damping(int ndim, const long* padded, long nbpml, long halo, double h, double* out);
/* Padded model with edge replication (seismic.cpp:100-142). */
int sfdo_make_model(int ndim, const long* interior, double h, long nbpml, int so,
                    const double* m_interior, long* padded, double* m, double* damp);
/* seismic.cpp:195-230 */
int sfdo_locate(int ndim, const long* interior, double h, long nbpml, int so, long npts,
                const double* coords, long* idx, double* w);
/* seismic.cpp:175-185 */
void sfdo_ricker(double f0, double t0, long nt, double dt, double* out);
/* seismic.cpp:187-193 */
double sfdo_critical_dt(int ndim, double h, int so, double m_min);

/* Operators at the generated-kernel level (argv semantics, codegen.cpp:247-265).
 * All grids are zeroed first (first touch, codegen.cpp:464-492).
 * forward: u rows = save ? nt+1 : 3; rec_data [nt][nrec] is written for t in [2,nt). */
int sfdo_forward(const sfdo_problem* p, int save, double* u, const double* m, const double* damp,
                 const long* src_idx, const double* src_w, const double* src_data,
                 const long* rec_idx, const double* rec_w, double* rec_data);
/* adjoint: v 3 slots; src_data [nt][nsrc] written for t-1, t in [2,nt). */
int sfdo_adjoint(const sfdo_problem* p, double* v, const double* m, const double* damp,
                 const long* src_idx, const double* src_w, double* src_data,
                 const long* rec_idx, const double* rec_w, const double* rec_data);
/* gradient: v 3 slots; u history (nt+1) rows; grad cells (zeroed here), includes the
 * host-side row-2 term of seismic.cpp:468-490. */
int sfdo_gradient(const sfdo_problem* p, double* v, const double* u, const double* m,
                  const double* damp, double* grad, const long* rec_idx, const double* rec_w,
                  const double* rec_data);

/* Forward time steps t in [t_begin, t_end) on an already initialised rolling
 * field (no zeroing), with optional per-corner injection masks and
 * per-receiver sampling masks (NULL = all); rec_data NULL skips sampling.
 * Test harness for the z-slab decomposition: ranks step their slabs and
 * exchange ghost planes between calls. */
int sfdo_forward_steps(const sfdo_problem* p, double* u, const double* m, const double* damp,
                       const long* src_idx, const double* src_w, const double* src_data,
                       const unsigned char* src_cmask, const long* rec_idx, const double* rec_w,
                       double* rec_data, const unsigned char* rec_mask, long t_begin,
                       long t_end);

/* rec_data[t][q] = sum_c w u[t%3][corner] for receivers with rec_mask[q]. */
int sfdo_sample_row(const sfdo_problem* p, const double* u, long t, const long* rec_idx,
                    const double* rec_w, double* rec_data, const unsigned char* rec_mask);

#ifdef __cplusplus
}
#endif
#endif
