/*
 * sfdb200 — B200 (sm_100a) backend for the damped acoustic stencil hot path
 * of stencilfd (/root/reference/proj), exported as a plain C ABI.
 *
 * The reference executes each operator as ONE call of a JIT-compiled C kernel
 * through the uniform trampoline `int <Name>_call(void **argv)`
 * (proj/src/codegen.cpp:598-607, resolved by dlsym in proj/src/runtime.cpp:246-248,
 * stored as `int (*call)(void**)` in runtime::CompiledKernel, runtime.hpp:65-71).
 * Its problem constants (extents, halo, nt, dt, h, FD taps) are baked into the
 * generated source; here they travel in an sfdb200_desc instead, and
 * sfdb200_call(desc, argv) is the drop-in for `<Name>_call(argv)` with the SAME
 * argv layout (codegen::signature, proj/src/codegen.cpp:247-265):
 *
 *   Forward  (seismic.cpp:241-267): u, m, damp, src_idx, src_w, src_data, rec_idx, rec_w, rec_data
 *   Adjoint  (seismic.cpp:269-296): v, m, damp, src_idx, src_w, src_data, rec_idx, rec_w, rec_data
 *   Gradient (seismic.cpp:298-331): v, u, m, damp, grad, rec_idx, rec_w, rec_data
 *   (+ optional trailing block-size `long*` args, accepted and ignored)
 *
 * Grids are host `double*` in the reference's padded row-major layout, sparse
 * indices `long*` [npoints][ndim], weights `double*` [npoints][2^ndim], traces
 * `double*` [nt][npoints].  Results are written in place like the reference
 * kernel (u/v slots, sampled traces, grad).  Return 0 on success; non-zero is
 * an error code with a thread-local message (sfdb200_last_error), which the
 * reference's runtime::run turns into RuntimeError (runtime.cpp:344-345).
 *
 * Semantics follow the generated kernel, including first-touch zeroing of the
 * written grids (codegen.cpp:464-492); for Gradient, `grad` by default also
 * holds the host-side row-2 term of seismic::gradient (seismic.cpp:468-490),
 * i.e. it is final, unless desc.flags has SFDB200_F_GRAD_NO_ROW2 (then it is
 * exactly what the generated Gradient kernel leaves for its caller).
 * Arithmetic is fp32 on the device (see DESIGN.md for the error budget).
 */
#ifndef SFDB200_H
#define SFDB200_H

#if defined(__GNUC__)
#define SFDB200_API __attribute__((visibility("default")))
#else
#define SFDB200_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum sfdb200_kind { SFDB200_FORWARD = 0, SFDB200_ADJOINT = 1, SFDB200_GRADIENT = 2 };

enum sfdb200_status {
    SFDB200_OK = 0,
    SFDB200_EINVAL = 1,   /* bad descriptor / argument (reference: std::invalid_argument) */
    SFDB200_ECUDA = 2,    /* CUDA runtime or driver failure */
    SFDB200_ENOMEM = 3,   /* device allocation failed */
    SFDB200_ENONFINITE = 4 /* non-finite output (reference: check_finite, seismic.cpp:39-44) */
};

/* What the reference bakes into the generated source (lowering.hpp:61-87). */
typedef struct sfdb200_desc {
    int kind;            /* sfdb200_kind */
    int ndim;            /* 2 or 3; d0 = z (slowest) */
    long padded[3];      /* padded extents n + 2*(nbpml + so/2) (seismic.hpp:29-31) */
    int space_order;     /* even, 2..16 */
    long nt;             /* trace samples; written slots [2, nt) (lowering.hpp:78-80) */
    double dt, h;
    long nsrc, nrec;     /* sparse-set sizes (Gradient: nsrc ignored) */
    int save;            /* Forward only: u holds nt+1 history rows (seismic.hpp:91-93) */
    int device;          /* CUDA device ordinal */
    int flags;           /* SFDB200_F_* (0: the operator-level semantics above) */
} sfdb200_desc;

/* Gradient: leave out the t = 2 term of the imaging condition, exactly as the
 * reference's generated Gradient kernel does: its caller seismic::gradient
 * adds grad -= v[2] u[2] / dt^2 over the updated region on the host
 * (seismic.cpp:468-490).  The shim the JIT driver emits for a generated
 * Gradient kernel sets it (bin/sfdb200-jit), so the
 * drop-in `Gradient_call` returns what the reference kernel returns. */
#define SFDB200_F_GRAD_NO_ROW2 1

typedef struct sfdb200_plan sfdb200_plan;

/* ---- reference-ABI entry points ---------------------------------------- */

/* Drop-in for `<Name>_call(void **argv)`: plans are cached per descriptor. */
SFDB200_API int sfdb200_call(const sfdb200_desc* desc, void** argv);

/* Explicit plan lifecycle (device buffers, streams, tensor maps). */
SFDB200_API int sfdb200_plan_create(const sfdb200_desc* desc, sfdb200_plan** out);
SFDB200_API int sfdb200_plan_destroy(sfdb200_plan* plan);
/* upload + execute + download, argv as above. */
SFDB200_API int sfdb200_run(sfdb200_plan* plan, void** argv);

/* ---- staged execution (device-resident timing) -------------------------- */

/* H2D + fp64->fp32 conversion of every input in argv (model, sparse sets,
 * traces; Gradient: the u history). */
SFDB200_API int sfdb200_upload(sfdb200_plan* plan, void** argv);
/* The whole device-resident time loop on the plan's stream; no host sync. */
SFDB200_API int sfdb200_execute(sfdb200_plan* plan);
/* D2H + fp32->fp64 of every output into argv; synchronises the stream. */
SFDB200_API int sfdb200_download(sfdb200_plan* plan, void** argv);
/* Gradient plans: take the u history from a saved Forward plan's device
 * buffer (same problem) instead of uploading a host copy. */
SFDB200_API int sfdb200_bind_history(sfdb200_plan* gradient_plan, const sfdb200_plan* forward_plan);

/* ---- history storage by uniform checkpointing -------
 * The reference keeps the whole saved history (spilling it to an mmap'd file,
 * proj/src/runtime.cpp:122-169).  A 3-D single-GPU Forward plan (save = 0)
 * with an interval k > 0 instead keeps rows u[jk], u[jk+1] (j >= 1) during
 * execute(); a Gradient plan bound to it recomputes each k-step segment of the
 * history from those rows (one extra forward sweep per step) into a k+2-row
 * buffer while it runs backwards.  Device memory: 2 (ceil((nt-2)/k) - 1) + k + 2
 * rows instead of nt + 1.  The gradient plan's argv[1] (u history) is ignored.
 * interval 0 turns checkpointing off. */
SFDB200_API int sfdb200_set_checkpointing(sfdb200_plan* forward_plan, long interval);
SFDB200_API int sfdb200_bind_checkpoints(sfdb200_plan* gradient_plan, sfdb200_plan* forward_plan);
/* Device bytes the checkpoint store and one segment buffer take (0 if off). */
SFDB200_API long sfdb200_checkpoint_bytes(const sfdb200_plan* forward_plan);
/* Launch on a caller stream (a cudaStream_t passed as void*); 0 = plan's own. */
SFDB200_API int sfdb200_set_stream(sfdb200_plan* plan, void* cuda_stream);
/* When on, execute() brackets every stencil launch with CUDA events. */
SFDB200_API int sfdb200_set_timing(sfdb200_plan* plan, int on);
/* Stencil-kernel time of the last timed execute(): total ms and launches. */
SFDB200_API int sfdb200_stencil_time(sfdb200_plan* plan, double* total_ms, long* launches);
/* Kernels launched by one execute() (stencil + sparse + bookkeeping). */
SFDB200_API long sfdb200_launches_per_execute(const sfdb200_plan* plan);
/* Updated points per step ((n + 2 nbpml)^ndim, lowering.cpp:111-121) and steps (nt-2). */
SFDB200_API long sfdb200_points_per_step(const sfdb200_plan* plan);
SFDB200_API long sfdb200_steps(const sfdb200_plan* plan);
/* The 3-D sweep configuration chosen for this plan, as a JSON object. */
SFDB200_API int sfdb200_plan_info(const sfdb200_plan* plan, char* buf, long len);
/* Host<->device bytes moved by upload()/download() for this plan. */
SFDB200_API long sfdb200_h2d_bytes(const sfdb200_plan* plan);
SFDB200_API long sfdb200_d2h_bytes(const sfdb200_plan* plan);

/* ---- multi-GPU: z-slab decomposition -------------------
 * One process per GPU.  Every rank creates a communicator from the same
 * 128-byte unique id (made by rank 0, shared by the caller, e.g. through
 * torch.distributed), then a plan for the GLOBAL problem: the rank keeps the
 * planes [z_begin, z_end) of the updated z range (sfdb200_slab) plus so/2
 * ghost planes a side, sweeps the so/2 planes next to each neighbour first and
 * exchanges them (NCCL send/recv on its own stream) while the interior runs.
 * upload() takes the global host arrays; download() writes the rank's owned
 * planes of u / v / grad and its owned receivers' trace columns (others are
 * left zero: summing the traces over ranks assembles the record). */
typedef struct sfdb200_comm sfdb200_comm;
SFDB200_API int sfdb200_comm_unique_id(void* id128);
SFDB200_API int sfdb200_comm_create(const void* id128, int world, int rank, int device,
                                    sfdb200_comm** out);
SFDB200_API int sfdb200_comm_destroy(sfdb200_comm* comm);
/* Test harness for one GPU: `world` emulated ranks in one process (no NCCL).
 * Their plans must share one stream (sfdb200_set_stream) and run together
 * through sfdb200_execute_group, which does the ghost exchange as device
 * copies between the plans, phase by phase in lockstep. */
SFDB200_API int sfdb200_comm_create_loopback(int world, int rank, int device,
                                             sfdb200_comm** out);
SFDB200_API int sfdb200_execute_group(sfdb200_plan** plans, int n);
SFDB200_API int sfdb200_plan_create_dist(const sfdb200_desc* global_desc, sfdb200_comm* comm,
                                         sfdb200_plan** out);
/* Fused P2P ghost exchange over NVLink (the default multi-GPU path when peer
 * access is available): a step is one sweep launch whose first
 * items are the boundary tiles; they write their planes (after their
 * injections) straight into the neighbours' ghost planes through CUDA IPC
 * mappings of the neighbours' field rows and publish the step into the
 * neighbours' step counters, while the interior items keep computing; a
 * one-thread poll kernel waits on the counters before the next step.  No NCCL
 * call remains on the data path.
 * sfdb200_plan_ipc_export fills SFDB200_IPC_BYTES bytes for the caller to pass
 * to the neighbours (e.g. all-gathered through torch.distributed);
 * sfdb200_plan_ipc_import opens the lower / upper neighbour's blob (NULL at a
 * slab end) and switches the plan to the P2P exchange.  It returns
 * SFDB200_EINVAL, leaving the NCCL exchange in place, when a neighbour's
 * device is not peer-accessible. */
#define SFDB200_IPC_BYTES 256
SFDB200_API int sfdb200_plan_ipc_export(const sfdb200_plan* plan, void* out);
SFDB200_API int sfdb200_plan_ipc_import(sfdb200_plan* plan, const void* lower, const void* upper);
/* Loopback harness: the emulated ranks of sfdb200_execute_group use the same
 * fused launch and peer stores into each other's field rows (one device, no
 * IPC; the lockstep phases of execute_group order the steps).  Call before
 * upload (the sparse tables depend on the boundary items). */
SFDB200_API int sfdb200_plan_peer_group(sfdb200_plan** plans, int n);
/* The step-counter primitives of the P2P exchange on one device: a stream
 * writes a counter (cuStreamWriteValue32) and waits for it (poll kernel, GEQ);
 * a counter that never arrives marks the exchange broken after the timeout. */
SFDB200_API int sfdb200_p2p_selftest(int device);
/* Waits for the plan's stream and reports a broken P2P exchange: a neighbour's
 * step counter that did not arrive within SFDB200_P2P_TIMEOUT_MS (default
 * 60000) makes the waits give up (no hang, no trap) and this call, like
 * sfdb200_download, return SFDB200_ECUDA; the plan's results are invalid.
 * SFDB200_OK otherwise (also for plans without the P2P exchange). */
SFDB200_API int sfdb200_plan_check(sfdb200_plan* plan);
/* Aborts the P2P exchange now (not in stream order): sets this rank's and
 * both neighbours' sticky broken flags, so waits already parked on any of them
 * return, later sweeps skip their peer stores and step publications, and
 * sfdb200_plan_check / sfdb200_download of every rank in the chain return
 * SFDB200_ECUDA.  For a caller that hits an error on one rank mid-run (the
 * neighbours fail within a step instead of after the P2P timeout).  Also
 * works on the loopback peer group.  SFDB200_EINVAL without a P2P exchange. */
SFDB200_API int sfdb200_plan_abort(sfdb200_plan* plan);
/* Owned updated global planes of `rank`: an even split of [so/2, Pz - so/2). */
SFDB200_API int sfdb200_slab(long padded_z, int space_order, int world, int rank, long* z_begin,
                             long* z_end);
/* Which sparse corners (injection) and points (sampling, by base plane) the
 * plan of `rank` owns, for global indices idx [npoints][ndim]; either output
 * may be NULL.  Every corner / point is owned by exactly one rank. */
SFDB200_API int sfdb200_slab_owns(long padded_z, int space_order, int world, int rank,
                                  long npoints, int ndim, const long* idx,
                                  unsigned char* corner_owned, unsigned char* point_owned);
/* The plan's owned planes and the global index of its local plane 0. */
SFDB200_API int sfdb200_plan_slab(const sfdb200_plan* plan, long* z_begin, long* z_end,
                                  long* zoff);

/* ---- host helpers mirroring sfd::seismic (bit-exact with the reference) -- */

/* fd_coefficients(2, so) as doubles, w[0..so] for offsets -so/2..so/2 (fd.cpp:8-60). */
SFDB200_API int sfdb200_fd2(int space_order, double* w);
/* make_model: padded extents, m (edge-replicated), damp (seismic.cpp:100-173). */
SFDB200_API int sfdb200_make_model(int ndim, const long* interior, double h, long nbpml, int space_order,
                       const double* m_interior, long* padded, double* m, double* damp);
/* build_damping (seismic.cpp:47-62,152-173): per-cell max of the axis tapers. */
SFDB200_API int sfdb200_build_damping(int ndim, const long* padded, long nbpml, long halo,
                                      double h, double* out);
/* locate_points (seismic.cpp:195-230): idx [n][ndim] (padded frame), w [n][2^ndim]. */
SFDB200_API int sfdb200_locate_points(int ndim, const long* interior, double h, long nbpml,
                          int space_order, long npoints, const double* coords, long* idx,
                          double* w);
/* The upload's host check: 1 when the 3-D damp field [Pz][Py][Px]
 * equals max(prof[z], prof[Pz + y], prof[Pz + Py + x]) bit for bit with the
 * profiles (Pz + Py + Px doubles, written) taken through the centre's per-axis
 * minima, i.e. the reference's build_damping form; 0 otherwise (the device
 * check over the uploaded field then decides); < 0 on bad arguments. */
SFDB200_API int sfdb200_damp_separable(const double* damp, long Pz, long Py, long Px, double* prof);
/* ricker (seismic.cpp:175-185) and critical_dt (seismic.cpp:187-193). */
SFDB200_API int sfdb200_ricker(double f0, double t0, long nt, double dt, double* out);
SFDB200_API double sfdb200_critical_dt(int ndim, double h, int space_order, double m_min);

/* objective (seismic.cpp:498-510): *phi = 1/2 sum_i (syn[i] - obs[i])^2 in
 * element order (bit-equal to the reference); residual (may be NULL) gets
 * syn - obs.  n = nt * npoints. */
SFDB200_API int sfdb200_objective(const double* syn, const double* obs, long n, double* residual,
                                  double* phi);

SFDB200_API const char* sfdb200_last_error(void);
SFDB200_API const char* sfdb200_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SFDB200_H */
