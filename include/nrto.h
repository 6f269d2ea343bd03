/*
 * nrto.h -- C ABI of the B200-native NRTO inner solver (libnrto.so).
 *
 * Solves, for a batch of independent robust trajectory-optimization problem
 * instances, the SOCP subproblem of one successive-linearization (SL)
 * iteration of cuNRTO (arXiv 2603.02642):
 *
 *   Problem 2
 *     min  sum_k (u_hat_k + du_k)^T R_u^k (u_hat_k + du_k) + 1/2 k_v^T Q_v k_v
 *     s.t. g_j + b_j^T du + p_j <= 0                       (g^lin,1; DESIGN R1)
 *          || A_hat_j k_v + b_hat_j ||_2 <= p_j            j = 1..n_g
 *          || F_u du ||_2 <= r_trust
 *
 * with two engines:
 *   NRTO_FULLADMM  Algorithm 1: Block-1 SOC projection (13),
 *                  Block-2 QP (14a) and gain update (14b), dual update (16).
 *   NRTO_DR        the NRTO inner ADMM (5a)-(5c) whose (5a)
 *                  subproblem (7) is solved by relaxed Douglas-Rachford
 *                  (11a)-(11c) with the affine prox of P:930-964.
 *
 * The data of Problem 2 (F_u, F_zeta, A_hat_j, b_hat_j, Q_v; SM §I)
 * is built ON THE DEVICE by nrto_setup from the SL-iteration primitives below
 * (Jacobians, constraint gradients, Psi, weights).  Workload assumption
 * (P:1483-1486): Gamma = I and S = blkdiag(S_0, ..., S_T), i.e. Psi is given
 * as T+1 diagonal blocks Psi_k with Psi_k^T Psi_k = S_k^{-1}.
 *
 * Conventions
 *   - All floating point is IEEE binary64 (double).  Precision of the paper is
 *     unstated (DESIGN R17).
 *   - Arrays are batch-major and instance-contiguous: X[b][...] with b in
 *     [0, batch).  Matrices are row-major unless stated.  k_v is column-major
 *     vec of K_k per time step: kv[b][k*n_u*n_x + i*n_u + m]
 *     = (K_k)[m][i].
 *   - Cone j is "state" (kind 0: g_j(x_{k_j}) <= 0, knot k_j in 1..T) or
 *     "control" (kind 1: h_j linear in u_k, knot = k in 0..T-1; DESIGN R14).
 *   - Ragged cone rows: state cone j stores the blocks 0..k_j of
 *     its n_z = (T+1) n_x vector ((k_j+1) n_x doubles; blocks k > k_j are
 *     identically zero); control cone j stores block k (n_x
 *     doubles).  nrto_layout returns the offsets; E = total length.
 *   - Calls are enqueued on the stream they are given (a cudaStream_t passed
 *     as void*, NULL = legacy default stream); results are valid after the
 *     stream syncs.  Internally nrto_inner_solve may run work on handle-owned
 *     streams (the overlapped QP, the control-cone kernel) and, for
 *     fixed-iteration solves without profiling, replay a CUDA graph of the
 *     whole iteration loop that it captured on an earlier call with the same
 *     device state; all of it is joined back to `stream` by events before the
 *     call's outputs are written.
 *   - Calls that BLOCK THE HOST (synchronise):
 *       nrto_setup        shape upload (synchronous cudaMemcpy) and the SPD
 *                         check of the setup factors (stream sync);
 *       nrto_refresh      the SPD check (stream sync after the setup kernels);
 *       nrto_inner_solve  with termination on (fixed_iters == 0): one device
 *                         -> host read of the active-instance count every
 *                         check_every outer iterations; the first DR solve
 *                         after a setup/refresh (SPD check of the DR factors);
 *                         any call with memory == NRTO_MEM_HOST (stream sync
 *                         after the output copies);
 *       nrto_solve_begin  the first DR use after a setup/refresh (as above);
 *       nrto_shard_cones, nrto_setup_general, nrto_profile_read, nrto_pass_bytes,
 *       nrto_case_stats_read, nrto_destroy.
 *     Everything else (fixed-iteration solves with device outputs,
 *     nrto_gain_update, nrto_soc_project, nrto_solve_iterate / _flags / _end
 *     with device outputs, nrto_dr_step) is asynchronous; nrto_buffer,
 *     nrto_set_allocator, nrto_layout, nrto_default_params touch no device.
 *   - Device memory is allocated at setup (handle-owned; cudaMalloc, or the
 *     caller's allocator after nrto_set_allocator; the first solve also
 *     allocates small staging / trace buffers with cudaMalloc) -- no
 *     allocation happens inside the iteration loop.
 *
 * Errors: functions return nrto_err; no C++ exception crosses the ABI.  On a
 * non-OK return nrto_last_error() gives a thread-local message.  Per-instance
 * non-convergence or non-finite iterates are reported in status[], never as
 * an error.
 */
#ifndef NRTO_H_
#define NRTO_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nrto_handle_s* nrto_handle;

typedef enum {
  NRTO_OK = 0,
  NRTO_EINVAL = -1,   /* bad shape / argument (dimension rule violated)          */
  NRTO_ENOTSPD = -2,  /* W_K not SPD, or a Riccati H_uu not SPD (setup error)     */
  NRTO_ECUDA = -3,    /* CUDA runtime error (message has the CUDA string)        */
  NRTO_ENOMEM = -4,   /* device allocation failed                               */
  NRTO_ESTATE = -5    /* call order violated (e.g. solve on a destroyed handle)  */
} nrto_err;

typedef enum { NRTO_FULLADMM = 0, NRTO_DR = 1 } nrto_engine;

/* per-instance outcome (status[b]) */
typedef enum { NRTO_CONVERGED = 0, NRTO_MAX_ITERS = 1, NRTO_DIVERGED = 2 } nrto_inst_status;

typedef enum { NRTO_MEM_DEVICE = 0, NRTO_MEM_HOST = 1 } nrto_mem;

/* Shape shared by every instance of a batch (host memory). */
typedef struct {
  int32_t n_x, n_u, T, n_g, batch;  /* 1 <= n_x <= 32, 1 <= n_u <= n_x, T >= 1,
                                       n_g >= 0, batch >= 1                     */
  const int32_t* cone_knot;         /* [n_g] state: k_j in 1..T; control: k in 0..T-1 */
  const int8_t* cone_kind;          /* [n_g] 0 = state row, 1 = control row      */
} nrto_shape;

/* SL-iteration primitives (read only during nrto_setup; caller-owned).
 * memory = NRTO_MEM_DEVICE: device pointers; NRTO_MEM_HOST: host pointers
 * (pinned preferred) that nrto_setup copies to the device itself.          */
typedef struct {
  int32_t memory;                   /* nrto_mem                                       */
  const double* A;                  /* [b][T][n_x][n_x]  dx_{k+1} = A_k dx_k + B_k du_k */
  const double* B;                  /* [b][T][n_x][n_u]                               */
  const double* grad;               /* [b][n_g][n_x] state: d g_j / d x_{k_j};
                                       control: h'_j in the first n_u slots          */
  const double* g0;                 /* [b][n_g] g_j(x_hat) or h_j(u_hat)              */
  const double* Psi;                /* [b][T+1][n_x][n_x] Psi_k, Psi_k^T Psi_k = S_k^-1 */
  const double* tau;                /* [b] ellipsoid radius tau > 0       */
  const double* W_K;                /* [b][T][n_u][n_u] R_K^T R_K (SPD)       */
  const double* R_u;                /* [b][T][n_u][n_u] R_u^k (SPD)                   */
  const double* u_hat;              /* [b][T][n_u]                                    */
  const double* r_trust;            /* [b] trust-region radius >= 0                   */
} nrto_data;

/* Hyper-parameters (DESIGN §4 lists the paper lines and readings). */
typedef struct {
  double rho;        /* FullADMM penalty rho                          */
  double rho_admm;   /* NRTO-ADMM penalty for the DR engine (R3)               */
  double alpha_dr;   /* DR relaxation alpha in (0,1)                   */
  double sigma_dr;   /* R_chi = sigma_dr I (R7)                                */
  double r_s;        /* R_s = r_s I (R7)                                       */
  double eps_p, eps_d;  /* r_p, r_d tolerances (R6)                */
  double eps_dr;     /* DR fixed-point residual tolerance (R8)      */
  double rho_qp, sigma_qp, alpha_qp;  /* (14a)/(5b) QP ADMM (R1)               */
  int32_t max_iter;       /* FullADMM L_max                                   */
  int32_t max_admm_iter;  /* NRTO-ADMM iterations (DR engine)                 */
  int32_t max_dr_iter;    /* DR iterations per (5a)                           */
  int32_t qp_iters;       /* QP ADMM iterations per (14a)/(5b), warm-started  */
  int32_t check_every;    /* termination test cadence (R11)                   */
  int32_t fixed_iters;    /* != 0: run exactly the maximum iteration counts   */
} nrto_params;

/* Caller-owned outputs.  Optional arrays may be NULL.                       */
typedef struct {
  int32_t memory;          /* nrto_mem of every pointer below                  */
  double* kv;              /* [b][T*n_u*n_x]  k_v (column-major vec(K_k))      */
  double* du;              /* [b][T*n_u]      delta u_hat                      */
  double* p;               /* [b][n_g]        p                                */
  double* p_tilde;         /* [b][n_g]        p~                               */
  double* lam_p;           /* [b][n_g]  FullADMM: scaled lambda_p; DR: lambda  */
  double* nu;              /* [b][E]  FullADMM nu (ragged), optional           */
  double* lam_nu;          /* [b][E]  FullADMM scaled lambda_nu, optional      */
  double* objective;       /* [b]  J of Problem 2 at (du, k_v), optional       */
  double* margin_cone;     /* [b][n_g] p~_j - ||A_hat_j k_v + b_hat_j||, opt.  */
  double* margin_lin;      /* [b][n_g] -(g_j + b_j^T du + p_j), optional       */
  int32_t* iters;          /* [b] iterations run (ADMM iterations for DR)      */
  int32_t* status;         /* [b] nrto_inst_status                             */
  double* r_p;             /* [b] final ||p - p~||                             */
  double* r_d;             /* [b] final rho ||p~^l - p~^(l-1)||                */
  double* hist;            /* [b][L][3] optional residual trace, L = max_iter
                              (FullADMM) / max_admm_iter (DR): row l-1 holds
                              (r_p, r_d, r_dr of the last DR iteration; 0 for
                              FullADMM) after outer iteration l (P:505-507,
                              P:380-382); rows after an instance stops are 0 */
} nrto_out;

/* Fill p with the defaults of DESIGN §4 (rho=10, rho_admm=40, alpha_dr=0.9,
 * sigma_dr=1e-6, r_s=1, eps_p=eps_d=1e-3, eps_dr=1e-4, rho_qp=1,
 * sigma_qp=1e-6, alpha_qp=1.6, max_iter=40, max_admm_iter=40,
 * max_dr_iter=100, qp_iters=10, check_every=1, fixed_iters=0). */
void nrto_default_params(nrto_params* p);

/* Ragged layout (host only, no CUDA).  E_out = sum_j L_j; offsets_out, if
 * not NULL, receives n_g+1 offsets (offsets_out[j] = start of cone j).
 * NRTO_EINVAL if a knot/kind violates the rules above. */
nrto_err nrto_layout(const nrto_shape* shape, int64_t* E_out, int64_t* offsets_out);

/* Setup (S0-S2 of SURVEY §8a) for one SL iteration: uploads/reads the
 * primitives, builds on the device the ragged b_hat_{j,k}, b_{j,k} (costate
 * sweeps), the per-step gain factors of M^{-1} = Q_v + rho sum_j
 * A_hat_j^T A_hat_j (block diagonal in time, solved by a generalized
 * eigen-decomposition chain) for both engines, and the Riccati factors of the
 * QP.  All state lives in handle-owned device memory; the inputs may be freed
 * once `stream` has synchronised.  *out receives a new handle. */
nrto_err nrto_setup(const nrto_shape* shape, const nrto_data* data,
                    const nrto_params* params, void* stream, nrto_handle* out);

/* Re-runs setup on an existing handle for a new SL iteration of the same
 * shape (new linearisation, same cone structure): uploads `data` and rebuilds
 * every S0-S2 product in the handle's memory without reallocating.  The DR
 * warm state is reset.  Errors as nrto_setup. */
nrto_err nrto_refresh(nrto_handle h, const nrto_data* data, void* stream);

/* Runs the inner solve with `engine` for every instance and writes `out`.
 * FullADMM cold-starts every call (R10); the DR engine keeps its (chi~, s~)
 * warm state in the handle across calls but restarts the outer ADMM.
 * Iterations are counted per instance; a converged instance is frozen while
 * others continue (R12). */
nrto_err nrto_inner_solve(nrto_handle h, int32_t engine, const nrto_out* out,
                          void* stream);

/* Standalone (14b) for FullADMM, device pointers:
 *   kv_next = q + calM kv_prev + calMbar nu
 *           = M (Q_v kv_prev + rho sum_j A_hat_j^T (nu_j - b_hat_j))
 * nu is ragged [b][E]; kv_prev, kv_next are [b][T*n_u*n_x]. */
nrto_err nrto_gain_update(nrto_handle h, const double* nu, const double* kv_prev,
                          double* kv_next, void* stream);

/* Batched ragged SOC projection, SM Eq.(18), device pointers:
 * for cone j with row y[off[j]..off[j+1]) and scalar t[j],
 * (t_out[j], y_out[row]) = Pi_{||y|| <= t}(t[j], y[row]).  y_out may alias y. */
nrto_err nrto_soc_project(const double* t, const double* y, const int64_t* offsets,
                          int64_t n_cones, double* t_out, double* y_out, void* stream);

/* Number of kernel launches issued by this handle since creation (host
 * counter; used to report bench.py's gpu_launches). */
int64_t nrto_launch_count(nrto_handle h);

/* Kernel classes timed by the optional CUDA-event profiler. */
typedef enum {
  NRTO_K_PASS = 0,     /* fused state-cone pass: S3 forward map + S4 norms + S5 state update */
  NRTO_K_ADJOINT = 1,  /* S7 adjoint reduction / correction list                           */
  NRTO_K_GAIN = 2,     /* S8 gain chain                                                    */
  NRTO_K_QP = 3,       /* S9 QP (+ dual update, residuals S6)                              */
  NRTO_K_OTHER = 4,    /* projection decisions, DR residual reduction, resets, finish      */
  NRTO_K_CTRL = 5,     /* control-cone pass (single-block cones)                           */
  NRTO_K_COUNT = 6
} nrto_kernel_class;

/* enable != 0: every launch of a timed class is bracketed by CUDA events on
 * the launching stream; nrto_profile_read synchronises on them and returns
 * the summed device time (ms) and the launch count of `kclass` since the
 * last read (then clears that class). */
nrto_err nrto_profile_enable(nrto_handle h, int32_t enable);
nrto_err nrto_profile_read(nrto_handle h, int32_t kclass, double* total_ms, int64_t* launches);

/* Algorithmic bytes moved by the fused state-cone pass (k_fa_tma) since the
 * last call, then reset: b_hat and b of every cone block, y^{l-1} read for
 * cones with s^{l-1} != 1 and y^l written where it is needed later (DESIGN §7,
 * lazy y).  0 when the TMA pass is not in use.  Synchronises the device. */
nrto_err nrto_pass_bytes(nrto_handle h, int64_t* bytes);

/* General uncertainty set: zeta = Gamma z with
 * z^T S z <= tau, Gamma in R^{(T+1) n_x x n_z}, S dense SPD, so A_hat_j =
 * sqrt(tau) Psi Gamma^T [A_bar_j; 0] and b_hat_j = sqrt(tau) Psi Gamma^T F_zeta^T
 * grad g_j couple all time blocks.  memory: as nrto_data.
 *   Gamma [b][(T+1) n_x][n_z] row-major;  Psi [b][n_z][n_z] with Psi^T Psi = S^-1. */
typedef struct {
  int32_t memory;
  int32_t n_z;
  const double* Gamma;
  const double* Psi;
} nrto_uncertainty;

/* Setup for a general set: as nrto_setup (data->Psi is ignored; data->tau is
 * used), plus the dense gain system M^-1 = Q_v + rho sum_j A_hat_j^T A_hat_j
 * formed on the device and factored by Cholesky once (T n_u n_x <=
 * 4096).  The handle supports nrto_inner_solve with NRTO_FULLADMM only (in-order
 * schedule); its nu / lam_nu outputs are DENSE [b][n_g][n_z] rows.
 * nrto_refresh / nrto_gain_update return NRTO_EINVAL on it; the DR engine too.
 * Errors as nrto_setup; NRTO_ENOTSPD if a Cholesky pivot of M^-1 is <= 0.
 * Synchronises the host. */
nrto_err nrto_setup_general(const nrto_shape* shape, const nrto_data* data,
                            const nrto_uncertainty* unc, const nrto_params* params,
                            void* stream, nrto_handle* out);

/* Incremental driving of the inner solve, for callers that interleave their
 * own work between outer iterations -- e.g. the batch-wide allreduce(MAX) of
 * the residual flags across ranks (one process per GPU, instances sharded;
 * SURVEY §8e), the multi-GPU form of the termination test of Algorithm 1
 * line 9 / P:505-507.  Same kernels and arithmetic as the in-order
 * schedule of nrto_inner_solve (termination mode); every call is asynchronous
 * on `stream` (no host synchronisation):
 *   nrto_solve_begin    reset for `engine` (FullADMM cold start R10; DR keeps
 *                       its warm state); no residual trace / case stats
 *   nrto_solve_iterate  run up to n_iters more outer iterations (capped at
 *                       max_iter / max_admm_iter); *done (host, may be NULL)
 *                       receives the outer iterations run so far.  Converged /
 *                       diverged instances stay frozen (R12).
 *   nrto_solve_flags    flags[4] (DEVICE doubles) = [max_b r_p/eps_p,
 *                       max_b r_d/eps_d, #active instances, any diverged]
 *                       (NaN propagates through the maxima)
 *   nrto_solve_end      finish (nu, lam_nu, margins, objective) and write `out`
 *                       exactly as nrto_inner_solve does.
 * NRTO_ESTATE if called out of order. */
nrto_err nrto_solve_begin(nrto_handle h, int32_t engine, void* stream);
nrto_err nrto_solve_iterate(nrto_handle h, int32_t n_iters, int32_t* done, void* stream);
nrto_err nrto_solve_flags(nrto_handle h, double* flags, void* stream);
nrto_err nrto_solve_end(nrto_handle h, const nrto_out* out, void* stream);

/* Projection-case statistics of the FullADMM engine (SM Eq.(18), P:992-1002;
 * the three cases of Fig. 3).  enable != 0: every later FullADMM
 * solve counts, per outer iteration l = 1..max_iter, the cones (over the whole
 * batch) whose Block-1 projection (13) fell in case 1 (||y|| <= t: kept),
 * case 2 (||y|| <= -t: origin) or case 3 (boundary).  Counting costs a few
 * warp-aggregated atomics per projection kernel.  nrto_case_stats_read copies
 * the counts of the LAST FullADMM solve into counts[L][3] (host int64, row l-1
 * = iteration l; rows the solve did not reach are 0) and synchronises the
 * device.  NRTO_EINVAL for counts == NULL or L < 0. */
nrto_err nrto_case_stats_enable(nrto_handle h, int32_t enable);
nrto_err nrto_case_stats_read(nrto_handle h, int64_t* counts, int32_t L);

/* Cone sharding of ONE instance over ranks: a handle set
 * up on the whole problem (nrto_setup) keeps the setup, the gain factors and the
 * QP over all rows (replicated on every rank), but after nrto_shard_cones its DR
 * pass and adjoint cover cones [cone_lo, cone_hi) only (cone_lo <= cone_hi <=
 * n_g; NRTO_EINVAL otherwise or for a general-set handle).  Synchronises the
 * device.  Such a handle is driven by the NRTO-ADMM + DR engine through
 *   nrto_solve_begin(h, NRTO_DR, s)
 *   for l = 1..L_admm:  nrto_dr_step(h, 0, l, s)                  (arm)
 *     for m = 1..L_dr:  nrto_dr_step(h, 1, l, s)                  (affine prox (11a))
 *                       nrto_dr_step(h, 2, l, s)                  (my cones: pass (11b/c),
 *                                                                  adjoint partial, r_dr partial)
 *                       caller: allreduce(SUM) of buffer 0 (Z)    over the ranks
 *     caller: zero buffer 1 (pi) outside [cone_lo, cone_hi), allreduce(SUM) it
 *     nrto_dr_step(h, 3, l, s)                                    (QP (5b) + (5c))
 *   nrto_solve_end(h, out, s)
 * (fixed iteration counts; the DR stop test needs the r_dr partials of buffer 2
 * summed over ranks and is the caller's).  Per-instance outputs are replicated;
 * per-cone outputs are valid for the rank's own cones.  nrto_inner_solve and
 * nrto_refresh return NRTO_EINVAL on a sharded handle.  nrto_dr_step: NRTO_ESTATE outside
 * nrto_solve_begin(NRTO_DR) .. nrto_solve_end, NRTO_EINVAL for a bad phase / l;
 * asynchronous on `stream`. */
nrto_err nrto_shard_cones(nrto_handle h, int32_t cone_lo, int32_t cone_hi);
nrto_err nrto_dr_step(nrto_handle h, int32_t phase, int32_t l, void* stream);
/* Device buffers of a handle for a caller's collectives (owned by the handle):
 * which = 0: Z [b][T][n_u][n_x] adjoint accumulator; 1: pi / p~ [b][n_g];
 * 2: r_dr partial squares per cone [b][n_g].  *count = doubles. */
nrto_err nrto_buffer(nrto_handle h, int32_t which, double** ptr, int64_t* count);

nrto_err nrto_destroy(nrto_handle h);

/* Workspace allocator ("an allocator hook lets the torch caching
 * allocator back it").  By default a handle's device workspace -- everything
 * nrto_setup / nrto_setup_general allocate for the handle's lifetime, ~70 KB per
 * Franka instance plus the O(E) cone arrays -- comes from cudaMalloc / cudaFree.
 * After nrto_set_allocator(alloc, release, ctx) every NEW handle allocates it with
 * alloc(ctx, bytes, stream) (a device pointer, or NULL on failure ->
 * NRTO_ENOMEM) and returns it with release(ctx, ptr, stream) in nrto_destroy (or
 * on a failed setup); `stream` is the setup stream.  The callbacks are called on
 * the calling thread, must not call back into nrto, and must keep the memory
 * valid until release.  Existing handles keep the allocator they were created
 * with.  alloc == NULL restores cudaMalloc / cudaFree.  Process-wide; not
 * thread-safe against concurrent setups.  Small internal scratch (staging of
 * host outputs, traces) stays on cudaMalloc. */
typedef void* (*nrto_alloc_fn)(void* ctx, size_t bytes, void* stream);
typedef void (*nrto_free_fn)(void* ctx, void* ptr, void* stream);
nrto_err nrto_set_allocator(nrto_alloc_fn alloc, nrto_free_fn release, void* ctx);

/* Thread-local message for the last non-OK return (never NULL). */
const char* nrto_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* NRTO_H_ */
