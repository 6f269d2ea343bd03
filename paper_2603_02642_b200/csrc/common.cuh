// Internal declarations of libnrto (not part of the ABI; see include/nrto.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <vector>
#include "../../include/nrto.h"

// slots of the QP's per-step bulk-copy ring for Acl_k (qp.cu); the TMA pass
// leaves room for one QP CTA of this size beside it (tma.cu)
#ifndef QP_RING
#define QP_RING 8
#endif

namespace nrto {

// Problem dimensions shared by every instance of a batch.
struct Dims {
  int nx, nu, T, ng, B;
  int64_t E;    // ragged cone-row length (sum_j L_j)
  int64_t EB;   // ragged B-data length (state: k_j nup, control: nup)
  int nup;      // B-data row stride: n_u rounded up to even (16-byte rows for TMA)
  int NK;       // T n_u n_x
};

// Factors of one engine's per-step gain chain and QP Riccati sweep.
struct EngineFactors {
  double* V;     // [B][T][nu][nu]  generalized eigenvectors of (Lambda_k, W'_k)
  double* den;   // [B][T][nu][nx]  1 / (2 + c tau sigma_a lambda_b)
  double* Kf;    // [B][T][nu][nx]  Riccati feedback of the QP x-step
  double* Acl;   // [B][T][nx][nx]  A_k - B_k Kf_k
  double* AclT;  // [B][T][nx][nx]  its transpose (row i = column i of Acl_k)
  double* Hinv;  // [B][T][nu][nu]  H_uu^{-1}
  double* HB;    // [B][T][nu][nx]  H_uu^{-1} B_k^T
  // chunked (parallel-in-time) recurrences of the QP (qp.cu k_qp_scan);
  // nullptr for large batches.  Chunk c covers steps [c M, min(T, (c+1) M) - 1]:
  double* PhiB;  // [B][T][nx][nx]  Acl_k^T Acl_{k+1}^T ... Acl_hi^T  (k in its chunk)
  double* PhiF;  // [B][T][nx][nx]  Acl_k Acl_{k-1} ... Acl_lo
};

// Plain-old-data view of all device state, passed to kernels by value.
struct Dev {
  Dims d;
  nrto_params prm;
  // shape
  const int32_t* knot; const int32_t* kind;
  const int64_t* off; const int64_t* offB;
  const int32_t* kptr; const int32_t* kcone;   // cones with a b-block at step k (k < T)
  const int32_t* sptr; const int32_t* srow;    // state rows at knot k (k = 0..T)
  const int32_t* cptr; const int32_t* crow;    // control rows at step k (k < T)
  const int32_t* qrow;   // [ng] rows in knot order: for p = 1..T state rows at knot p, then control rows at step p-1 (QP)
  // primitives (device copies)
  const double *A, *Bm, *grad, *g0, *Psi, *tau, *W, *Ru, *uhat, *rtrust;
  // setup products
  double* bhat;   // [B][E]  (control segments unused)
  double* Bd;     // [B][EB]
  double* Zb;     // [B][T][nu][nx]  sum_j b_{j,k} b_hat_{j,k}^T
  double* Lam;    // [B][T][nu][nu]  sum_j b_{j,k} b_{j,k}^T
  double* U;      // [B][T][nx][nx]  eigenvectors of Sigma_k = Psi_k^T Psi_k
  double* Ulam;   // [B][T][nx]      their eigenvalues (valid at representative steps)
  int32_t* Urep;  // [B][T]          representative step of each Psi_k run
  EngineFactors fa, dr;
  // iterate state
  double* Y;      // [B][E] FullADMM: projection input y^l; DR: eta~
  double* s;      // [B][ng] FullADMM: scale s^l of the last projection
  double* tin;    // [B][ng] FullADMM: t = p + lam_p for the next projection
  double* pt;     // [B][ng] p~ (FullADMM) / pi of the last prox (DR)
  double* ptprev; // [B][ng]
  double* p;      // [B][ng] QP x p-part (= p)
  double* lamp;   // [B][ng] FullADMM lam_p (scaled) / DR lambda (unscaled)
  double* K;      // [B][NK] k_v (column-major vec per step)
  double* Ccur;   // [B][T][nx][nu]  sqrt(tau) Psi_k K_k^T for the current k_v
  double* Cprev;  // [B][T][nx][nu]  for the previous k_v
  double* D;      // [B][T][nx][nu]  2 Ccur - Cprev (FullADMM forward map)
  double* Z;      // [B][T][nu][nx]  adjoint accumulator sum_j b (s y)^T
  double* Zg;     // [B][T][nu][nx]  nrto_gain_update's own accumulator (keeps the DR warm Z)
  // QP state
  double *du, *zl, *yl, *zb, *yb;     // [B][T][nu], [B][ng] x2, [B][T+1][nx] x2
  double *rp, *wq, *rx, *ru, *kff, *dxt, *dut;  // scratch
  // DR state
  double *Kt, *pit, *tt, *rdr_part, *rdr;
  int32_t* dr_active;
  // per-instance control
  int32_t *status, *iters, *active;
  double *r_p, *r_d;
  // fused FullADMM pass (fused.cu)
  int fused;               // 0: generic k_fa_pass + adjoint; 1: k_fa_fused_r (all tiles) +
                           // correction; 2: k_fa_tma (state tiles) + k_fa_ctrl + correction
  int nctrl;               // number of control cones
  int iter;                // outer iteration l of the launch (set by the host loop)
  double* hist;            // [B][hist_L][3] residual trace (nullptr: not requested)
  int hist_L;
  unsigned long long* case_cnt;   // [hist_L][3] projection cases 1/2/3 per iteration (nullptr: off)
  int ylazy;               // 1: lazy y storage in this iteration
  unsigned long long* pass_bytes;  // algorithmic bytes moved by k_fa_tma (device counter)
  double* nrm2;            // [B][ng] ||y^l||^2 written by the fused pass
  // TMA path predicted adjoint: Z_pred,k = c_l (G_k D_k^T + H_k) with
  // G_k = sum b b^T, H_k = sum b b_hat^T over state cones with s^{l-1} = 1.
  double* G;               // [B][T][nu][nu]
  double* H;               // [B][T][nu][nx]
  double* G0;              // [B][T][nu][nu] all state cones (setup)
  double* H0;              // [B][T][nu][nx]
  double* dG;              // [B][T][nu][nu] this iteration's leave/enter update
  double* dH;              // [B][T][nu][nx]
  int4* rowpk;             // [B][ng] packed gradient-row record (qp.cu, k_sparse_rows)
  double* cu2;             // [B][T][nu] -2 R_u u_hat (qp.cu, setup)
  double* gval;            // [B][ng][8] its nonzero values
  double* Zctrl;           // [B][T][nu][nx] exact adjoint of the control cones (fused == 2)
  int ntiles, nsplit, nwitems;
  int nsm;                 // multiprocessor count of the device (queried once at setup)
  int nstate_tiles;        // state tiles come first in `tiles`
  // TMA path: tile-interleaved copies of b_hat and b for the state tiles,
  // block-major [k][cone of tile][i] so a chunk of a tile is one bulk copy.
  int32_t* ttb;            // [nstate_tiles][2] tile base (b_hat_t, Bd_t) within an instance
  int64_t Est, EBst;       // per-instance sizes of b_hat_t / Bd_t
  double* bhat_t;          // [B][Est]
  int32_t* psame;          // [B][T] Psi_k == Psi_{k-1} (setup)
  int32_t* ktile0;         // [T+1] first state tile with knot > k (tiles ascend in knot)
  double* Bd_t;            // [B][EBst]
  const int32_t* tiles;    // [ntiles][12] kind, knot, nc, klo, cone[8]
  const int32_t* witems;   // [nwitems][4] b, t0, t1, split index
  double* Zpart;           // [B][nsplit][T][nu][nx] per-work-item adjoint partials
  double* Zc;              // [B][T][nu][nx] correction adjoint
  int32_t* clist;          // [B][ng] mispredicted cones of the last pass
  double* cw;              // [B][ng] their weights s^l - shat
  int32_t* ncorr;          // [B]
  // persistent DR loop (persist.cu); drQ = 0: not used
  int drQ;                 // cone chunks per instance
  const int32_t* drchunk;  // [drQ + 1] first cone of each chunk
  const int32_t* drkr;     // [drQ][2] steps [klo, khi) with b-blocks in the chunk
  double* drZpart;         // [B][drQ][T][nu][nx] chunk adjoint partials
  double* drrq;            // [B][drQ] chunk sums of ||s~^l - s~^{l-1}||^2
  unsigned long long* drbar;   // grid-barrier counter (zeroed by k_dr_arm)
  int drEc, drEBc;         // largest chunk: eta~ elements, b-row elements
  int scanM, scanC;        // QP recurrence chunks: length M, count C (0: no scan QP)
  // cone sharding of one instance over ranks (nrto_shard_cones, NEXT-3(i)): this
  // handle's DR pass and adjoint cover cones [cone_lo, cone_hi) only
  int cone_lo, cone_hi;
  // grid-wide QP for one large instance (qp.cu k_qp_grid): qpgrid = 1 when used
  int qpgrid;
  double* qg_s;            // [(T+1) nx] s_k
  double* qg_a;            // [T nx]     a_k, then e_k
  double* qg_part;         // [2][1024]  per-CTA partial sums
  unsigned long long* qg_bar;   // grid-barrier counter (zeroed before each launch)
};

}  // namespace nrto

namespace nrto {
// General uncertainty set state (general.cu)
struct GenState {
  int nz = 0;
  double* tau = nullptr;   // [B] the instances' tau (the regular setup ran with tau = 1)
  double* W = nullptr;     // [B][n_z][NX]  sqrt(tau) Psi Gamma^T
  double* Bh = nullptr;    // [B][n_g][n_z] b_hat_j
  double* L = nullptr;     // [B][NK][NK]   Cholesky factor of M^{-1}
  double* lam = nullptr;   // [B][n_g][n_z] scaled lam_nu
  double* nu = nullptr;    // [B][n_g][n_z]
  double* a = nullptr;     // [B][n_g][n_z] scratch: A_hat k + b_hat / nu - b_hat
  double* V = nullptr;     // [B][n_g][NX]  scratch: A_bar k + c  /  (nu - b_hat) W
  double* Cf = nullptr;    // [B][n_g][NX]  raw costates c_j (dense rows)
  double* rhs = nullptr;   // [B][NK]
  void* allocs[16];
  int nallocs = 0;
};
}  // namespace nrto

struct nrto_prof_rec { int cls; cudaEvent_t a, b; };

struct nrto_handle_s {
  nrto_alloc_fn alloc_fn = nullptr;   // workspace allocator of this handle (nullptr: cudaMalloc)
  nrto_free_fn free_fn = nullptr;
  void* alloc_ctx = nullptr;
  void* alloc_stream = nullptr;
  double* hist_buf = nullptr;   // device residual-trace buffer (grown on demand)
  size_t hist_cap = 0;
  int tma_margin = 0;      // k_fa_tma launch mode: 1 = finish margins (||C^L b + b_hat||)
  nrto::Dev dev;
  int64_t launches = 0;
  int dr_fresh = 1;
  int dr_ready = 0;        // DR engine factors built for the current setup
  void* allocs[128];
  int nallocs = 0;
  cudaStream_t stream = 0;
  // optional CUDA-event profiler (nrto_profile_enable)
  int prof = 0;
  std::vector<nrto_prof_rec> recs;
  std::vector<cudaEvent_t> pool;
  // second stream for the QP(l) || pass(l+1) overlap (fixed-iteration mode)
  cudaStream_t aux = nullptr;     // low priority: QP
  cudaStream_t hi = nullptr;      // high priority: cone pass chain
  cudaStream_t hi2 = nullptr;     // high priority: control cones beside the pass
  cudaEvent_t ev_g = nullptr, ev_c = nullptr;
  cudaEvent_t ev_proj = nullptr, ev_qp = nullptr, ev_in = nullptr, ev_out = nullptr;
  // CUDA graph of the fixed-iteration DR loop (api.cu): replayed while the device
  // state descriptor it was captured with (Dev, by value) is unchanged
  cudaStream_t gst = nullptr;
  cudaGraphExec_t dr_exec = nullptr;
  nrto::Dev dr_key;
  int64_t dr_graph_launches = 0;
  cudaGraphExec_t fa_exec = nullptr;   // same for the in-order fixed-iteration FullADMM loop
  nrto::Dev fa_key;
  int64_t fa_graph_launches = 0;
  // persistent staging for host-memory outputs and the active-count poll
  double* stage_ng2 = nullptr;   // [2][B][ng]  margins
  double* stage_b = nullptr;     // [B]         objective
  double* stage_e2 = nullptr;    // [2][B][E]   nu, lam_nu (allocated on first host request)
  int32_t* dcount = nullptr;
  int case_stats = 0;                       // nrto_case_stats_enable
  unsigned long long* case_buf = nullptr;   // [case_cap][3]
  int64_t case_cap = 0;
  int case_L = 0;                           // rows written by the last FullADMM solve
  int general = 0;                          // general (Gamma, S) set: nrto_setup_general
  int gen_refresh_ok = 0;
  nrto::GenState gen;
  int inc_engine = -1;                      // incremental solve in progress (nrto_solve_begin)
  int inc_l = 0;                            // outer iterations run by it
  int dr_loop_grid = 0;                     // persistent DR loop grid (0: not usable)
  int qp_grid = 0;                          // grid-wide QP grid size (0: not usable)
  int sharded = 0;                          // nrto_shard_cones called
};

namespace nrto {

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum for blockDim.x a multiple of 32 (<= 1024); all threads get it.
__device__ __forceinline__ double block_sum(double v, double* sh /*[32]*/) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = (l < nw) ? sh[l] : 0.0;
  r = warp_sum(r);
  return r;
}

// SM Eq.(18): case order a <= t, a <= -t, otherwise (R13).
// Returns t' and writes the scale s with y' = s y.
__device__ __forceinline__ double soc_case(double t, double a, double* s) {
  if (a <= t) { *s = 1.0; return t; }
  if (a <= -t) { *s = 0.0; return 0.0; }
  const double h = 0.5 * (t + a);
  *s = h / a;
  return h;
}

// Correction-list entries: cone index | kRecompute (lazy y: rebuild y^l).
constexpr int kListMask = (1 << 28) - 1;
constexpr int kRecompute = 1 << 30;   // y^l not stored by the pass: rebuild it
constexpr int kLeave = 1 << 29;       // state cone leaves {s = 1}: G -= b b^T, H -= b b_hat^T
constexpr int kEnter = 1 << 28;       // state cone enters {s = 1}: G += b b^T, H += b b_hat^T

// Predicted projection scale shat of the fused pass (fused.cu, tma.cu).
// l = 1 (cold start, t = p^0 + lam_p^0 = 0): a state cone with a > 0 is in
// case 3 with s = (0 + a)/(2a) = 1/2 exactly, so shat = 1/2.  l > 1: shat =
// [s^{l-1} == 1] (case 1 persists).  Mispredictions are corrected exactly.
// Residual trace row l-1 of instance b (QP kernels, after r_p / r_d of iteration l).
__device__ __forceinline__ void record_hist(const Dev& v, int b, int l, double rp, double rd,
                                            int engine) {
  if (v.hist && l >= 1 && l <= v.hist_L) {
    double* h = v.hist + ((int64_t)b * v.hist_L + (l - 1)) * 3;
    h[0] = rp; h[1] = rd; h[2] = engine == NRTO_FULLADMM ? 0.0 : v.rdr[b];
  }
}

// Projection-case statistics (nrto_case_stats_enable): s = 1 <=> case 1 (kept),
// s = 0 <=> case 2 (origin), else case 3 (boundary) -- soc_case never returns
// 0 or 1 in case 3 since |t| < a there.  Warp-aggregated counters per iteration.
__device__ __forceinline__ void count_case(const Dev& v, double s) {
  if (!v.case_cnt || v.iter < 1 || v.iter > v.hist_L) return;
  const unsigned m = __activemask();
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  const int c1 = __popc(__ballot_sync(m, s == 1.0));
  const int c2 = __popc(__ballot_sync(m, s == 0.0));
  const int c3 = __popc(m) - c1 - c2;
  if (lane == leader) {
    unsigned long long* c = v.case_cnt + (int64_t)(v.iter - 1) * 3;
    if (c1) atomicAdd(c + 0, (unsigned long long)c1);
    if (c2) atomicAdd(c + 1, (unsigned long long)c2);
    if (c3) atomicAdd(c + 2, (unsigned long long)c3);
  }
}

__device__ __forceinline__ double shat_of(const Dev& v, double sprev) {
  if (v.iter == 1) return 0.5;
  return (sprev == 1.0) ? 1.0 : 0.0;
}

// Gain chain solve for one (instance, step): K = V [(V^T R U) ./ den] U^T,
// R given in sR (nu x nx).  Uses scratch sX (nu x nx); nt threads cooperate.
template <int NXC = 0, int NUC = 0>
__device__ __forceinline__ void chain_solve(const double* V, const double* U, const double* den,
                                            double* sR, double* sX, int nu_rt, int nx_rt, int tid, int nt) {
  const int nx = NXC > 0 ? NXC : nx_rt, nu = NUC > 0 ? NUC : nu_rt;
  for (int r = tid; r < nu * nx; r += nt) {        // sX = V^T R
    const int a = r / nx, c = r % nx;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < nu; ++q) acc += V[q * nu + a] * sR[q * nx + c];
    sX[r] = acc;
  }
  __syncthreads();
  for (int r = tid; r < nu * nx; r += nt) {        // sR = (sX U) ./ den
    const int a = r / nx, c = r % nx;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < nx; ++q) acc += sX[a * nx + q] * U[q * nx + c];
    sR[r] = acc * den[r];
  }
  __syncthreads();
  for (int r = tid; r < nu * nx; r += nt) {        // sX = V sR
    const int a = r / nx, c = r % nx;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < nu; ++q) acc += V[a * nu + q] * sR[q * nx + c];
    sX[r] = acc;
  }
  __syncthreads();
  for (int r = tid; r < nu * nx; r += nt) {        // sR = sX U^T  (= K)
    const int a = r / nx, c = r % nx;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < nx; ++q) acc += sX[a * nx + q] * U[c * nx + q];
    sR[r] = acc;
  }
  __syncthreads();
}

// Geometry of cone j's ragged row.
struct ConeGeom {
  int kind, knot, L, klo, nbB;
  int64_t off, offB;
};
__device__ __forceinline__ ConeGeom cone_geom(const Dev& v, int j) {
  ConeGeom g;
  g.kind = v.kind[j];
  g.knot = v.knot[j];
  g.off = v.off[j];
  g.offB = v.offB[j];
  g.L = (g.kind == 0) ? (g.knot + 1) * v.d.nx : v.d.nx;
  g.klo = (g.kind == 0) ? 0 : g.knot;
  g.nbB = (g.kind == 0) ? g.knot : 1;
  return g;
}

// Warp-level versions: one warp per (instance, step), 8 per CTA (the 7x14
// chain has 98 outputs, so a CTA per step mostly idles and the tiny CTAs
// crowd the SMs the concurrently running QP needs).
// NXC, NUC > 0: sizes fixed at compile time (bench shapes; loops fully unrolled,
// same summation order as the runtime-size version).
template <int NXC = 0, int NUC = 0>
__device__ __forceinline__ void chain_solve_w(const double* V, const double* U, const double* den,
                                              double* sR, double* sX, int nu_rt, int nx_rt, int lane) {
  const int nx = NXC > 0 ? NXC : nx_rt, nu = NUC > 0 ? NUC : nu_rt;
#pragma unroll
  for (int r = lane; r < nu * nx; r += 32) {
    const int a = r / nx, c = r % nx;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < nu; ++q) acc += V[q * nu + a] * sR[q * nx + c];
    sX[r] = acc;
  }
  __syncwarp();
#pragma unroll
  for (int r = lane; r < nu * nx; r += 32) {
    const int a = r / nx, c = r % nx;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < nx; ++q) acc += sX[a * nx + q] * U[q * nx + c];
    sR[r] = acc * den[r];
  }
  __syncwarp();
#pragma unroll
  for (int r = lane; r < nu * nx; r += 32) {
    const int a = r / nx, c = r % nx;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < nu; ++q) acc += V[a * nu + q] * sR[q * nx + c];
    sX[r] = acc;
  }
  __syncwarp();
#pragma unroll
  for (int r = lane; r < nu * nx; r += 32) {
    const int a = r / nx, c = r % nx;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < nx; ++q) acc += sX[a * nx + q] * U[c * nx + q];
    sR[r] = acc;
  }
  __syncwarp();
}

// Launchers (defined in the .cu files; return cudaGetLastError()).
cudaError_t launch_setup(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_fa_reset(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_dr_reset(nrto_handle_s* h, int full, cudaStream_t st);
cudaError_t launch_dr_arm(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_fa_pass(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_fa_gain(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_dr_gain(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_dr_pass(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_dr_reduce(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_qp(nrto_handle_s* h, int engine, int l, cudaStream_t st);
cudaError_t launch_adjoint(nrto_handle_s* h, const double* y, const double* scale,
                           const int32_t* act, cudaStream_t st);
cudaError_t launch_finish(nrto_handle_s* h, int engine, const nrto_out* o, cudaStream_t st);
cudaError_t launch_gain_update(nrto_handle_s* h, const double* nu, const double* kv_prev,
                               double* kv_next, cudaStream_t st);
cudaError_t launch_soc_project(const double* t, const double* y, const int64_t* off,
                               int64_t n, double* to, double* yo, cudaStream_t st);
cudaError_t launch_count_active(nrto_handle_s* h, int32_t* d_count, int dr, cudaStream_t st);
cudaError_t launch_solve_flags(nrto_handle_s* h, double* flags, cudaStream_t st);
cudaError_t launch_finish_inst(nrto_handle_s* h, double* margin_lin, double* objective, cudaStream_t st);
cudaError_t gen_setup(nrto_handle_s* h, const double* Gamma, const double* Psi, int nz, bool host,
                      cudaStream_t st, int* spd_err);
cudaError_t gen_reset(nrto_handle_s* h, cudaStream_t st);
cudaError_t gen_iteration(nrto_handle_s* h, int l, cudaStream_t st);
cudaError_t gen_finish(nrto_handle_s* h, double* mcone, cudaStream_t st);
void gen_free(nrto_handle_s* h);
int read_setup_error(cudaStream_t st);
cudaError_t launch_engine_factors(nrto_handle_s* h, int engine, cudaStream_t st);
cudaError_t launch_sparse_rows(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_gram_tiles(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_fa_ctrl(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_fa_fused(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_zlist(nrto_handle_s* h, const double* y, const int32_t* clist, const double* cw,
                         const double* scale, const int32_t* ncnt, int nfixed, const int32_t* act,
                         double* Zout, cudaStream_t st, int lazy = 0, int ghmode = 0,
                         double* dG = nullptr, double* dH = nullptr, int prezeroed = 0);
cudaError_t launch_dr_adjoint(nrto_handle_s* h, cudaStream_t st);
bool fused_supported(const Dims& d);
bool tma_supported(const Dims& d);
cudaError_t launch_setup_mma(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_fa_tma(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_project(nrto_handle_s* h, cudaStream_t st);
cudaError_t launch_qp_sparse(nrto_handle_s* h, int engine, int l, cudaStream_t st, int grid = 0);
// persistent DR loop (persist.cu)
void dr_loop_plan(const Dims& d, const int32_t* knot, const int8_t* kind, int nsm,
                  std::vector<int32_t>& chunk, std::vector<int32_t>& kr, int& Ec, int& EBc);
int dr_loop_grid(const Dev& v);
bool dr_loop_supported(const nrto_handle_s* h);
cudaError_t launch_dr_loop(nrto_handle_s* h, int ndr, cudaStream_t st);
// chunked-scan QP (qp.cu): used for batches up to kScanMaxBatch instances
constexpr int kScanMaxBatch = 64;
void scan_plan(int T, int& M, int& C);
cudaError_t launch_scan_factors(nrto_handle_s* h, int engine, cudaStream_t st);
// whole FullADMM loop of a small instance per CTA (qp.cu)
bool fa_small_ok(const nrto_handle_s* h);
bool qp_grid_plan(const Dims& d, int nsm, int& M, int& C);
int qp_grid_size(const nrto_handle_s* h);
cudaError_t launch_fa_small(nrto_handle_s* h, int L, cudaStream_t st);

}  // namespace nrto
