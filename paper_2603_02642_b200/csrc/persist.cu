// Persistent DR loop for small batches.
//
// One cooperative launch runs all DR iterations (11a-c) of one
// NRTO-ADMM iteration for the batch; the per-iteration kernels of the
// launch-per-phase path (k_dr_gain, k_dr_pass_*, the list adjoint, k_dr_reduce:
// four launches, ~26 us per DR iteration for one c2 instance) become two phases
// separated by grid barriers:
//   G  per (instance, step k): Z_k = sum_j b_{j,k} eta~_{j,k}^T from the chunk
//      partials of the previous pass (fixed chunk order), the affine prox (11a)
//      in Schur form (F3): R = sigma K~ + r_s sqrt(tau) (Z_k - Zb_k) Psi_k,
//      K = chain solve, K~ += alpha (K - K~), C_k = sqrt(tau) Psi_k K^T.
//   P  per (instance, cone chunk): the cone step of k_dr_pass (P:343-359,
//      P:966-1002) for every cone of the chunk with C of the chunk's steps and
//      the cones' b rows staged in shared memory, then the chunk's adjoint
//      partial Z_k^(q) = sum_{j in q} b_{j,k} eta~_{j,k}^T from the new eta~
//      still in shared memory, and the chunk's sum of ||s~^l - s~^{l-1}||^2.
// Every CTA derives r_dr and the DR stop test itself from the chunk
// sums (same order in every CTA), so the loop exits in step without a host poll.
// All cross-CTA data is read through L2 (ld.global.cg): L1 is not coherent.
#include "common.cuh"
#include <algorithm>
#include <cstdlib>
#include <vector>

namespace nrto {

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long x;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
  return x;
}

// 8-byte cp.async into shared memory (immutable data, or data only this CTA writes:
// the copy may be served from L1)
__device__ __forceinline__ void dr_cpa8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src) : "memory");
}
__device__ __forceinline__ void dr_cpa_wait() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
}

// Grid barrier of a cooperative launch: the counter is zeroed by k_dr_arm before
// the launch; the n-th barrier waits for n * gridDim.x arrivals.
__device__ __forceinline__ void grid_barrier(unsigned long long* ctr, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    while (ld_acquire_u64(ctr) < target) {
    }
  }
  __syncthreads();
}

// Persistent shared-memory layout of k_dr_loop (doubles), host and device agree.
// Each CTA owns at most one cone chunk (item) and up to `tpc` (instance, step) tasks
// for the whole launch; their state lives in shared memory between iterations.
struct DrLayout {
  int NA, NN, NG, ngrp, tpc, ncmax, Ec, EBc, Q;
  int64_t task, tasks;        // per-task block, all tasks
  int64_t scr;                // phase-G scratch
  int64_t rec;                // cone records of the item
  int64_t item;               // item arrays
  int64_t kr;                 // chunk step ranges (ints, as doubles)
  int64_t total;
};
__host__ __device__ inline DrLayout dr_layout(const Dims& d, int Q, int Ec, int EBc, int ncmax, int tpc,
                                              int nthreads) {
  DrLayout L;
  L.NA = d.nu * d.nx; L.NN = d.nx * d.nx; L.NG = d.nu * d.nu;
  L.ngrp = nthreads / L.NA > 0 ? nthreads / L.NA : 1;
  if (L.ngrp > 8) L.ngrp = 8;      // the partial-sum groups are combined sequentially
  L.tpc = tpc; L.ncmax = ncmax; L.Ec = Ec; L.EBc = EBc; L.Q = Q;
  L.task = 5 * L.NA + 2 * L.NN + L.NG + 2;         // Kt, K, den, Zb, (spare), P, U, V, st, valid
  L.tasks = L.task * tpc;
  L.scr = (int64_t)L.NA * (3 + L.ngrp);            // Z, R, X, group partials
  L.rec = 10 * (int64_t)ncmax;
  // b_hat, eta~, a, squares, b rows, C slice, element map (cone int32 + offsets int2)
  L.item = 4 * (int64_t)Ec + EBc + (int64_t)d.T * L.NA + 2 * (int64_t)Ec +
           ((int64_t)d.T + 2) / 2 + 1 + EBc;                      // + step lists (offsets, int2 entries)
  L.kr = (2 * (int64_t)Q + 1) / 2 + 1;
  L.total = L.tasks + L.scr + L.rec + L.item + L.kr;
  return L;
}

constexpr int kDrThreads = 512;

// Debug phase clocks of CTA 0 (globaltimer, ns) for iterations 2..5: read with
// nrto_debug_dr_clocks (not part of nrto.h).
__device__ unsigned long long g_dr_clk[64];
__device__ unsigned long long g_dr_pclk[2 * 1024];   // per CTA: P-phase ns, G-phase ns (iteration 3)
__device__ unsigned long long g_dr_sub[1024 * 8];    // per CTA: P sub-phase timestamps (iteration 3)
#define DR_SUB(ph) \
  do { if (m == 3 && tid == 0 && blockIdx.x < 1024) g_dr_sub[blockIdx.x * 8 + (ph)] = gtimer(); } while (0)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define DR_CLK(ph) \
  do { if (blockIdx.x == 0 && tid == 0 && m >= 2 && m <= 5) g_dr_clk[(m - 2) * 8 + (ph)] = gtimer(); } while (0)

template <int NUM>
__global__ void __launch_bounds__(kDrThreads, 1) k_dr_loop(Dev v, int ndr, int ncmax, int tpc) {
  extern __shared__ double sm[];
  __shared__ int sact[32];      // DR-active per instance (same in every CTA)
  __shared__ int sran[32];      // instance ran the previous pass
  const Dims d = v.d;
  const int nx = d.nx, nu = NUM > 0 ? NUM : d.nu, T = d.T, Q = v.drQ, B = d.B;
  const int tid = threadIdx.x, nt = blockDim.x, G = gridDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const DrLayout Ly = dr_layout(d, Q, v.drEc, v.drEBc, ncmax, tpc, nt);
  const int NA = Ly.NA, NN = Ly.NN, NG = Ly.NG;
  const double sg = v.prm.sigma_dr, rs = v.prm.r_s, al = v.prm.alpha_dr, rho = v.prm.rho_admm;
  double* sTask = sm;
  double* sZ = sm + Ly.tasks;
  double* sR = sZ + NA;
  double* sX = sR + NA;
  double* sZg = sX + NA;
  int64_t* cof = reinterpret_cast<int64_t*>(sm + Ly.tasks + Ly.scr);  // [ncmax] eta~ offsets
  int64_t* cofB = cof + ncmax;                                        // [ncmax] b-row offsets
  int* cinf = reinterpret_cast<int*>(cofB + ncmax);                   // [ncmax][4]
  double* sd2 = reinterpret_cast<double*>(cinf + 4 * ncmax);          // [ncmax]
  double* spit = sd2 + ncmax;                                         // [ncmax] pi~
  double* stt = spit + ncmax;                                         // [ncmax] t~
  double* spl = stt + ncmax;                                          // [ncmax] rho p + lambda
  double* spi = spl + ncmax;                                          // [ncmax] pi of the last prox
  double* sn2c = spi + ncmax;                                         // [ncmax] projection scale
  double* sBh = sm + Ly.tasks + Ly.scr + Ly.rec;                      // [Ec]
  double* sY = sBh + Ly.Ec;                                           // [Ec] eta~ (resident)
  double* sA = sY + Ly.Ec;                                            // [Ec]
  double* sQ = sA + Ly.Ec;                                            // [Ec] squares
  double* sB = sQ + Ly.Ec;                                            // [EBc]
  double* sC = sB + Ly.EBc;                                           // [T][nx][nu]
  int* eki = reinterpret_cast<int*>(sC + (int64_t)T * NA);            // [Ec] cone index
  int2* eof = reinterpret_cast<int2*>(eki + 2 * ((Ly.Ec + 1) / 2));   // [Ec] C / b-row offsets
  int* kp = reinterpret_cast<int*>(eof + Ly.Ec);                      // [khi - klo + 1] list offsets
  int2* kl = reinterpret_cast<int2*>(kp + 2 * ((T + 2) / 2 + 1));     // (b row, eta~ block) offsets of
                                                                      // the cones with a block at k
  int* skr = reinterpret_cast<int*>(kl + Ly.EBc);                     // [Q][2]
  // ---- my item (cone chunk) and tasks
  const int item = blockIdx.x < B * Q ? blockIdx.x : -1;
  const int ib = item >= 0 ? item / Q : 0, iq = item >= 0 ? item % Q : 0;
  const int j0 = item >= 0 ? __ldg(v.drchunk + iq) : 0;
  const int nc = item >= 0 ? __ldg(v.drchunk + iq + 1) - j0 : 0;
  const int klo = item >= 0 ? __ldg(v.drkr + 2 * iq) : 0, khi = item >= 0 ? __ldg(v.drkr + 2 * iq + 1) : 0;
  const int64_t off0 = item >= 0 ? __ldg(v.off + j0) : 0, offB0 = item >= 0 ? __ldg(v.offB + j0) : 0;
  const int64_t nE = item >= 0 ? __ldg(v.off + j0 + nc) - off0 : 0;
  const int64_t nB = item >= 0 ? __ldg(v.offB + j0 + nc) - offB0 : 0;
  // ---- load everything this CTA keeps for the launch (one memory round)
  if (tid < B) { sact[tid] = v.active[tid] && v.dr_active[tid]; sran[tid] = 0; }
  for (int r = tid; r < 2 * Q; r += nt) skr[r] = __ldg(v.drkr + r);
  for (int t = 0; t < tpc; ++t) {
    const int task = blockIdx.x + t * G;
    double* tk = sTask + t * Ly.task;
    if (task >= B * T) { if (tid == 0) tk[Ly.task - 1] = 0.0; continue; }
    const int b = task / T, k = task % T;
    const int64_t bk = (int64_t)b * T + k;
    const int kr = __ldg(v.Urep + bk);
    double* Kt = tk; double* Kk = Kt + NA; double* den = Kk + NA; double* Zb = den + NA;
    double* P = Zb + 2 * NA; double* U = P + NN; double* V = U + NN;
    const double* Ktg = v.Kt + (int64_t)b * d.NK + (int64_t)k * NA;
    const double* Kg = v.K + (int64_t)b * d.NK + (int64_t)k * NA;
    for (int r = tid; r < NA; r += nt) {
      dr_cpa8(Kt + r, Ktg + r); dr_cpa8(Kk + r, Kg + r);
      dr_cpa8(den + r, v.dr.den + bk * NA + r); dr_cpa8(Zb + r, v.Zb + bk * NA + r);
    }
    const double* Pk = v.Psi + ((int64_t)b * (T + 1) + kr) * NN;
    const double* Uk = v.U + ((int64_t)b * T + kr) * NN;
    for (int r = tid; r < NN; r += nt) { dr_cpa8(P + r, Pk + r); dr_cpa8(U + r, Uk + r); }
    for (int r = tid; r < NG; r += nt) dr_cpa8(V + r, v.dr.V + bk * NG + r);
    if (tid == 0) { V[NG] = sqrt(__ldg(v.tau + b)); V[NG + 1] = 1.0; }
  }
  if (item >= 0) {
    const int64_t eo = (int64_t)ib * d.E + off0;
    for (int64_t r = tid; r < nE; r += nt) { dr_cpa8(sBh + r, v.bhat + eo + r); dr_cpa8(sY + r, v.Y + eo + r); }
    const double* Bdg = v.Bd + (int64_t)ib * d.EB + offB0;
    for (int64_t r = tid; r < nB; r += nt) dr_cpa8(sB + r, Bdg + r);
    for (int c = tid; c < nc; c += nt) {
      const int j = j0 + c, kd = __ldg(v.kind + j), kn = __ldg(v.knot + j);
      cof[c] = __ldg(v.off + j) - off0;
      cofB[c] = __ldg(v.offB + j) - offB0;
      cinf[4 * c + 0] = kd; cinf[4 * c + 1] = kn;
      cinf[4 * c + 2] = kd == 0 ? 0 : kn; cinf[4 * c + 3] = kd == 0 ? kn : 1;
      const int64_t ij = (int64_t)ib * d.ng + j;
      spit[c] = __ldg(v.pit + ij); stt[c] = __ldg(v.tt + ij);
      spl[c] = rho * __ldg(v.p + ij) + __ldg(v.lamp + ij);   // p, lambda: fixed during the DR loop
      spi[c] = __ldg(v.pt + ij);
      sd2[c] = __ldg(v.rdr_part + ij);
    }
  }
  dr_cpa_wait();
  __syncthreads();
  // element map of the chunk: cone, block, component of every eta~ element
  for (int c = warp; c < nc; c += nw) {
    const int L = cinf[4 * c] == 0 ? (cinf[4 * c + 1] + 1) * nx : nx;
    const int o = (int)cof[c];
    const int cklo = cinf[4 * c + 2], nbB = cinf[4 * c + 3], kd = cinf[4 * c];
    for (int e = lane; e < L; e += 32) {
      const int kb = e / nx, i = e - kb * nx;
      eki[o + e] = c;
      // .x: offset of C_k row i in the C slice (-1: no b-block), bit 30: state cone (b_hat)
      // .y: offset of b_{j,k} in the chunk's b rows
      const int ci = kb < nbB ? ((cklo + kb - klo) * nx + i) * nu : -1;
      eof[o + e] = make_int2((kd == 0 ? (1 << 30) : 0) | (ci < 0 ? (1 << 30) - 1 : ci),
                             (int)cofB[c] + kb * d.nup);
    }
  }
  // step -> cone lists of the chunk (cone order), for the adjoint partial
  for (int k = klo + tid; k < khi; k += nt) {
    int n = 0;
    for (int c = 0; c < nc; ++c) n += (k >= cinf[4 * c + 2] && k < cinf[4 * c + 2] + cinf[4 * c + 3]);
    kp[k - klo + 1] = n;
  }
  __syncthreads();
  if (tid == 0) {
    kp[0] = 0;
    for (int k = 1; k <= khi - klo; ++k) kp[k] += kp[k - 1];
  }
  __syncthreads();
  for (int k = klo + tid; k < khi; k += nt) {
    int n = kp[k - klo];
    for (int c = 0; c < nc; ++c)
      if (k >= cinf[4 * c + 2] && k < cinf[4 * c + 2] + cinf[4 * c + 3]) {
        const int kb = k - cinf[4 * c + 2];
        kl[n++] = make_int2((int)cofB[c] + kb * d.nup, (int)cof[c] + kb * nx);
      }
  }
  __syncthreads();
  unsigned long long nbar = 0;
  for (int m = 1;; ++m) {
    DR_CLK(0);
    // ---- head: r_dr of pass m-1 and the stop test, identically in every CTA; the
    //      chunk partials of this CTA's first step are loaded in the same memory round
    const int ngrp = Ly.ngrp;
    bool pre0 = false;
    if (m > 1) {
      if (tid < B) sran[tid] = sact[tid];
      __syncthreads();
      if (blockIdx.x < B * T && sran[blockIdx.x / T]) {
        const int k = blockIdx.x % T;
        const int g = tid / NA, o = tid - g * NA;
        if (g < ngrp) {
          double acc = 0.0;
          const double* zp = v.drZpart + (int64_t)blockIdx.x * Q * NA + o;   // [B][T][Q][NA]
#pragma unroll 8
          for (int q = g; q < Q; q += ngrp) {
            const double z = (k >= skr[2 * q] && k < skr[2 * q + 1]) ? __ldcg(zp + (int64_t)q * NA) : 0.0;
            acc += z;
          }
          sZg[g * NA + o] = acc;
        }
        pre0 = true;
      }
      // fixed iteration counts: no stop test, r_dr is only reported (after the last pass)
      const bool need_rdr = !v.prm.fixed_iters || m > ndr;
      for (int b = warp; b < B && need_rdr; b += nw) {
        if (!sran[b]) continue;
        double a = 0.0;
#pragma unroll 4
        for (int q = lane; q < Q; q += 32) a += __ldcg(v.drrq + (int64_t)b * Q + q);   // loads in flight together
        a = warp_sum(a);
        if (lane == 0) {
          const double r = sqrt(a);
          if (blockIdx.x == 0) v.rdr[b] = r;
          if (!v.prm.fixed_iters && r <= v.prm.eps_dr) {
            sact[b] = 0;
            if (blockIdx.x == 0) v.dr_active[b] = 0;
          }
        }
      }
      __syncthreads();
    }
    DR_CLK(5);
    const unsigned long long tG0 = (m == 3 && tid == 0) ? gtimer() : 0ULL;
    int any = 0;
    for (int b = 0; b < B; ++b) any |= sact[b];
    const bool run = any && m <= ndr;
    // ---- phase G: adjoint of eta~^{m-1} per step (stored to Z for the warm start of
    //      the next call) and, while running, the affine prox (11a)
    for (int t = 0; t < tpc; ++t) {
      const int task = blockIdx.x + t * G;
      if (task >= B * T) break;
      const int b = task / T, k = task % T;
      const bool need_z = m > 1 && sran[b];
      const bool gain = run && sact[b];
      if (!need_z && !gain) continue;
      const int64_t bk = (int64_t)b * T + k;
      double* tk = sTask + t * Ly.task;
      double* Kt = tk; double* Kk = Kt + NA; double* den = Kk + NA; double* Zb = den + NA;
      double* P = Zb + 2 * NA; double* U = P + NN; double* V = U + NN;
      const double st = V[NG];
      if (m == 1) {
        for (int r = tid; r < NA; r += nt) sZ[r] = __ldcg(v.Z + bk * NA + r);
      } else {
        if (!(t == 0 && pre0)) {
          const int g = tid / NA, o = tid - g * NA;
          if (g < ngrp) {
            double acc = 0.0;
            const double* zp = v.drZpart + bk * Q * NA + o;     // [B][T][Q][NA]
#pragma unroll 8
            for (int q = g; q < Q; q += ngrp) {
              const double z = (k >= skr[2 * q] && k < skr[2 * q + 1]) ? __ldcg(zp + (int64_t)q * NA) : 0.0;
              acc += z;
            }
            sZg[g * NA + o] = acc;
          }
        }
        __syncthreads();
        for (int r = tid; r < NA; r += nt) {
          double z = 0.0;
          for (int g2 = 0; g2 < ngrp; ++g2) z += sZg[g2 * NA + r];
          sZ[r] = z;
          v.Z[bk * NA + r] = z;
        }
      }
      __syncthreads();
      if (!gain) continue;
      for (int r = tid; r < NA; r += nt) sX[r] = sZ[r] - Zb[r];
      __syncthreads();
      for (int r = tid; r < NA; r += nt) {
        const int mm = r / nx, i = r % nx;
        double gp = 0.0;
        for (int q = 0; q < nx; ++q) gp += sX[mm * nx + q] * P[q * nx + i];
        sR[r] = sg * Kt[i * nu + mm] + rs * st * gp;
      }
      __syncthreads();
      chain_solve<0, NUM>(V, U, den, sR, sX, nu, nx, tid, nt);
      for (int r = tid; r < NA; r += nt) {
        const int mm = r / nx, i = r % nx;
        Kk[i * nu + mm] = sR[r];
        Kt[i * nu + mm] += al * (sR[r] - Kt[i * nu + mm]);
      }
      for (int r = tid; r < NA; r += nt) {
        const int i = r / nu, mm = r % nu;
        double acc = 0.0;
        for (int q = 0; q < nx; ++q) acc += P[i * nx + q] * sR[mm * nx + q];
        v.Ccur[bk * NA + r] = st * acc;
      }
      __syncthreads();
    }
    if (!run) break;
    DR_CLK(1);
    if (m == 3 && tid == 0 && blockIdx.x < 1024) g_dr_pclk[2 * blockIdx.x + 1] = gtimer() - tG0;
    grid_barrier(v.drbar, (++nbar) * (unsigned long long)G);
    DR_CLK(2);
    const unsigned long long tP0 = (m == 3 && tid == 0) ? gtimer() : 0ULL;
    // ---- phase P: cone steps of my chunk, the chunk adjoint partial
    if (item >= 0 && sact[ib]) {
      {
        const double* Cg = v.Ccur + ((int64_t)ib * T + klo) * NA;
        const int nC = (khi - klo) * NA;
#pragma unroll 8
        for (int r = tid; r < nC; r += nt) sC[r] = __ldcg(Cg + r);
      }
      DR_SUB(0);
      __syncthreads();
      DR_SUB(1);
      // forward map a = C b + b_hat and (2a - eta~)^2, flat over the chunk's elements
#pragma unroll 4
      for (int e = tid; e < nE; e += nt) {
        const int2 f = eof[e];
        double a = (f.x & (1 << 30)) ? sBh[e] : 0.0;        // b_hat (state cones)
        const int ci = f.x & ((1 << 30) - 1);
        if (ci != (1 << 30) - 1) {                           // C_k b_{j,k} (blocks with b)
          const double* Cr = sC + ci;
          const double* br = sB + f.y;
          if constexpr (NUM > 0) {
#pragma unroll
            for (int mm = 0; mm < NUM; ++mm) a += Cr[mm] * br[mm];
          } else {
            for (int mm = 0; mm < nu; ++mm) a += Cr[mm] * br[mm];
          }
        }
        sA[e] = a;
        const double er = 2.0 * a - sY[e];
        sQ[e] = er * er;
      }
      __syncthreads();
      DR_SUB(2);
      // per cone: norm, projection of s_ref = 2 s - s~, the t-part updates
      // (short cones: a thread each; long cones: a warp each)
      auto cone_proj = [&](int c, double n2) {
        const double pit = spit[c], tt = stt[c];
        const double pi = (sg * pit + spl[c] + rs * tt) / (rho + sg + rs);
        double sc;
        const double tpi = soc_case(2.0 * pi - tt, sqrt(n2), &sc);
        const double ttn = tt + al * (tpi - pi);
        stt[c] = ttn;
        spit[c] = pit + al * (pi - pit);
        spi[c] = pi;
        sd2[c] = (ttn - tt) * (ttn - tt);
        sn2c[c] = sc;
      };
      for (int c = tid; c < nc; c += nt) {
        const int L = cinf[4 * c] == 0 ? (cinf[4 * c + 1] + 1) * nx : nx;
        if (L > 64) continue;
        const double* q2 = sQ + cof[c];
        double n2 = 0.0;
        for (int e = 0; e < L; ++e) n2 += q2[e];
        cone_proj(c, n2);
      }
      for (int c = warp; c < nc; c += nw) {
        const int L = cinf[4 * c] == 0 ? (cinf[4 * c + 1] + 1) * nx : nx;
        if (L <= 64) continue;
        const double* q2 = sQ + cof[c];
        double n2 = 0.0;
        for (int e = lane; e < L; e += 32) n2 += q2[e];
        n2 = warp_sum(n2);
        if (lane == 0) cone_proj(c, n2);
      }
      __syncthreads();
      DR_SUB(3);
      // eta~ += alpha (Pi(s_ref) - s), flat; squared change per element
#pragma unroll 4
      for (int e = tid; e < nE; e += nt) {
        const int c = eki[e];
        const double a = sA[e], et = sY[e];
        const double er = 2.0 * a - et;
        const double en = et + al * (sn2c[c] * er - a);
        sY[e] = en;
        sQ[e] = (en - et) * (en - et);
      }
      __syncthreads();
      DR_SUB(4);
      for (int c = tid; c < nc; c += nt) {
        const int L = cinf[4 * c] == 0 ? (cinf[4 * c + 1] + 1) * nx : nx;
        if (L > 64) continue;
        const double* q2 = sQ + cof[c];
        double d2 = 0.0;
        for (int e = 0; e < L; ++e) d2 += q2[e];
        sd2[c] += d2;
      }
      for (int c = warp; c < nc; c += nw) {
        const int L = cinf[4 * c] == 0 ? (cinf[4 * c + 1] + 1) * nx : nx;
        if (L <= 64) continue;
        const double* q2 = sQ + cof[c];
        double d2 = 0.0;
        for (int e = lane; e < L; e += 32) d2 += q2[e];
        d2 = warp_sum(d2);
        if (lane == 0) sd2[c] += d2;
      }
      // chunk partial Z_k^(q) = sum_{j in q} b_{j,k} eta~_{j,k}^T (cone order)
      double* Zq = v.drZpart + (int64_t)iq * NA;
      for (int r = tid; r < (khi - klo) * NA; r += nt) {
        const int k = klo + r / NA, o = r % NA, mm = o / nx, i = o % nx;
        double acc = 0.0;
        for (int q = kp[k - klo]; q < kp[k - klo + 1]; ++q) {
          const int2 o = kl[q];
          acc += sB[o.x + mm] * sY[o.y + i];
        }
        Zq[((int64_t)ib * T + k) * Q * NA + o] = acc;
      }
      __syncthreads();                               // sd2 of every cone written
      if (warp == 0) {                               // chunk sum (fixed order: lane strides, tree)
        double a = 0.0;
        for (int c = lane; c < nc; c += 32) a += sd2[c];
        a = warp_sum(a);
        if (lane == 0) v.drrq[(int64_t)ib * Q + iq] = a;
      }
      DR_SUB(5);
    }
    DR_CLK(3);
    if (m == 3 && tid == 0 && blockIdx.x < 1024) g_dr_pclk[2 * blockIdx.x] = gtimer() - tP0;
    grid_barrier(v.drbar, (++nbar) * (unsigned long long)G);
    DR_CLK(4);
  }
  // ---- write back the state kept in shared memory
  for (int t = 0; t < tpc; ++t) {
    const int task = blockIdx.x + t * G;
    if (task >= B * T) break;
    const int b = task / T, k = task % T;
    const double* tk = sTask + t * Ly.task;
    double* Ktg = v.Kt + (int64_t)b * d.NK + (int64_t)k * NA;
    double* Kg = v.K + (int64_t)b * d.NK + (int64_t)k * NA;
    for (int r = tid; r < NA; r += nt) { Ktg[r] = tk[r]; Kg[r] = tk[NA + r]; }
  }
  if (item >= 0) {
    double* Yg = v.Y + (int64_t)ib * d.E + off0;
    for (int64_t r = tid; r < nE; r += nt) Yg[r] = sY[r];
    for (int c = tid; c < nc; c += nt) {
      const int64_t ij = (int64_t)ib * d.ng + j0 + c;
      v.pit[ij] = spit[c]; v.tt[ij] = stt[c]; v.pt[ij] = spi[c]; v.rdr_part[ij] = sd2[c];
    }
  }
}

bool dr_loop_supported(const nrto_handle_s* h) {
  const Dev& v = h->dev;
  static const int env = [] { const char* e = getenv("NRTO_DR_PERSIST"); return e ? atoi(e) : 1; }();
  return env && v.drQ > 0 && v.d.B <= 32 && v.d.nu <= 8 && v.d.nx <= 32 && h->dr_loop_grid > 0;
}

// Host side of the chunking (nrto_setup): cones in index order, closed when the
// chunk's work (eta~ + b row elements + a per-cone constant) reaches the target
// or it holds kDrChunkCones cones.
constexpr int kDrChunkCones = 64;

void dr_loop_plan(const Dims& d, const int32_t* knot, const int8_t* kind, int nsm,
                  std::vector<int32_t>& chunk, std::vector<int32_t>& kr, int& Ec, int& EBc) {
  chunk.clear(); kr.clear(); Ec = 0; EBc = 0;
  if (d.ng == 0 || d.B > 32) return;
  static const int env_q = [] { const char* e = getenv("NRTO_DR_CHUNKS"); return e ? atoi(e) : 0; }();
  auto work = [&](int j) -> int64_t {
    const int64_t L = kind[j] == 0 ? (int64_t)(knot[j] + 1) * d.nx : d.nx;
    const int64_t nb = kind[j] == 0 ? knot[j] : 1;
    return L + nb * d.nup + 32;
  };
  int64_t tot = 0;
  for (int j = 0; j < d.ng; ++j) tot += work(j);
  // #SMs / 2B chunks, but >= ~1024 work units each: a tiny instance in few chunks
  // means few CTAs at the grid barriers (c1: 44 -> 4 chunks, 12.3 -> 10.6 us per DR
  // iteration; c2 keeps 74)
  const int target_q = env_q > 0 ? env_q
                                 : (int)std::max<int64_t>(1, std::min<int64_t>(nsm / (2 * d.B), (tot + 1023) / 1024));
  const int64_t goal = std::max<int64_t>(1, (tot + target_q - 1) / target_q);
  int j = 0;
  while (j < d.ng) {
    const int j0 = j;
    int64_t w = 0, e = 0, eb = 0;
    int klo = d.T, khi = 0;
    while (j < d.ng && (j == j0 || (w + work(j) <= goal && j - j0 < kDrChunkCones))) {
      w += work(j);
      const int L = kind[j] == 0 ? (knot[j] + 1) * d.nx : d.nx;
      const int cl = kind[j] == 0 ? 0 : knot[j], nb = kind[j] == 0 ? knot[j] : 1;
      e += L; eb += (int64_t)nb * d.nup;
      if (nb > 0) { klo = std::min(klo, cl); khi = std::max(khi, cl + nb); }
      ++j;
    }
    if (klo >= khi) { klo = 0; khi = 0; }
    chunk.push_back(j0);
    kr.push_back(klo); kr.push_back(khi);
    Ec = (int)std::max<int64_t>(Ec, e);
    EBc = (int)std::max<int64_t>(EBc, eb);
  }
  chunk.push_back(d.ng);
}

// Tasks per CTA for a grid of G CTAs.
static int dr_tpc(const Dev& v, int G) { return (v.d.B * v.d.T + G - 1) / G; }

size_t dr_loop_smem(const Dev& v, int G) {
  const DrLayout L = dr_layout(v.d, v.drQ, v.drEc, v.drEBc, kDrChunkCones, dr_tpc(v, G), kDrThreads);
  return (size_t)L.total * sizeof(double);
}

// Grid of the cooperative launch: one CTA per SM, every chunk of every instance
// owned by its own CTA (0: not usable -> launch-per-phase path).
int dr_loop_grid(const Dev& v) {
  if (v.drQ <= 0 || v.d.B * v.drQ > v.nsm) return 0;
  int G = std::max(v.d.B * v.drQ, std::min(v.nsm, v.d.B * v.d.T));
  if (dr_tpc(v, G) > 8) return 0;
  const size_t smem = dr_loop_smem(v, G);
  if (smem > 220 * 1024) return 0;
  for (void* kern : {(void*)k_dr_loop<4>, (void*)k_dr_loop<0>}) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
  }
  int occ = 0;
  auto kern = v.d.nu == 4 ? (void*)k_dr_loop<4> : (void*)k_dr_loop<0>;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kDrThreads, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    return 0;
  }
  return G <= occ * v.nsm ? G : 0;
}

cudaError_t launch_dr_loop(nrto_handle_s* h, int ndr, cudaStream_t st) {
  const Dev& v = h->dev;
  const int G = h->dr_loop_grid;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kDrThreads);
  cfg.dynamicSmemBytes = dr_loop_smem(v, G);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int tpc = dr_tpc(v, G);
  cudaError_t e;
  if (v.d.nu == 4)
    e = cudaLaunchKernelEx(&cfg, k_dr_loop<4>, v, ndr, kDrChunkCones, tpc);
  else
    e = cudaLaunchKernelEx(&cfg, k_dr_loop<0>, v, ndr, kDrChunkCones, tpc);
  h->launches++;
  return e;
}

}  // namespace nrto

extern "C" int nrto_debug_dr_clocks(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, nrto::g_dr_clk, sizeof(unsigned long long) * 64);
}
extern "C" int nrto_debug_dr_pclocks(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, nrto::g_dr_pclk, sizeof(unsigned long long) * 2048);
}
extern "C" int nrto_debug_dr_sub(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, nrto::g_dr_sub, sizeof(unsigned long long) * 8192);
}
