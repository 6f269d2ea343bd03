// Per-iteration kernels of the inner loop and the
// output/finish kernels.
#include "common.cuh"
#include <cstdlib>

namespace nrto {

// ---------------------------------------------------------------------------
// FullADMM fused pass: Block-1 (13) of iteration l, with the dual update (16)
// of iteration l-1 folded in.  The stored per-cone row is the projection
// input y^l = A_hat k_v^{l-1} + b_hat + lam_nu^{l-1}; with nu^{l-1} =
// s^{l-1} y^{l-1} and (16), y^l = (2 C^{l-1} - C^{l-2}) b + b_hat +
// (1 - s^{l-1}) y^{l-1}, where C_k = sqrt(tau) Psi_k K_k^T.
// One warp per cone; norm by shuffle; closed-form projection.
__global__ void k_fa_pass(Dev v) {
  const Dims d = v.d;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gw >= (int64_t)d.B * d.ng) return;
  const int b = (int)(gw / d.ng), j = (int)(gw % d.ng);
  if (!v.active[b]) return;
  const int lane = threadIdx.x & 31;
  const int nx = d.nx, nu = d.nu;
  const ConeGeom g = cone_geom(v, j);
  const int64_t ij = (int64_t)b * d.ng + j;
  const double omsp = 1.0 - v.s[ij];
  double* Y = v.Y + (int64_t)b * d.E + g.off;
  const double* bh = v.bhat + (int64_t)b * d.E + g.off;
  const double* Bd = v.Bd + (int64_t)b * d.EB + g.offB;
  const double* Dm = v.D + (int64_t)b * d.T * nx * nu;
  double n2 = 0.0;
  for (int e = lane; e < g.L; e += 32) {
    const int kb = e / nx, i = e - kb * nx;
    double acc = (g.kind == 0) ? bh[e] : 0.0;
    if (kb < g.nbB) {
      const double* Dr = Dm + ((int64_t)(g.klo + kb) * nx + i) * nu;
      const double* br = Bd + kb * d.nup;
      for (int m = 0; m < nu; ++m) acc += Dr[m] * br[m];
    }
    const double y = acc + omsp * Y[e];
    Y[e] = y;
    n2 += y * y;
  }
  n2 = warp_sum(n2);
  if (lane == 0) {
    double s;
    const double tp = soc_case(v.tin[ij], sqrt(n2), &s);
    v.s[ij] = s;
    v.pt[ij] = tp;
    count_case(v, s);
  }
}

// Adjoint reduction S7: Z_k[m][i] = sum_j scale_j b_{j,k}[m] y_{j,k}[i] over the
// cones with a b-block at step k (fixed order).  With scale = s this is
// sum_j b nu^T (FullADMM); with scale = NULL it is sum_j b eta~^T (DR).
__global__ void k_adjoint(Dev v, const double* __restrict__ y, const double* __restrict__ scale,
                          const int32_t* __restrict__ act) {
  const Dims d = v.d;
  const int b = blockIdx.x / d.T, k = blockIdx.x % d.T;
  if (act && !act[b]) return;
  const int nx = d.nx, nu = d.nu;
  const double* yb = y + (int64_t)b * d.E;
  const double* Bd = v.Bd + (int64_t)b * d.EB;
  for (int o = threadIdx.x; o < nu * nx; o += blockDim.x) {
    const int m = o / nx, i = o % nx;
    double acc = 0.0;
    for (int c = v.kptr[k]; c < v.kptr[k + 1]; ++c) {
      const int j = v.kcone[c];
      const int kb = (v.kind[j] == 0) ? k : 0;
      double t = Bd[v.offB[j] + kb * d.nup + m] * yb[v.off[j] + kb * nx + i];
      if (scale) t *= scale[(int64_t)b * d.ng + j];
      acc += t;
    }
    v.Z[((int64_t)b * d.T + k) * nu * nx + o] = acc;
  }
}

// FullADMM (14b) per (instance, step k):
//   R = 2 W K^{l-1} + rho sqrt(tau) (Z - Zb) Psi_k   (= block k of
//   Q_v k^{l-1} + rho sum_j A_hat_j^T (nu_j - b_hat_j))
//   K^l = M_k R (chain), C^l = sqrt(tau) Psi_k K^lT, D = 2 C^l - C^{l-1}.
// mode 0: in-loop (updates K, C, D).  mode 1: nrto_gain_update (kin -> kout).
__global__ void k_fa_gain(Dev v, int mode, const double* kin, double* kout) {
  extern __shared__ double sm[];
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu;
  const int b = blockIdx.x / d.T, k = blockIdx.x % d.T;
  if (mode == 0 && !v.active[b]) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t bk = (int64_t)b * d.T + k;
  double* sR = sm;
  double* sX = sR + nu * nx;
  double* sK = sX + nu * nx;
  const double st = sqrt(v.tau[b]);
  const double* Pk = v.Psi + ((int64_t)b * (d.T + 1) + k) * nx * nx;
  const double* Wk = v.W + bk * nu * nu;
  const double* Kp = (mode == 0 ? v.K : kin) + (int64_t)b * d.NK + (int64_t)k * nu * nx;
  const bool fz = (mode == 0) && v.fused;
  for (int r = tid; r < nu * nx; r += nt) {   // G = Z - Zb into sX ; K_prev into sK
    double z;
    if (fz) {                                  // fused pass partials + correction (+ control)
      z = v.Zc[bk * nu * nx + r];
      if (v.fused == 2) z += v.Zctrl[bk * nu * nx + r];
      const double* zp = v.Zpart + ((int64_t)b * v.nsplit * d.T + k) * nu * nx + r;
      for (int sp = 0; sp < v.nsplit; ++sp) z += zp[(int64_t)sp * d.T * nu * nx];
    } else {
      z = v.Z[bk * nu * nx + r];
    }
    sX[r] = z - v.Zb[bk * nu * nx + r];
    const int m = r / nx, i = r % nx;
    sK[r] = Kp[i * nu + m];
  }
  if (fz && k == 0 && tid == 0) v.ncorr[b] = 0;   // correction list consumed
  __syncthreads();
  const double rho = v.prm.rho;
  for (int r = tid; r < nu * nx; r += nt) {
    const int m = r / nx, i = r % nx;
    double gp = 0.0, wk = 0.0;
    for (int q = 0; q < nx; ++q) gp += sX[m * nx + q] * Pk[q * nx + i];
    for (int q = 0; q < nu; ++q) wk += Wk[m * nu + q] * sK[q * nx + i];
    sR[r] = 2.0 * wk + rho * st * gp;
  }
  __syncthreads();
  chain_solve(v.fa.V + bk * nu * nu, v.U + bk * nx * nx, v.fa.den + bk * nu * nx, sR, sX,
              nu, nx, tid, nt);
  double* Ko = (mode == 0 ? v.K : kout) + (int64_t)b * d.NK + (int64_t)k * nu * nx;
  for (int r = tid; r < nu * nx; r += nt) {
    const int m = r / nx, i = r % nx;
    Ko[i * nu + m] = sR[r];
  }
  if (mode != 0) return;
  for (int r = tid; r < nx * nu; r += nt) {   // C = sqrt(tau) Psi K^T ; D = 2C - Cold
    const int i = r / nu, m = r % nu;
    double acc = 0.0;
    for (int q = 0; q < nx; ++q) acc += Pk[i * nx + q] * sR[m * nx + q];
    const double c = st * acc;
    const int64_t idx = bk * nx * nu + r;
    const double cold = v.Ccur[idx];
    v.Cprev[idx] = cold;
    v.Ccur[idx] = c;
    v.D[idx] = 2.0 * c - cold;
  }
}

template <int NXC = 0, int NUC = 0>
__global__ void __launch_bounds__(256) k_fa_gain_w(Dev v) {
  extern __shared__ double sm[];
  const Dims d = v.d;
  const int nx = NXC > 0 ? NXC : d.nx, nu = NUC > 0 ? NUC : d.nu;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (gw >= (int64_t)d.B * d.T) return;
  const int b = (int)(gw / d.T), k = (int)(gw % d.T);
  if (!v.active[b]) return;
  const int64_t bk = (int64_t)b * d.T + k;
  double* sR = sm + (size_t)warp * 3 * nu * nx;
  double* sX = sR + nu * nx;
  double* sK = sX + nu * nx;
  const double st = sqrt(v.tau[b]);
  // Psi_k and the Sigma_k eigenvectors U_k are read from the first step of their
  // run of bit-identical Psi blocks (Urep, setup): same values, one cached copy
  // per instance instead of T
  const int kr = v.Urep[bk];
  const double* Pk = v.Psi + ((int64_t)b * (d.T + 1) + kr) * nx * nx;
  const double* Wk = v.W + bk * nu * nu;
  double* Kb = v.K + (int64_t)b * d.NK + (int64_t)k * nu * nx;
  if (v.fused == 2) {
    // TMA path: Z_k = c_l (G_k D_k^T + H_k) [predicted, cones with s^{l-1} = 1;
    // c_1 = 1/2] + Zc [list corrections] + Zctrl [control cones]; then the
    // leave/enter updates of this iteration give G, H of the next one.
    const double cl = (v.iter == 1) ? 0.5 : 1.0;
    const double* Gk = v.G + bk * nu * nu;
    const double* Dk = v.D + bk * nx * nu;
#pragma unroll
  #pragma unroll
  for (int r = lane; r < nu * nx; r += 32) {
      const int m = r / nx, i = r % nx;
      double pr = v.H[bk * nu * nx + r];
#pragma unroll
      for (int q = 0; q < nu; ++q) pr += Gk[m * nu + q] * Dk[i * nu + q];
      sX[r] = cl * pr + v.Zc[bk * nu * nx + r] + v.Zctrl[bk * nu * nx + r] - v.Zb[bk * nu * nx + r];
      sK[r] = Kb[i * nu + m];
    }
    __syncwarp();
    // l = 1: G, H restart from the entering cones (k_project lists s^1 = 1 only)
    if (v.iter == 1) {
      for (int r = lane; r < nu * nx; r += 32) v.H[bk * nu * nx + r] = v.dH[bk * nu * nx + r];
      for (int r = lane; r < nu * nu; r += 32) v.G[bk * nu * nu + r] = v.dG[bk * nu * nu + r];
    } else {
      for (int r = lane; r < nu * nx; r += 32) v.H[bk * nu * nx + r] += v.dH[bk * nu * nx + r];
      for (int r = lane; r < nu * nu; r += 32) v.G[bk * nu * nu + r] += v.dG[bk * nu * nu + r];
    }
  } else {
#pragma unroll
  #pragma unroll
  for (int r = lane; r < nu * nx; r += 32) {
      double z = v.Zc[bk * nu * nx + r];
      const double* zp = v.Zpart + ((int64_t)b * v.nsplit * d.T + k) * nu * nx + r;
      for (int sp = 0; sp < v.nsplit; ++sp) z += zp[(int64_t)sp * d.T * nu * nx];
      sX[r] = z - v.Zb[bk * nu * nx + r];
      const int m = r / nx, i = r % nx;
      sK[r] = Kb[i * nu + m];
    }
  }
  if (k == 0 && lane == 0) v.ncorr[b] = 0;      // correction list consumed
  __syncwarp();
  const double rho = v.prm.rho;
#pragma unroll
  for (int r = lane; r < nu * nx; r += 32) {
    const int m = r / nx, i = r % nx;
    double gp = 0.0, wk = 0.0;
#pragma unroll
    for (int q = 0; q < nx; ++q) gp += sX[m * nx + q] * Pk[q * nx + i];
#pragma unroll
    for (int q = 0; q < nu; ++q) wk += Wk[m * nu + q] * sK[q * nx + i];
    sR[r] = 2.0 * wk + rho * st * gp;
  }
  __syncwarp();
  chain_solve_w<NXC, NUC>(v.fa.V + bk * nu * nu, v.U + ((int64_t)b * d.T + kr) * nx * nx, v.fa.den + bk * nu * nx, sR, sX,
                nu, nx, lane);
#pragma unroll
  for (int r = lane; r < nu * nx; r += 32) {
    const int m = r / nx, i = r % nx;
    Kb[i * nu + m] = sR[r];
  }
#pragma unroll
  for (int r = lane; r < nx * nu; r += 32) {    // C = sqrt(tau) Psi K^T ; D = 2C - Cold
    const int i = r / nu, m = r % nu;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < nx; ++q) acc += Pk[i * nx + q] * sR[m * nx + q];
    const double c = st * acc;
    const int64_t idx = bk * nx * nu + r;
    const double cold = v.Ccur[idx];
    v.Cprev[idx] = cold;
    v.Ccur[idx] = c;
    v.D[idx] = 2.0 * c - cold;
  }
}

// ---------------------------------------------------------------------------
// DR engine.  Affine prox (11a) via the Schur form of K_KKT (F3):
//   (Q_v + sigma I + r_s sum A^T A) k = sigma k~ + r_s sum A^T (eta~ - b_hat)
// per step k: R = sigma K~ + r_s sqrt(tau) (Z - Zb) Psi_k, chain with (W+sigma/2, r_s);
// then chi~ += alpha (chi - chi~) for the k_v part (11c).
__device__ __forceinline__ void cpa8_g(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src) : "memory");
}
// One CTA per (instance, k).  Every operand (Z, Zb, K~, Psi_k, V, U, den) is
// staged into shared memory with cp.async first -- one global round trip
// instead of one per small-matrix loop step (single-instance DR is latency
// bound); Psi_k / U_k come from the first step of their identical-Psi run.
template <int NXC = 0, int NUC = 0>
__global__ void k_dr_gain(Dev v) {
  extern __shared__ double sm[];
  const Dims d = v.d;
  const int nx = NXC > 0 ? NXC : d.nx, nu = NUC > 0 ? NUC : d.nu;
  const int NA = nu * nx, NN = nx * nx, NG = nu * nu;
  const int b = blockIdx.x / d.T, k = blockIdx.x % d.T;
  if (!v.active[b] || !v.dr_active[b]) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t bk = (int64_t)b * d.T + k;
  double* sR = sm;
  double* sX = sR + NA;
  double* sZ = sX + NA;
  double* sKt = sZ + NA;
  double* sden = sKt + NA;
  double* sP = sden + NA;
  double* sU = sP + NN;
  double* sV = sU + NN;
  const int kr = v.Urep[bk];
  const double st = sqrt(v.tau[b]);
  double* Kt = v.Kt + (int64_t)b * d.NK + (int64_t)k * nu * nx;
  const double sg = v.prm.sigma_dr, rs = v.prm.r_s, al = v.prm.alpha_dr;
  {
    const double* Z = v.Z + bk * NA;
    const double* Pk = v.Psi + ((int64_t)b * (d.T + 1) + kr) * NN;
    const double* Uk = v.U + ((int64_t)b * d.T + kr) * NN;
    for (int r = tid; r < NA; r += nt) {
      cpa8_g(sZ + r, Z + r); cpa8_g(sX + r, v.Zb + bk * NA + r);
      cpa8_g(sKt + r, Kt + r); cpa8_g(sden + r, v.dr.den + bk * NA + r);
    }
    for (int r = tid; r < NN; r += nt) { cpa8_g(sP + r, Pk + r); cpa8_g(sU + r, Uk + r); }
    for (int r = tid; r < NG; r += nt) cpa8_g(sV + r, v.dr.V + bk * NG + r);
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  for (int r = tid; r < NA; r += nt) sX[r] = sZ[r] - sX[r];
  __syncthreads();
  for (int r = tid; r < NA; r += nt) {
    const int m = r / nx, i = r % nx;
    double gp = 0.0;
#pragma unroll
    for (int q = 0; q < nx; ++q) gp += sX[m * nx + q] * sP[q * nx + i];
    sR[r] = sg * sKt[i * nu + m] + rs * st * gp;
  }
  __syncthreads();
  chain_solve<NXC, NUC>(sV, sU, sden, sR, sX, nu, nx, tid, nt);
  double* Ko = v.K + (int64_t)b * d.NK + (int64_t)k * nu * nx;
  for (int r = tid; r < NA; r += nt) {
    const int m = r / nx, i = r % nx;
    Ko[i * nu + m] = sR[r];
    Kt[i * nu + m] = sKt[i * nu + m] + al * (sR[r] - sKt[i * nu + m]);
  }
  for (int r = tid; r < NA; r += nt) {
    const int i = r / nu, m = r % nu;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < nx; ++q) acc += sP[i * nx + q] * sR[m * nx + q];
    v.Ccur[bk * NA + r] = st * acc;
  }
}

// DR cone step, one warp per cone:
//   pi = (sigma pi~ + rho p + lambda + r_s t~)/(rho + sigma + r_s)  (p~ part of (11a))
//   s = (pi, a), a = A_hat k + b_hat ; s_ref = 2 s - s~ ; s~ += alpha (Pi(s_ref) - s)
//   pi~ += alpha (pi - pi~) ; r_dr partial = ||s~_new - s~||^2
// NUM > 0: n_u fixed at compile time; the element loops are unrolled so that a
// lane keeps several elements' loads in flight (long c4 cones: 9.6 k elements).
template <int NUM>
__global__ void __launch_bounds__(256) k_dr_pass(Dev v) {
  const Dims d = v.d;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gw >= (int64_t)d.B * d.ng) return;
  const int b = (int)(gw / d.ng), j = (int)(gw % d.ng);
  if (!v.active[b] || !v.dr_active[b]) return;
  {   // Z is re-accumulated by the (split) adjoint right after this pass: zero it here
    const int64_t nz = (int64_t)d.T * d.nu * d.nx;
    double* Zb = v.Z + (int64_t)b * nz;
    for (int64_t e = (int64_t)j * 32 + (threadIdx.x & 31); e < nz; e += (int64_t)d.ng * 32) Zb[e] = 0.0;
  }
  if (j < v.cone_lo || j >= v.cone_hi) return;     // cone-sharded handle: not my cone
  const int lane = threadIdx.x & 31;
  const int nx = d.nx, nu = NUM > 0 ? NUM : d.nu;
  const ConeGeom g = cone_geom(v, j);
  const int64_t ij = (int64_t)b * d.ng + j;
  const double sg = v.prm.sigma_dr, rs = v.prm.r_s, al = v.prm.alpha_dr, rho = v.prm.rho_admm;
  const double pit = v.pit[ij], tt = v.tt[ij];
  const double pi = (sg * pit + rho * v.p[ij] + v.lamp[ij] + rs * tt) / (rho + sg + rs);
  double* Y = v.Y + (int64_t)b * d.E + g.off;
  const double* bh = v.bhat + (int64_t)b * d.E + g.off;
  const double* Bd = v.Bd + (int64_t)b * d.EB + g.offB;
  const double* Cm = v.Ccur + (int64_t)b * d.T * nx * nu;
  double n2 = 0.0;
#pragma unroll 4
  for (int e = lane; e < g.L; e += 32) {
    const int kb = e / nx, i = e - kb * nx;
    double a = (g.kind == 0) ? bh[e] : 0.0;
    if (kb < g.nbB) {
      const double* Cr = Cm + ((int64_t)(g.klo + kb) * nx + i) * nu;
      const double* br = Bd + kb * d.nup;
      if constexpr (NUM > 0) {
#pragma unroll
        for (int m = 0; m < NUM; ++m) a += __ldg(Cr + m) * __ldg(br + m);
      } else {
        for (int m = 0; m < nu; ++m) a += Cr[m] * br[m];
      }
    }
    const double er = 2.0 * a - Y[e];
    n2 += er * er;
  }
  n2 = warp_sum(n2);
  double sc;
  const double tpi = soc_case(2.0 * pi - tt, sqrt(n2), &sc);
  double d2 = 0.0;
#pragma unroll 4
  for (int e = lane; e < g.L; e += 32) {
    const int kb = e / nx, i = e - kb * nx;
    double a = (g.kind == 0) ? bh[e] : 0.0;
    if (kb < g.nbB) {
      const double* Cr = Cm + ((int64_t)(g.klo + kb) * nx + i) * nu;
      const double* br = Bd + kb * d.nup;
      if constexpr (NUM > 0) {
#pragma unroll
        for (int m = 0; m < NUM; ++m) a += __ldg(Cr + m) * __ldg(br + m);
      } else {
        for (int m = 0; m < nu; ++m) a += Cr[m] * br[m];
      }
    }
    const double et = Y[e];
    const double er = 2.0 * a - et;
    const double en = et + al * (sc * er - a);
    Y[e] = en;
    d2 += (en - et) * (en - et);
  }
  d2 = warp_sum(d2);
  if (lane == 0) {
    const double ttn = tt + al * (tpi - pi);
    d2 += (ttn - tt) * (ttn - tt);
    v.tt[ij] = ttn;
    v.pit[ij] = pit + al * (pi - pit);
    v.pt[ij] = pi;
    v.rdr_part[ij] = d2;
  }
}

// Same arithmetic as k_dr_pass, element for element; the forward map a and the
// old eta~ of the cone are computed / loaded once (first sweep, loads batched by
// unrolling, n_u fixed at compile time) and kept in the warp's shared memory for
// the update sweep instead of being recomputed from global memory.
template <int NUM>
__global__ void __launch_bounds__(128) k_dr_pass_s(Dev v, int lmax) {
  extern __shared__ double sm[];
  const Dims d = v.d;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gw >= (int64_t)d.B * d.ng) return;
  const int b = (int)(gw / d.ng), j = (int)(gw % d.ng);
  if (!v.active[b] || !v.dr_active[b]) return;
  {   // Z is re-accumulated by the (split) adjoint right after this pass: zero it here
    const int64_t nz = (int64_t)d.T * d.nu * d.nx;
    double* Zb = v.Z + (int64_t)b * nz;
    for (int64_t e = (int64_t)j * 32 + (threadIdx.x & 31); e < nz; e += (int64_t)d.ng * 32) Zb[e] = 0.0;
  }
  if (j < v.cone_lo || j >= v.cone_hi) return;     // cone-sharded handle: not my cone
  const int lane = threadIdx.x & 31;
  const int nx = d.nx, nu = NUM > 0 ? NUM : d.nu;
  double* sa = sm + (size_t)(threadIdx.x >> 5) * 2 * lmax;
  double* sy = sa + lmax;
  const ConeGeom g = cone_geom(v, j);
  const int64_t ij = (int64_t)b * d.ng + j;
  const double sg = v.prm.sigma_dr, rs = v.prm.r_s, al = v.prm.alpha_dr, rho = v.prm.rho_admm;
  const double pit = v.pit[ij], tt = v.tt[ij];
  const double pi = (sg * pit + rho * v.p[ij] + v.lamp[ij] + rs * tt) / (rho + sg + rs);
  double* Y = v.Y + (int64_t)b * d.E + g.off;
  const double* bh = v.bhat + (int64_t)b * d.E + g.off;
  const double* Bd = v.Bd + (int64_t)b * d.EB + g.offB;
  const double* Cm = v.Ccur + (int64_t)b * d.T * nx * nu;
  double n2 = 0.0;
#pragma unroll 4
  for (int e = lane; e < g.L; e += 32) {
    const int kb = e / nx, i = e - kb * nx;
    double a = (g.kind == 0) ? bh[e] : 0.0;
    if (kb < g.nbB) {
      const double* Cr = Cm + ((int64_t)(g.klo + kb) * nx + i) * nu;
      const double* br = Bd + kb * d.nup;
      if constexpr (NUM > 0) {
#pragma unroll
        for (int m = 0; m < NUM; ++m) a += Cr[m] * br[m];
      } else {
        for (int m = 0; m < nu; ++m) a += Cr[m] * br[m];
      }
    }
    const double et = Y[e];
    sa[e] = a;
    sy[e] = et;
    const double er = 2.0 * a - et;
    n2 += er * er;
  }
  n2 = warp_sum(n2);
  double sc;
  const double tpi = soc_case(2.0 * pi - tt, sqrt(n2), &sc);
  double d2 = 0.0;
  for (int e = lane; e < g.L; e += 32) {
    const double a = sa[e], et = sy[e];
    const double er = 2.0 * a - et;
    const double en = et + al * (sc * er - a);
    Y[e] = en;
    d2 += (en - et) * (en - et);
  }
  d2 = warp_sum(d2);
  if (lane == 0) {
    const double ttn = tt + al * (tpi - pi);
    d2 += (ttn - tt) * (ttn - tt);
    v.tt[ij] = ttn;
    v.pit[ij] = pit + al * (pi - pit);
    v.pt[ij] = pi;
    v.rdr_part[ij] = d2;
  }
}

// Small batches (latency bound, e.g. one c2 instance): one 128-thread CTA per
// cone instead of one warp, so a long cone (up to (T+1) n_x elements) is covered
// by 4x the lanes; same element arithmetic as k_dr_pass, the norm is a block
// reduction (partial sums in a different order).
template <int NUM>
__global__ void __launch_bounds__(128) k_dr_pass_c(Dev v, int lmax) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  const Dims d = v.d;
  const int64_t gc = blockIdx.x;
  if (gc >= (int64_t)d.B * d.ng) return;
  const int b = (int)(gc / d.ng), j = (int)(gc % d.ng);
  if (!v.active[b] || !v.dr_active[b]) return;
  {   // Z is re-accumulated by the (split) adjoint right after this pass: zero it here
    const int64_t nz = (int64_t)d.T * d.nu * d.nx;
    double* Zb = v.Z + (int64_t)b * nz;
    for (int64_t e = (int64_t)j * blockDim.x + threadIdx.x; e < nz; e += (int64_t)d.ng * blockDim.x) Zb[e] = 0.0;
  }
  if (j < v.cone_lo || j >= v.cone_hi) return;     // cone-sharded handle: not my cone
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nx = d.nx, nu = NUM > 0 ? NUM : d.nu;
  double* sa = sm;
  double* sy = sa + lmax;
  const ConeGeom g = cone_geom(v, j);
  const int64_t ij = (int64_t)b * d.ng + j;
  const double sg = v.prm.sigma_dr, rs = v.prm.r_s, al = v.prm.alpha_dr, rho = v.prm.rho_admm;
  const double pit = v.pit[ij], tt = v.tt[ij];
  const double pi = (sg * pit + rho * v.p[ij] + v.lamp[ij] + rs * tt) / (rho + sg + rs);
  double* Y = v.Y + (int64_t)b * d.E + g.off;
  const double* bh = v.bhat + (int64_t)b * d.E + g.off;
  const double* Bd = v.Bd + (int64_t)b * d.EB + g.offB;
  const double* Cm = v.Ccur + (int64_t)b * d.T * nx * nu;
  double n2 = 0.0;
#pragma unroll 2
  for (int e = tid; e < g.L; e += nt) {
    const int kb = e / nx, i = e - kb * nx;
    double a = (g.kind == 0) ? bh[e] : 0.0;
    if (kb < g.nbB) {
      const double* Cr = Cm + ((int64_t)(g.klo + kb) * nx + i) * nu;
      const double* br = Bd + kb * d.nup;
      if constexpr (NUM > 0) {
#pragma unroll
        for (int m = 0; m < NUM; ++m) a += Cr[m] * br[m];
      } else {
        for (int m = 0; m < nu; ++m) a += Cr[m] * br[m];
      }
    }
    const double et = Y[e];
    sa[e] = a;
    sy[e] = et;
    const double er = 2.0 * a - et;
    n2 += er * er;
  }
  n2 = block_sum(n2, red);
  double sc;
  const double tpi = soc_case(2.0 * pi - tt, sqrt(n2), &sc);
  double d2 = 0.0;
  for (int e = tid; e < g.L; e += nt) {
    const double a = sa[e], et = sy[e];
    const double er = 2.0 * a - et;
    const double en = et + al * (sc * er - a);
    Y[e] = en;
    d2 += (en - et) * (en - et);
  }
  d2 = block_sum(d2, red);
  if (tid == 0) {
    const double ttn = tt + al * (tpi - pi);
    d2 += (ttn - tt) * (ttn - tt);
    v.tt[ij] = ttn;
    v.pit[ij] = pit + al * (pi - pit);
    v.pt[ij] = pi;
    v.rdr_part[ij] = d2;
  }
}

// r_dr = ||s~^l - s~^{l-1}||_2 per instance; DR stop test.
__global__ void k_dr_reduce(Dev v) {
  __shared__ double sh[32];
  const Dims d = v.d;
  const int b = blockIdx.x;
  if (!v.active[b] || !v.dr_active[b]) return;
  double acc = 0.0;
  for (int j = threadIdx.x; j < d.ng; j += blockDim.x) acc += v.rdr_part[(int64_t)b * d.ng + j];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    const double r = sqrt(acc);
    v.rdr[b] = r;
    if (!v.prm.fixed_iters && r <= v.prm.eps_dr) v.dr_active[b] = 0;
  }
}

// ---------------------------------------------------------------------------
// Finish: per cone outputs.  FullADMM: nu^L = s y^L,
// lam_nu^L = (1 - s) y^L + (C^L - C^{L-1}) b  ( = lam^{L-1} + a(k^L) - nu^L ).
// Both engines: margin_cone = p~ - ||C^L b + b_hat||.
__global__ void k_finish_cones(Dev v, int engine, double* nu_out, double* lam_out,
                               double* mc_out, int state_norms) {
  const Dims d = v.d;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gw >= (int64_t)d.B * d.ng) return;
  const int b = (int)(gw / d.ng), j = (int)(gw % d.ng);
  const int lane = threadIdx.x & 31;
  const int nx = d.nx, nu = d.nu;
  const ConeGeom g = cone_geom(v, j);
  const int64_t ij = (int64_t)b * d.ng + j;
  const double* Y = v.Y + (int64_t)b * d.E + g.off;
  const double* bh = v.bhat + (int64_t)b * d.E + g.off;
  const double* Bd = v.Bd + (int64_t)b * d.EB + g.offB;
  const double* Cc = v.Ccur + (int64_t)b * d.T * nx * nu;
  const double* Cp = v.Cprev + (int64_t)b * d.T * nx * nu;
  const double s = v.s[ij];
  // state_norms: ||C^L b + b_hat||^2 of state cones already in nrm2 (k_fa_tma margin mode)
  const bool pre = state_norms && g.kind == 0;
  const bool outs = engine == NRTO_FULLADMM && (nu_out || lam_out);
  if (pre && !outs) {
    if (lane == 0 && mc_out) mc_out[ij] = v.pt[ij] - sqrt(v.nrm2[ij]);
    return;
  }
  double n2 = 0.0;
  for (int e = lane; e < g.L; e += 32) {
    const int kb = e / nx, i = e - kb * nx;
    double a = (g.kind == 0) ? bh[e] : 0.0, dlt = 0.0;
    if (kb < g.nbB) {
      const int64_t r = ((int64_t)(g.klo + kb) * nx + i) * nu;
      const double* br = Bd + kb * d.nup;
      for (int m = 0; m < nu; ++m) { a += Cc[r + m] * br[m]; dlt += (Cc[r + m] - Cp[r + m]) * br[m]; }
    }
    n2 += a * a;
    if (outs) {
      const double y = Y[e];
      if (nu_out) nu_out[(int64_t)b * d.E + g.off + e] = s * y;
      if (lam_out) lam_out[(int64_t)b * d.E + g.off + e] = (1.0 - s) * y + dlt;
    }
  }
  n2 = warp_sum(n2);
  if (pre) n2 = v.nrm2[ij];
  if (lane == 0 && mc_out) mc_out[ij] = v.pt[ij] - sqrt(n2);
}

// Finish per instance: dx = F_u du by rollout, margin_lin, objective J.
__global__ void k_finish_inst(Dev v, double* ml_out, double* obj_out) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu;
  const int b = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  double* dx = sm;   // (T+1)*nx
  const double* du = v.du + (int64_t)b * d.T * nu;
  for (int r = tid; r < nx; r += nt) dx[r] = 0.0;
  __syncthreads();
  for (int k = 0; k < d.T; ++k) {
    const double* A = v.A + ((int64_t)b * d.T + k) * nx * nx;
    const double* B = v.Bm + ((int64_t)b * d.T + k) * nx * nu;
    for (int i = tid; i < nx; i += nt) {
      double acc = 0.0;
      for (int q = 0; q < nx; ++q) acc += A[i * nx + q] * dx[k * nx + q];
      for (int q = 0; q < nu; ++q) acc += B[i * nu + q] * du[k * nu + q];
      dx[(k + 1) * nx + i] = acc;
    }
    __syncthreads();
  }
  if (ml_out) {
    const double* grad = v.grad + (int64_t)b * d.ng * nx;
    for (int j = tid; j < d.ng; j += nt) {
      const int k = v.knot[j];
      double bd = 0.0;
      if (v.kind[j] == 0) for (int q = 0; q < nx; ++q) bd += grad[j * nx + q] * dx[k * nx + q];
      else for (int q = 0; q < nu; ++q) bd += grad[j * nx + q] * du[k * nu + q];
      const int64_t ij = (int64_t)b * d.ng + j;
      ml_out[ij] = -(v.g0[ij] + bd + v.p[ij]);
    }
  }
  if (obj_out) {
    double acc = 0.0;
    for (int r = tid; r < d.T * nu; r += nt) {       // (u_hat + du)^T R_u (u_hat + du)
      const int k = r / nu, m = r % nu;
      const double* Ru = v.Ru + ((int64_t)b * d.T + k) * nu * nu;
      const double* uh = v.uhat + ((int64_t)b * d.T + k) * nu;
      double rr = 0.0;
      for (int q = 0; q < nu; ++q) rr += Ru[m * nu + q] * (uh[q] + du[k * nu + q]);
      acc += (uh[m] + du[k * nu + m]) * rr;
    }
    const double* Kb = v.K + (int64_t)b * d.NK;
    for (int r = tid; r < d.NK; r += nt) {           // 1/2 k^T Q_v k = sum <K, W K>
      const int k = r / (nu * nx), rem = r % (nu * nx), i = rem / nu, m = rem % nu;
      const double* Wk = v.W + ((int64_t)b * d.T + k) * nu * nu;
      double wk = 0.0;
      for (int q = 0; q < nu; ++q) wk += Wk[m * nu + q] * Kb[k * nu * nx + i * nu + q];
      acc += Kb[r] * wk;
    }
    acc = block_sum(acc, red);
    if (tid == 0) obj_out[b] = acc;
  }
}

__global__ void k_count_active(Dev v, int32_t* out, int dr) {
  __shared__ double sh[32];
  double c = 0.0;
  for (int b = threadIdx.x; b < v.d.B; b += blockDim.x)
    c += (v.active[b] && (!dr || v.dr_active[b])) ? 1.0 : 0.0;
  c = block_sum(c, sh);
  if (threadIdx.x == 0) *out = (int32_t)c;
}

// Batch residual flags (nrto_solve_flags): [max_b r_p/eps_p, max_b r_d/eps_d,
// #active instances, any instance diverged] -- the operand of the batch-wide
// allreduce(MAX) of the multi-rank termination test.
__global__ void k_solve_flags(Dev v, double* out) {
  __shared__ double sh[4][32];
  double rp = 0.0, rd = 0.0, act = 0.0, dv = 0.0;
  const double ep = v.prm.eps_p > 0 ? v.prm.eps_p : 1.0, ed = v.prm.eps_d > 0 ? v.prm.eps_d : 1.0;
  for (int b = threadIdx.x; b < v.d.B; b += blockDim.x) {
    const double a = v.r_p[b] / ep, c = v.r_d[b] / ed;
    rp = (a > rp || a != a) ? a : rp;      // NaN propagates (diverged)
    rd = (c > rd || c != c) ? c : rd;
    act += v.active[b] ? 1.0 : 0.0;
    dv = (v.status[b] == NRTO_DIVERGED) ? 1.0 : dv;
  }
  double r[4] = {rp, rd, act, dv};
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double x = r[q];
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, x, o);
      x = (q == 2) ? x + y : ((y > x || y != y) ? y : x);
    }
    if (lane == 0) sh[q][w] = x;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    const int q = threadIdx.x;
    double x = (q == 2) ? 0.0 : sh[q][0];
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      const double y = sh[q][i];
      x = (q == 2) ? x + y : ((y > x || y != y) ? y : x);
    }
    out[q] = x;
  }
}

// Standalone batched SOC projection (nrto_soc_project).
__global__ void k_soc_project(const double* t, const double* y, const int64_t* off, int64_t n,
                              double* to, double* yo) {
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= n) return;
  const int lane = threadIdx.x & 31;
  const int64_t a = off[w], e = off[w + 1];
  double n2 = 0.0;
  for (int64_t r = a + lane; r < e; r += 32) n2 += y[r] * y[r];
  n2 = warp_sum(n2);
  double s;
  const double tp = soc_case(t[w], sqrt(n2), &s);
  for (int64_t r = a + lane; r < e; r += 32) yo[r] = s * y[r];
  if (lane == 0) to[w] = tp;
}

// ---------------------------------------------------------------------------
static inline unsigned warp_grid(int64_t warps, int wpb) {
  return (unsigned)((warps + wpb - 1) / wpb);
}

cudaError_t launch_adjoint(nrto_handle_s* h, const double* y, const double* scale,
                           const int32_t* act, cudaStream_t st) {
  Dev& v = h->dev;
  if (v.d.nu <= 8 && v.d.nx <= 32)
    return launch_zlist(h, y, nullptr, nullptr, scale, nullptr, v.d.ng, act, v.Z, st);
  k_adjoint<<<v.d.B * v.d.T, 128, 0, st>>>(v, y, scale, act);
  h->launches++;
  return cudaGetLastError();
}

cudaError_t launch_fa_pass(nrto_handle_s* h, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  if ((int64_t)d.B * d.ng > 0) {
    k_fa_pass<<<warp_grid((int64_t)d.B * d.ng, 8), 256, 0, st>>>(v);
    h->launches++;
  }
  return cudaGetLastError();
}

cudaError_t launch_fa_gain(nrto_handle_s* h, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  if (v.fused) {
    const int64_t nw = (int64_t)d.B * d.T;
    // small CTAs (NRTO_GAIN_WARPS, default 4) fit beside the co-resident QP CTAs
    static const int gwp = [] { const char* e = getenv("NRTO_GAIN_WARPS"); return e ? atoi(e) : 4; }();
    const unsigned gg = (unsigned)((nw + gwp - 1) / gwp);
    const size_t gsm = gwp * 3 * d.nu * d.nx * sizeof(double);
    if (d.nx == 14 && d.nu == 7) k_fa_gain_w<14, 7><<<gg, 32 * gwp, gsm, st>>>(v);
    else if (d.nx == 12 && d.nu == 4) k_fa_gain_w<12, 4><<<gg, 32 * gwp, gsm, st>>>(v);
    else k_fa_gain_w<><<<gg, 32 * gwp, gsm, st>>>(v);
    h->launches++;
    return cudaGetLastError();
  }
  k_fa_gain<<<d.B * d.T, 128, 3 * d.nu * d.nx * sizeof(double), st>>>(v, 0, nullptr, nullptr);
  h->launches++;
  return cudaGetLastError();
}

cudaError_t launch_dr_gain(nrto_handle_s* h, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  const size_t smem = (5 * (size_t)d.nu * d.nx + 2 * (size_t)d.nx * d.nx + (size_t)d.nu * d.nu) * sizeof(double);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_dr_gain<>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (d.nx == 12 && d.nu == 4) k_dr_gain<12, 4><<<d.B * d.T, 128, smem, st>>>(v);
  else if (d.nx == 14 && d.nu == 7) k_dr_gain<14, 7><<<d.B * d.T, 128, smem, st>>>(v);
  else k_dr_gain<><<<d.B * d.T, 128, smem, st>>>(v);
  h->launches++;
  return cudaGetLastError();
}

cudaError_t launch_dr_pass(nrto_handle_s* h, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  if ((int64_t)d.B * d.ng > 0) {
    const int lmax = (d.T + 1) * d.nx;                 // longest cone
    const size_t smem = 4 * 2 * (size_t)lmax * sizeof(double);
    const int64_t ncone = (int64_t)d.B * d.ng;
    if (ncone <= 8192 && 2 * (size_t)lmax * sizeof(double) <= 48 * 1024) {   // CTA per cone
      const size_t sm1 = 2 * (size_t)lmax * sizeof(double);
      if (d.nu == 4) k_dr_pass_c<4><<<(unsigned)ncone, 128, sm1, st>>>(v, lmax);
      else if (d.nu == 7) k_dr_pass_c<7><<<(unsigned)ncone, 128, sm1, st>>>(v, lmax);
      else k_dr_pass_c<0><<<(unsigned)ncone, 128, sm1, st>>>(v, lmax);
    } else if (smem <= 100 * 1024) {
      const unsigned grid = warp_grid((int64_t)d.B * d.ng, 4);
      if (smem > 48 * 1024) {
        cudaFuncSetAttribute(k_dr_pass_s<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_dr_pass_s<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_dr_pass_s<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      }
      if (d.nu == 4) k_dr_pass_s<4><<<grid, 128, smem, st>>>(v, lmax);
      else if (d.nu == 7) k_dr_pass_s<7><<<grid, 128, smem, st>>>(v, lmax);
      else k_dr_pass_s<0><<<grid, 128, smem, st>>>(v, lmax);
    } else {
      if (d.nu == 4) k_dr_pass<4><<<warp_grid((int64_t)d.B * d.ng, 8), 256, 0, st>>>(v);
      else if (d.nu == 7) k_dr_pass<7><<<warp_grid((int64_t)d.B * d.ng, 8), 256, 0, st>>>(v);
      else k_dr_pass<0><<<warp_grid((int64_t)d.B * d.ng, 8), 256, 0, st>>>(v);
    }
    h->launches++;
  }
  return cudaGetLastError();
}

// DR adjoint Z_k = sum_j b_{j,k} eta~_{j,k}^T over every cone; Z was zeroed by the pass.
cudaError_t launch_dr_adjoint(nrto_handle_s* h, cudaStream_t st) {
  Dev& v = h->dev;
  if (v.d.nu <= 8 && v.d.nx <= 16)
    return launch_zlist(h, v.Y, nullptr, nullptr, nullptr, nullptr, v.d.ng, v.dr_active, v.Z, st, 0, 0,
                        nullptr, nullptr, 1);
  return launch_adjoint(h, v.Y, nullptr, v.dr_active, st);
}

cudaError_t launch_dr_reduce(nrto_handle_s* h, cudaStream_t st) {
  // one partial per thread for n_g <= 1024 (the per-instance sum is a latency chain otherwise)
  k_dr_reduce<<<h->dev.d.B, h->dev.d.ng >= 512 ? 1024 : 256, 0, st>>>(h->dev);
  h->launches++;
  return cudaGetLastError();
}

cudaError_t launch_finish(nrto_handle_s* h, int engine, const nrto_out* o, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  int pre = 0;
  if (v.fused == 2 && o->margin_cone && v.nwitems > 0) {   // state-cone margins by the TMA pass
    h->tma_margin = 1;
    cudaError_t e = launch_fa_tma(h, st);
    h->tma_margin = 0;
    if (e != cudaSuccess) return e;
    pre = 1;
  }
  if ((int64_t)d.B * d.ng > 0) {
    k_finish_cones<<<warp_grid((int64_t)d.B * d.ng, 8), 256, 0, st>>>(
        v, engine, o->nu, o->lam_nu, o->margin_cone, pre);
    h->launches++;
  }
  const size_t fsm = (size_t)(d.T + 1) * d.nx * sizeof(double);   // rollout dx (long horizons > 48 KB)
  if (fsm > 48 * 1024) {
    if (fsm > 227 * 1024) return cudaErrorInvalidValue;
    cudaFuncSetAttribute(k_finish_inst, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
  }
  k_finish_inst<<<d.B, 128, fsm, st>>>(v, o->margin_lin, o->objective);
  h->launches++;
  return cudaGetLastError();
}

cudaError_t launch_finish_inst(nrto_handle_s* h, double* margin_lin, double* objective, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  const size_t fsm = (size_t)(d.T + 1) * d.nx * sizeof(double);
  if (fsm > 48 * 1024) {
    if (fsm > 227 * 1024) return cudaErrorInvalidValue;
    cudaFuncSetAttribute(k_finish_inst, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
  }
  k_finish_inst<<<d.B, 128, fsm, st>>>(v, margin_lin, objective);
  h->launches++;
  return cudaGetLastError();
}

cudaError_t launch_gain_update(nrto_handle_s* h, const double* nu, const double* kv_prev,
                               double* kv_next, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  // accumulate into the handle's own Zg, not Z: Z carries the DR engine's warm
  // adjoint of eta~ between solves, which a standalone gain update must keep
  double* const zkeep = v.Z;
  v.Z = v.Zg;
  cudaError_t e = launch_adjoint(h, nu, nullptr, nullptr, st);
  if (e == cudaSuccess) {
    k_fa_gain<<<d.B * d.T, 128, 3 * d.nu * d.nx * sizeof(double), st>>>(v, 1, kv_prev, kv_next);
    h->launches++;
    e = cudaGetLastError();
  }
  v.Z = zkeep;
  return e;
}

cudaError_t launch_soc_project(const double* t, const double* y, const int64_t* off, int64_t n,
                               double* to, double* yo, cudaStream_t st) {
  if (n > 0) k_soc_project<<<warp_grid(n, 8), 256, 0, st>>>(t, y, off, n, to, yo);
  return cudaGetLastError();
}

cudaError_t launch_solve_flags(nrto_handle_s* h, double* flags, cudaStream_t st) {
  k_solve_flags<<<1, 256, 0, st>>>(h->dev, flags);
  h->launches++;
  return cudaGetLastError();
}

cudaError_t launch_count_active(nrto_handle_s* h, int32_t* d_count, int dr, cudaStream_t st) {
  k_count_active<<<1, 256, 0, st>>>(h->dev, d_count, dr);
  h->launches++;
  return cudaGetLastError();
}

}  // namespace nrto
