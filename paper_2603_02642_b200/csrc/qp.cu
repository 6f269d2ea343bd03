// (14a) / (5b) QP by OSQP-form ADMM with a Riccati x-step (DESIGN R1),
// fused with the dual update and the residual / termination test of the outer
// iteration: FullADMM (16) + P:505-507, or NRTO-ADMM (5c).
#include "common.cuh"
#include <cmath>
#include <cstdlib>
#include <algorithm>

namespace nrto {

// min(a, b) of the row projection z_l = min(., -g_l) that PROPAGATES NaN (IEEE fmin
// returns the non-NaN operand): a non-finite input must end as NRTO_DIVERGED
__device__ __forceinline__ double nan_min(double a, double b) {
  return (a != a || b != b) ? a + b : fmin(a, b);
}

// One CTA per instance.  x = (du, p), z = (z_lin, z_ball), y dual.
//   rhs_p = sigma p + rho v + rho_q z_lin - y_lin
//   w     = rho_q z_lin - y_lin - beta rhs_p,           beta = rho_q/(rho+sigma+rho_q)
//   (R~ + F_u^T Q~ F_u) du~ = r_u + F_u^T r_x  with r_u = sigma du - 2 R_u u_hat + scatter_ctrl(w),
//                                                  r_x = scatter_state(w) + rho_q z_ball - y_ball
//   p~' = (rhs_p - rho_q B du~)/(rho+sigma+rho_q),  z~ = (B du~ + p~', F_u du~)
//   x <- a x~ + (1-a) x ; z <- Pi(a z~ + (1-a) z + y/rho_q) ; y += rho_q (a z~ + (1-a) z - z_new)
__global__ void __launch_bounds__(128) k_qp(Dev v, int engine, int l) {
  __shared__ double sv[2][32];
  __shared__ double red[32];
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, T = d.T, ng = d.ng;
  const int b = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  if (!v.active[b]) return;
  const EngineFactors& F = engine == NRTO_FULLADMM ? v.fa : v.dr;
  const double rho = engine == NRTO_FULLADMM ? v.prm.rho : v.prm.rho_admm;
  const double rq = v.prm.rho_qp, sq = v.prm.sigma_qp, aq = v.prm.alpha_qp;
  const double den = rho + sq + rq, beta = rq / den;
  const int64_t bg = (int64_t)b * ng;
  const double* grad = v.grad + bg * nx;
  const double* g0 = v.g0 + bg;
  double* p = v.p + bg; double* zl = v.zl + bg; double* yl = v.yl + bg;
  double* rp = v.rp + bg; double* wq = v.wq + bg;
  const double* pt = v.pt + bg; double* lam = v.lamp + bg;
  double* zb = v.zb + (int64_t)b * (T + 1) * nx; double* yb = v.yb + (int64_t)b * (T + 1) * nx;
  double* rx = v.rx + (int64_t)b * (T + 1) * nx; double* dxt = v.dxt + (int64_t)b * (T + 1) * nx;
  double* du = v.du + (int64_t)b * T * nu; double* ru = v.ru + (int64_t)b * T * nu;
  double* kff = v.kff + (int64_t)b * T * nu; double* dut = v.dut + (int64_t)b * T * nu;
  const double* Ru = v.Ru + (int64_t)b * T * nu * nu;
  const double* uh = v.uhat + (int64_t)b * T * nu;
  const double* Bm = v.Bm + (int64_t)b * T * nx * nu;
  const double* Kf = F.Kf + (int64_t)b * T * nu * nx;
  const double* Acl = F.Acl + (int64_t)b * T * nx * nx;
  const double* Hi = F.Hinv + (int64_t)b * T * nu * nu;
  const double* HB = F.HB + (int64_t)b * T * nu * nx;
  const double rtr = v.rtrust[b];
  const double rinv = (engine == NRTO_FULLADMM) ? 1.0 : 1.0 / rho;

  for (int it = 0; it < v.prm.qp_iters; ++it) {
    for (int j = tid; j < ng; j += nt) {
      const double vj = pt[j] - lam[j] * rinv;   // FullADMM: p~ - lam_p ; DR: p~ - lambda/rho
      const double r = sq * p[j] + rho * vj + rq * zl[j] - yl[j];
      rp[j] = r;
      wq[j] = rq * zl[j] - yl[j] - beta * r;
    }
    __syncthreads();
    for (int r = tid; r < (T + 1) * nx; r += nt) {
      const int k = r / nx, i = r % nx;
      double acc = 0.0;
      if (k > 0) {
        acc = rq * zb[r] - yb[r];
        for (int q = v.sptr[k]; q < v.sptr[k + 1]; ++q) {
          const int j = v.srow[q];
          acc += grad[j * nx + i] * wq[j];
        }
      }
      rx[r] = acc;
    }
    for (int r = tid; r < T * nu; r += nt) {
      const int k = r / nu, m = r % nu;
      double acc = sq * du[r];
      for (int q = 0; q < nu; ++q) acc -= 2.0 * Ru[(k * nu + m) * nu + q] * uh[k * nu + q];
      for (int q = v.cptr[k]; q < v.cptr[k + 1]; ++q) {
        const int j = v.crow[q];
        acc += grad[j * nx + m] * wq[j];
      }
      ru[r] = acc;
    }
    __syncthreads();
    // backward sweep: s_k = r_x,k + Acl_k^T s_{k+1} - Kf_k^T r_u,k ;
    //                 kff_k = H_uu^-1 r_u,k + H_uu^-1 B_k^T s_{k+1}
    int cur = 0;
    if (tid < nx) sv[0][tid] = rx[T * nx + tid];
    __syncthreads();
    for (int k = T - 1; k >= 0; --k) {
      const double* s = sv[cur];
      if (tid < nx) {
        const double* Ac = Acl + (int64_t)k * nx * nx;
        const double* Kk = Kf + (int64_t)k * nu * nx;
        double acc = rx[k * nx + tid];
        for (int r = 0; r < nx; ++r) acc += Ac[r * nx + tid] * s[r];
        for (int m = 0; m < nu; ++m) acc -= Kk[m * nx + tid] * ru[k * nu + m];
        sv[cur ^ 1][tid] = acc;
      } else if (tid >= 32 && tid < 32 + nu) {
        const int m = tid - 32;
        const double* H = Hi + (int64_t)k * nu * nu;
        const double* hb = HB + (int64_t)k * nu * nx;
        double acc = 0.0;
        for (int q = 0; q < nu; ++q) acc += H[m * nu + q] * ru[k * nu + q];
        for (int r = 0; r < nx; ++r) acc += hb[m * nx + r] * s[r];
        kff[k * nu + m] = acc;
      }
      __syncthreads();
      cur ^= 1;
    }
    // forward sweep: du~_k = kff_k - Kf_k dx_k ; dx_{k+1} = Acl_k dx_k + B_k kff_k
    if (tid < nx) dxt[tid] = 0.0;
    __syncthreads();
    for (int k = 0; k < T; ++k) {
      const double* x = dxt + k * nx;
      if (tid < nx) {
        const double* Ac = Acl + (int64_t)k * nx * nx;
        const double* Bk = Bm + (int64_t)k * nx * nu;
        double acc = 0.0;
        for (int r = 0; r < nx; ++r) acc += Ac[tid * nx + r] * x[r];
        for (int m = 0; m < nu; ++m) acc += Bk[tid * nu + m] * kff[k * nu + m];
        dxt[(k + 1) * nx + tid] = acc;
      } else if (tid >= 32 && tid < 32 + nu) {
        const int m = tid - 32;
        const double* Kk = Kf + (int64_t)k * nu * nx;
        double acc = kff[k * nu + m];
        for (int r = 0; r < nx; ++r) acc -= Kk[m * nx + r] * x[r];
        dut[k * nu + m] = acc;
      }
      __syncthreads();
    }
    // linear rows
    for (int j = tid; j < ng; j += nt) {
      const int k = v.knot[j];
      double bd = 0.0;
      if (v.kind[j] == 0) for (int q = 0; q < nx; ++q) bd += grad[j * nx + q] * dxt[k * nx + q];
      else for (int q = 0; q < nu; ++q) bd += grad[j * nx + q] * dut[k * nu + q];
      const double ptl = (rp[j] - rq * bd) / den;
      const double ztl = bd + ptl;
      p[j] = aq * ptl + (1.0 - aq) * p[j];
      const double zh = aq * ztl + (1.0 - aq) * zl[j];
      const double zn = nan_min(zh + yl[j] / rq, -g0[j]);
      yl[j] += rq * (zh - zn);
      zl[j] = zn;
    }
    for (int r = tid; r < T * nu; r += nt) du[r] = aq * dut[r] + (1.0 - aq) * du[r];
    __syncthreads();   // dxt is overwritten below
    // trust-region ball on F_u du (all knots; knot 0 is identically 0)
    double nb = 0.0;
    for (int r = tid; r < (T + 1) * nx; r += nt) {
      const double zh = aq * dxt[r] + (1.0 - aq) * zb[r];
      dxt[r] = zh;
      const double w = zh + yb[r] / rq;
      nb += w * w;
    }
    nb = sqrt(block_sum(nb, red));
    const double scl = (nb > rtr) ? rtr / nb : 1.0;
    for (int r = tid; r < (T + 1) * nx; r += nt) {
      const double zh = dxt[r];
      const double zn = scl * (zh + yb[r] / rq);
      yb[r] += rq * (zh - zn);
      zb[r] = zn;
    }
    __syncthreads();
  }
  // ---- dual update + residuals of the outer iteration
  double ap = 0.0, ad = 0.0;
  double* tin = v.tin + bg;
  double* ptp = v.ptprev + bg;
  for (int j = tid; j < ng; j += nt) {
    const double dp = p[j] - pt[j];
    if (engine == NRTO_FULLADMM) {       // (16): lam_p += p - p~ ; next t = p + lam_p
      lam[j] += dp;
      tin[j] = p[j] + lam[j];
    } else {                              // (5c): lambda += rho (p - p~)   (R4)
      lam[j] += rho * dp;
    }
    ap += dp * dp;
    const double dd = pt[j] - ptp[j];
    ad += dd * dd;
    ptp[j] = pt[j];
  }
  ap = block_sum(ap, red);
  ad = block_sum(ad, red);
  if (tid == 0) {
    const double rpv = sqrt(ap), rdv = rho * sqrt(ad);
    v.r_p[b] = rpv;
    v.r_d[b] = rdv;
    record_hist(v, b, l, rpv, rdv, engine);
    v.iters[b] = l;
    if (!isfinite(rpv) || !isfinite(rdv)) {
      v.status[b] = NRTO_DIVERGED;
      v.active[b] = 0;
    } else if (!v.prm.fixed_iters && (l % v.prm.check_every) == 0 && rpv <= v.prm.eps_p &&
               rdv <= v.prm.eps_d) {
      v.status[b] = NRTO_CONVERGED;
      v.active[b] = 0;
    }
  }
}

// Staged variant: the per-step closed-loop matrices Acl_k of the instance are
// copied to shared memory once per call, the k-independent parts of the
// Riccati solve are computed in parallel phases, and only the two linear
// recurrences  s_k = a_k + Acl_k^T s_{k+1}  (backward) and
// dx_{k+1} = Acl_k dx_k + e_k  (forward) run sequentially, on one warp with
// the vector held in registers and exchanged by shuffles:
//   a_k  = r_x,k - Kf_k^T r_u,k          kff_k = H^-1 r_u,k + H^-1 B_k^T s_{k+1}
//   e_k  = B_k kff_k                      du~_k = kff_k - Kf_k dx_k
__global__ void __launch_bounds__(1024) k_qp_staged(Dev v, int engine, int l, int stageA) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, T = d.T, ng = d.ng;
  const int b = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  if (!v.active[b]) return;
  const EngineFactors& F = engine == NRTO_FULLADMM ? v.fa : v.dr;
  const double rho = engine == NRTO_FULLADMM ? v.prm.rho : v.prm.rho_admm;
  const double rq = v.prm.rho_qp, sq = v.prm.sigma_qp, aq = v.prm.alpha_qp;
  const double den = rho + sq + rq, beta = rq / den;
  const int64_t bg = (int64_t)b * ng;
  const double* grad = v.grad + bg * nx;
  const double* g0 = v.g0 + bg;
  double* p = v.p + bg; double* zl = v.zl + bg; double* yl = v.yl + bg;
  double* rp = v.rp + bg; double* wq = v.wq + bg;
  const double* pt = v.pt + bg; double* lam = v.lamp + bg;
  double* zb = v.zb + (int64_t)b * (T + 1) * nx; double* yb = v.yb + (int64_t)b * (T + 1) * nx;
  double* du = v.du + (int64_t)b * T * nu;
  const double* Ru = v.Ru + (int64_t)b * T * nu * nu;
  const double* uh = v.uhat + (int64_t)b * T * nu;
  const double* Bm = v.Bm + (int64_t)b * T * nx * nu;
  const double* Kf = F.Kf + (int64_t)b * T * nu * nx;
  const double* AclG = F.Acl + (int64_t)b * T * nx * nx;
  const double* Hi = F.Hinv + (int64_t)b * T * nu * nu;
  const double* HB = F.HB + (int64_t)b * T * nu * nx;
  const double rtr = v.rtrust[b];
  const double rinv = (engine == NRTO_FULLADMM) ? 1.0 : 1.0 / rho;
  // shared memory
  double* sS = sm;                          // [(T+1) nx]  s_k, then dx_k, then z^_ball
  double* sA = sS + (T + 1) * nx;           // [T nx]      a_k, then e_k
  double* sK = sA + T * nx;                 // [T nu]      kff_k
  double* sR = sK + T * nu;                 // [T nu]      r_u,k, then du~_k
  double* sAcl = sR + T * nu;               // [T nx nx]   (stageA)
  const double* Acl = stageA ? sAcl : AclG;
  if (stageA)
    for (int r = tid; r < T * nx * nx; r += nt) sAcl[r] = AclG[r];

  for (int it = 0; it < v.prm.qp_iters; ++it) {
    for (int j = tid; j < ng; j += nt) {
      const double vj = pt[j] - lam[j] * rinv;   // FullADMM: p~ - lam_p ; DR: p~ - lambda/rho
      const double r = sq * p[j] + rho * vj + rq * zl[j] - yl[j];
      rp[j] = r;
      wq[j] = rq * zl[j] - yl[j] - beta * r;
    }
    __syncthreads();
    for (int r = tid; r < T * nu; r += nt) {      // r_u
      const int k = r / nu, m = r % nu;
      double acc = sq * du[r];
#pragma unroll 4
      for (int q = 0; q < nu; ++q) acc -= 2.0 * __ldg(Ru + (k * nu + m) * nu + q) * __ldg(uh + k * nu + q);
#pragma unroll 4
      for (int q = __ldg(v.cptr + k); q < __ldg(v.cptr + k + 1); ++q) {
        const int j = __ldg(v.crow + q);
        acc += __ldg(grad + j * nx + m) * wq[j];
      }
      sR[r] = acc;
    }
    __syncthreads();
    for (int r = tid; r < (T + 1) * nx; r += nt) { // r_x and a_k
      const int k = r / nx, i = r % nx;
      double acc = 0.0;
      if (k > 0) {
        acc = rq * zb[r] - yb[r];
#pragma unroll 8
        for (int q = __ldg(v.sptr + k); q < __ldg(v.sptr + k + 1); ++q) {
          const int j = __ldg(v.srow + q);
          acc += __ldg(grad + j * nx + i) * wq[j];
        }
      }
      if (k < T) {
        const double* Kk = Kf + (int64_t)k * nu * nx;
#pragma unroll 4
        for (int m = 0; m < nu; ++m) acc -= __ldg(Kk + m * nx + i) * sR[k * nu + m];
        sA[r] = acc;
      } else {
        sS[r] = acc;
      }
    }
    __syncthreads();
    if (tid < 32) {                               // backward recurrence (one warp)
      double s = (tid < nx) ? sS[T * nx + tid] : 0.0;
      const int ic = tid < nx ? tid : 0;
      for (int k = T - 1; k >= 0; --k) {
        const double* Ak = Acl + (size_t)k * nx * nx + ic;
        double a0 = sA[k * nx + ic], a1 = 0.0, a2 = 0.0, a3 = 0.0;   // 4 chains (ILP)
        int r = 0;
        for (; r + 4 <= nx; r += 4) {
          a0 += Ak[(r + 0) * nx] * __shfl_sync(0xffffffffu, s, r + 0);
          a1 += Ak[(r + 1) * nx] * __shfl_sync(0xffffffffu, s, r + 1);
          a2 += Ak[(r + 2) * nx] * __shfl_sync(0xffffffffu, s, r + 2);
          a3 += Ak[(r + 3) * nx] * __shfl_sync(0xffffffffu, s, r + 3);
        }
        for (; r < nx; ++r) a0 += Ak[r * nx] * __shfl_sync(0xffffffffu, s, r);
        s = (a0 + a1) + (a2 + a3);
        if (tid < nx) sS[k * nx + tid] = s;
      }
    }
    __syncthreads();
    for (int r = tid; r < T * nu; r += nt) {      // kff_k
      const int k = r / nu, m = r % nu;
      const double* H = Hi + (int64_t)k * nu * nu;
      const double* hb = HB + (int64_t)k * nu * nx;
      double acc = 0.0;
#pragma unroll 4
      for (int q = 0; q < nu; ++q) acc += __ldg(H + m * nu + q) * sR[k * nu + q];
#pragma unroll 4
      for (int i = 0; i < nx; ++i) acc += __ldg(hb + m * nx + i) * sS[(k + 1) * nx + i];
      sK[r] = acc;
    }
    __syncthreads();
    for (int r = tid; r < T * nx; r += nt) {      // e_k = B_k kff_k
      const int k = r / nx, i = r % nx;
      const double* Bk = Bm + (int64_t)k * nx * nu;
      double acc = 0.0;
#pragma unroll 4
      for (int m = 0; m < nu; ++m) acc += __ldg(Bk + i * nu + m) * sK[k * nu + m];
      sA[r] = acc;
    }
    __syncthreads();
    if (tid < 32) {                               // forward recurrence (one warp)
      double x = 0.0;
      const int ic = tid < nx ? tid : 0;
      if (tid < nx) sS[tid] = 0.0;
      for (int k = 0; k < T; ++k) {
        const double* Ak = Acl + (size_t)k * nx * nx + ic * nx;
        double a0 = sA[k * nx + ic], a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int r = 0;
        for (; r + 4 <= nx; r += 4) {
          a0 += Ak[r + 0] * __shfl_sync(0xffffffffu, x, r + 0);
          a1 += Ak[r + 1] * __shfl_sync(0xffffffffu, x, r + 1);
          a2 += Ak[r + 2] * __shfl_sync(0xffffffffu, x, r + 2);
          a3 += Ak[r + 3] * __shfl_sync(0xffffffffu, x, r + 3);
        }
        for (; r < nx; ++r) a0 += Ak[r] * __shfl_sync(0xffffffffu, x, r);
        x = (a0 + a1) + (a2 + a3);
        if (tid < nx) sS[(k + 1) * nx + tid] = x;
      }
    }
    __syncthreads();
    for (int r = tid; r < T * nu; r += nt) {      // du~_k
      const int k = r / nu, m = r % nu;
      const double* Kk = Kf + (int64_t)k * nu * nx;
      double acc = sK[r];
#pragma unroll 4
      for (int q = 0; q < nx; ++q) acc -= __ldg(Kk + m * nx + q) * sS[k * nx + q];
      sR[r] = acc;
    }
    __syncthreads();
    for (int j = tid; j < ng; j += nt) {          // linear rows
      const int k = v.knot[j];
      double bd = 0.0;
      if (v.kind[j] == 0) {
#pragma unroll 4
        for (int q = 0; q < nx; ++q) bd += __ldg(grad + j * nx + q) * sS[k * nx + q];
      } else {
#pragma unroll 4
        for (int q = 0; q < nu; ++q) bd += __ldg(grad + j * nx + q) * sR[k * nu + q];
      }
      const double ptl = (rp[j] - rq * bd) / den;
      const double ztl = bd + ptl;
      p[j] = aq * ptl + (1.0 - aq) * p[j];
      const double zh = aq * ztl + (1.0 - aq) * zl[j];
      const double zn = nan_min(zh + yl[j] / rq, -g0[j]);
      yl[j] += rq * (zh - zn);
      zl[j] = zn;
    }
    for (int r = tid; r < T * nu; r += nt) du[r] = aq * sR[r] + (1.0 - aq) * du[r];
    __syncthreads();
    double nb = 0.0;                              // trust-region ball on F_u du
    for (int r = tid; r < (T + 1) * nx; r += nt) {
      const double zh = aq * sS[r] + (1.0 - aq) * zb[r];
      sS[r] = zh;
      const double w = zh + yb[r] / rq;
      nb += w * w;
    }
    nb = sqrt(block_sum(nb, red));
    const double scl = (nb > rtr) ? rtr / nb : 1.0;
    for (int r = tid; r < (T + 1) * nx; r += nt) {
      const double zh = sS[r];
      const double zn = scl * (zh + yb[r] / rq);
      yb[r] += rq * (zh - zn);
      zb[r] = zn;
    }
    __syncthreads();
  }
  // ---- dual update + residuals of the outer iteration
  double ap = 0.0, ad = 0.0;
  double* tin = v.tin + bg;
  double* ptp = v.ptprev + bg;
  for (int j = tid; j < ng; j += nt) {
    const double dp = p[j] - pt[j];
    if (engine == NRTO_FULLADMM) {       // (16): lam_p += p - p~ ; next t = p + lam_p
      lam[j] += dp;
      tin[j] = p[j] + lam[j];
    } else {                              // (5c): lambda += rho (p - p~)   (R4)
      lam[j] += rho * dp;
    }
    ap += dp * dp;
    const double dd = pt[j] - ptp[j];
    ad += dd * dd;
    ptp[j] = pt[j];
  }
  ap = block_sum(ap, red);
  ad = block_sum(ad, red);
  if (tid == 0) {
    const double rpv = sqrt(ap), rdv = rho * sqrt(ad);
    v.r_p[b] = rpv;
    v.r_d[b] = rdv;
    record_hist(v, b, l, rpv, rdv, engine);
    v.iters[b] = l;
    if (!isfinite(rpv) || !isfinite(rdv)) {
      v.status[b] = NRTO_DIVERGED;
      v.active[b] = 0;
    } else if (!v.prm.fixed_iters && (l % v.prm.check_every) == 0 && rpv <= v.prm.eps_p &&
               rdv <= v.prm.eps_d) {
      v.status[b] = NRTO_CONVERGED;
      v.active[b] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// cp.async helpers of the sparse-row QP below.
__device__ __forceinline__ void cpa8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src) : "memory");
}
__device__ __forceinline__ void cpa16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kQPRing = QP_RING;   // power of two (common.cuh)
#ifndef QP_MINB
#define QP_MINB 4
#endif
#ifndef QP_THREADS
#define QP_THREADS 256
#endif
#ifndef QP_CHUNK            // recurrence steps per bulk copy (divides QP_RING)
#define QP_CHUNK 4
#endif

// ---------------------------------------------------------------------------
// Sparse-row QP, sized to co-reside with the TMA cone pass (256 threads, <= 48
// registers, ~24 KB shared memory).  The constraint gradients are kept in a
// compressed row form built at setup (<= 8 nonzeros per row, else dense), and
// the row phase of QP iteration m gathers (B du~)_j, updates (p, z, y)_j and
// immediately scatters the NEXT iteration's w_j grad_j into the knot
// accumulators S_k / U_k with FP64 RED.ADD -- each row is read once per QP
// iteration (SURVEY F4 products with B and B^T).
constexpr int kRowNZ = 8;

// Packed row record (setup, k_sparse_rows): {knot, kind | nz << 8, idx0..3, idx4..7}
// (nz = 255: dense row, read from grad).  The values sit in gval[row][8].
__device__ __forceinline__ int rec_idx(const int4& r, int s) {
  const uint32_t w = (s < 4) ? (uint32_t)r.z : (uint32_t)r.w;
  return (int)((w >> (8 * (s & 3))) & 0xffu);
}

// Rows of one QP iteration, 4 rows per thread in flight: (it) gather
// bd_j = <grad_j, x_k> (x = dx~ for state rows, du~ for control rows), update
// (p, z, y)_j, and (more) form the next iteration's rhs_p / w_j and scatter
// w_j grad_j into S_k / U_k (FP64 RED.ADD).  first: only the rhs / scatter.
constexpr int kRowBatch = QP_THREADS >= 256 ? 2 : 4;
template <bool FIRST, int U>
__device__ __forceinline__ void qp_rows(const Dev& v, int64_t bg, int ng, int tid, int nt,
                                        const double* __restrict__ grad,
                                        const double* __restrict__ g0, double* p, double* zl,
                                        double* yl, double* vv, const double* pt,
                                        const double* lam, const double* sX, const double* gR,
                                        double* gS, double* gU, bool more, double rho, double rq,
                                        double sq, double aq, double den, double beta,
                                        double rinv) {
  // reciprocals instead of FP64 divisions in the per-row updates (a division is a
  // ~40-instruction Newton sequence; <= 1 ulp different per operation)
  const double iden = 1.0 / den, irq = 1.0 / rq;
  // vv[j] = v_j = p~_j - lam_j rinv, constant over the QP iterations of a launch
  // (formed in the FIRST pass); rhs_p,j = sq p_j + rho v_j + rq z_j - y_j is
  // recomputed from the row's current (p, z, y) instead of being stored.
  const int nx = v.d.nx, nu = v.d.nu;
  const int4* __restrict__ rows = v.rowpk + bg;
  const double* __restrict__ gval = v.gval + bg * kRowNZ;
  for (int j0 = tid; j0 < ng; j0 += U * nt) {
    int4 rc[U];
    double2 g01[U];
    double vj[U], pj[U], zlj[U], ylj[U], g0j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * nt;
      if (j < ng) {
        rc[u] = rows[j];
        g01[u] = *reinterpret_cast<const double2*>(gval + (int64_t)j * kRowNZ);
        pj[u] = p[j]; zlj[u] = zl[j]; ylj[u] = yl[j];
        if (FIRST) vj[u] = pt[j] - lam[j] * rinv;
        else { vj[u] = vv[j]; g0j[u] = g0[j]; }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * nt;
      if (j >= ng) continue;
      const int k = rc[u].x, kind = rc[u].y & 0xff, nz = (rc[u].y >> 8) & 0xff;
      const double* gj = grad + (int64_t)j * nx;
      double pn = pj[u], zn = zlj[u], yn = ylj[u];
      if (FIRST) vv[j] = vj[u];
      if (!FIRST) {
        const double* x = (kind == 0) ? sX + (int64_t)k * nx : gR + (int64_t)k * nu;
        double bd = 0.0;
        if (nz <= kRowNZ) {
          if (nz > 0) bd += g01[u].x * x[rec_idx(rc[u], 0)];
          if (nz > 1) bd += g01[u].y * x[rec_idx(rc[u], 1)];
          for (int q = 2; q < nz; ++q) bd += gval[(int64_t)j * kRowNZ + q] * x[rec_idx(rc[u], q)];
        } else {
          const int n = (kind == 0) ? nx : nu;
          for (int i = 0; i < n; ++i) bd += gj[i] * x[i];
        }
        const double r0 = sq * pj[u] + rho * vj[u] + rq * zlj[u] - ylj[u];
        const double ptl = (r0 - rq * bd) * iden;
        pn = aq * ptl + (1.0 - aq) * pj[u];
        const double zh = aq * (bd + ptl) + (1.0 - aq) * zlj[u];
        zn = nan_min(zh + ylj[u] * irq, -g0j[u]);
        yn = ylj[u] + rq * (zh - zn);
        p[j] = pn; zl[j] = zn; yl[j] = yn;
      }
      if (FIRST || more) {
        const double r = sq * pn + rho * vj[u] + rq * zn - yn;
        const double w = rq * zn - yn - beta * r;
        double* dst = (kind == 0) ? gS + (int64_t)k * nx : gU + (int64_t)k * nu;
        if (nz <= kRowNZ) {
          if (nz > 0) atomicAdd(dst + rec_idx(rc[u], 0), w * g01[u].x);
          if (nz > 1) atomicAdd(dst + rec_idx(rc[u], 1), w * g01[u].y);
          for (int q = 2; q < nz; ++q)
            atomicAdd(dst + rec_idx(rc[u], q), w * gval[(int64_t)j * kRowNZ + q]);
        } else {
          const int n = (kind == 0) ? nx : nu;
          for (int i = 0; i < n; ++i) atomicAdd(dst + i, w * gj[i]);
        }
      }
    }
  }
}

// Spin until a shared-memory epoch flag reaches `ep` (producer: data, membar.cta,
// flag), then order the following reads after it.
__device__ __forceinline__ void qp_spin(volatile int16_t* f, int16_t ep) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared((const void*)f);
  for (;;) {
    unsigned short x;
    asm volatile("ld.acquire.cta.shared.b16 %0, [%1];" : "=h"(x) : "r"(a) : "memory");
    if ((int16_t)x >= ep) break;
    __nanosleep(20);
  }
}
// Publish an epoch flag: release store (orders this thread's earlier accesses,
// incl. the data the flag announces, before it at CTA scope).
__device__ __forceinline__ void qp_publish(volatile int16_t* f, int16_t ep) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared((const void*)f);
  asm volatile("st.release.cta.shared.b16 [%0], %1;" ::"r"(a), "h"((unsigned short)ep) : "memory");
}

// Rows of one QP iteration in knot order (v.qrow: for p = 1..T the state rows at
// knot p, then the control rows at step p-1), each processed once dx_k (fx[k],
// state rows) / du~_k (fu[k], control rows) is published; same arithmetic as
// qp_rows<false>.
template <int U>
__device__ __forceinline__ void qp_rows_pipe(const Dev& v, int64_t bg, int ng, int tid, int nt,
                                             const double* __restrict__ grad,
                                             const double* __restrict__ g0, double* p, double* zl,
                                             double* yl, double* vv, const double* sX,
                                             const double* gR, double* gS, double* gU, bool more,
                                             volatile int16_t* fx, volatile int16_t* fu, int16_t ep,
                                             double rho, double rq,
                                             double sq, double aq, double den, double beta) {
  // reciprocals instead of FP64 divisions in the per-row updates (a division is a
  // ~40-instruction Newton sequence; <= 1 ulp different per operation)
  const double iden = 1.0 / den, irq = 1.0 / rq;
  const int nx = v.d.nx, nu = v.d.nu;
  const int4* __restrict__ rows = v.rowpk + bg;
  const double* __restrict__ gval = v.gval + bg * kRowNZ;
  for (int q0 = tid; q0 < ng; q0 += U * nt) {
    int4 rc[U];
    double2 g01[U];
    int jj[U];
    double vj[U], pj[U], zlj[U], ylj[U], g0j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = q0 + u * nt;
      if (q < ng) {
        const int j = v.qrow[q];
        jj[u] = j;
        rc[u] = rows[j];
        g01[u] = *reinterpret_cast<const double2*>(gval + (int64_t)j * kRowNZ);
        pj[u] = p[j]; zlj[u] = zl[j]; ylj[u] = yl[j]; vj[u] = vv[j]; g0j[u] = g0[j];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = q0 + u * nt;
      if (q >= ng) continue;
      const int j = jj[u];
      const int k = rc[u].x, kind = rc[u].y & 0xff, nz = (rc[u].y >> 8) & 0xff;
      qp_spin(kind == 0 ? &fx[k] : &fu[k], ep);
      const double* gj = grad + (int64_t)j * nx;
      double bd = 0.0;
      if (kind == 0) {
        const double* x = sX + (int64_t)k * nx;
        if (nz <= kRowNZ) {
          if (nz > 0) bd += g01[u].x * x[rec_idx(rc[u], 0)];
          if (nz > 1) bd += g01[u].y * x[rec_idx(rc[u], 1)];
          for (int s = 2; s < nz; ++s) bd += gval[(int64_t)j * kRowNZ + s] * x[rec_idx(rc[u], s)];
        } else {
          for (int i = 0; i < nx; ++i) bd += gj[i] * x[i];
        }
      } else {
        const double* x = gR + (int64_t)k * nu;
        if (nz <= kRowNZ) {
          if (nz > 0) bd += g01[u].x * __ldcg(x + rec_idx(rc[u], 0));
          if (nz > 1) bd += g01[u].y * __ldcg(x + rec_idx(rc[u], 1));
          for (int s = 2; s < nz; ++s) bd += gval[(int64_t)j * kRowNZ + s] * __ldcg(x + rec_idx(rc[u], s));
        } else {
          for (int i = 0; i < nu; ++i) bd += gj[i] * __ldcg(x + i);
        }
      }
      const double r0 = sq * pj[u] + rho * vj[u] + rq * zlj[u] - ylj[u];
      const double ptl = (r0 - rq * bd) * iden;
      const double pn = aq * ptl + (1.0 - aq) * pj[u];
      const double zh = aq * (bd + ptl) + (1.0 - aq) * zlj[u];
      const double zn = nan_min(zh + ylj[u] * irq, -g0j[u]);
      const double yn = ylj[u] + rq * (zh - zn);
      p[j] = pn; zl[j] = zn; yl[j] = yn;
      if (more) {
        const double r = sq * pn + rho * vj[u] + rq * zn - yn;
        const double w = rq * zn - yn - beta * r;
        double* dst = (kind == 0) ? gS + (int64_t)k * nx : gU + (int64_t)k * nu;
        if (nz <= kRowNZ) {
          if (nz > 0) atomicAdd(dst + rec_idx(rc[u], 0), w * g01[u].x);
          if (nz > 1) atomicAdd(dst + rec_idx(rc[u], 1), w * g01[u].y);
          for (int s = 2; s < nz; ++s)
            atomicAdd(dst + rec_idx(rc[u], s), w * gval[(int64_t)j * kRowNZ + s]);
        } else {
          const int n = (kind == 0) ? nx : nu;
          for (int i = 0; i < n; ++i) atomicAdd(dst + i, w * gj[i]);
        }
      }
    }
  }
}

// Debug timing of one QP CTA (instance 0, first two QP iterations): clock64 at
// every phase boundary, read with nrto_debug_qp_clocks (not part of nrto.h).
__device__ long long g_qp_clk[64];
#define QP_CLK(ph) \
  do { if (b == 0 && tid == 0 && it_dbg < 2) g_qp_clk[it_dbg * 32 + (ph)] = clock64(); } while (0)

// sum_{q < n} fa(q) fb(q) + acc.  NM > 0 (n <= NM): loads issued
// 8 at a time (predicated) so dependent latency is paid once per batch, not per
// term; NM = 0: plain loop.
template <int NM, class FA, class FB>
__device__ __forceinline__ double dotn(int n, FA fa, FB fb, double acc) {
  if constexpr (NM > 0) {
    double c[4] = {acc, 0.0, 0.0, 0.0};
#pragma unroll
    for (int q0 = 0; q0 < NM; q0 += 8) {
      double av[8], bv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = q0 + u;
        const bool ok = q < NM && q < n;
        av[u] = ok ? fa(q) : 0.0;
        bv[u] = ok ? fb(q) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) c[u & 3] = fma(av[u], bv[u], c[u & 3]);
    }
    return (c[0] + c[1]) + (c[2] + c[3]);
  } else {
    for (int q = 0; q < n; ++q) acc += fa(q) * fb(q);
    return acc;
  }
}

// mbarrier / bulk-copy helpers for the recurrence ring (TMA, SASS UBLKCP)
__device__ __forceinline__ void qp_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void qp_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void qp_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "QPW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra QPW_%=;\n"
      "}\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

// NXM, NUM > 0: the exact n_x, n_u, fixed at compile time (shape-specialised
// instances for the benchmark shapes: every small loop fully unrolled, loads
// issued together); 0: runtime sizes.
template <int NXM, int NUM, bool PIPE>
__device__ __forceinline__ void qp_instance(const Dev& v, int engine, int l, int b, double* sm,
                                            double* red) {
  const Dims d = v.d;
  const int nx = NXM > 0 ? NXM : d.nx, nu = NUM > 0 ? NUM : d.nu, T = d.T, ng = d.ng;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (!v.active[b]) return;
  const EngineFactors& F = engine == NRTO_FULLADMM ? v.fa : v.dr;
  const double rho = engine == NRTO_FULLADMM ? v.prm.rho : v.prm.rho_admm;
  const double rq = v.prm.rho_qp, sq = v.prm.sigma_qp, aq = v.prm.alpha_qp;
  const double den = rho + sq + rq, beta = rq / den, irq = 1.0 / rq;
  const int64_t bg = (int64_t)b * ng;
  const double* __restrict__ grad = v.grad + bg * nx;
  const double* __restrict__ g0 = v.g0 + bg;
  double* p = v.p + bg; double* zl = v.zl + bg; double* yl = v.yl + bg;
  double* rp = v.rp + bg;
  const double* pt = v.pt + bg; double* lam = v.lamp + bg;
  double* zb = v.zb + (int64_t)b * (T + 1) * nx; double* yb = v.yb + (int64_t)b * (T + 1) * nx;
  double* du = v.du + (int64_t)b * T * nu;
  double* gK = v.kff + (int64_t)b * T * nu;           // kff_k
  double* gR = v.ru + (int64_t)b * T * nu;            // r_u,k, then du~_k
  double* gS = v.rx + (int64_t)b * (T + 1) * nx;      // S_k = sum_{state j@k} w_j grad_j (atomic)
  double* gU = v.dut + (int64_t)b * T * nu;           // U_k = sum_{ctrl j@k} w_j h'_j   (atomic)
  const double* __restrict__ cu2 = v.cu2 + (int64_t)b * T * nu;
  const double* __restrict__ Bm = v.Bm + (int64_t)b * T * nx * nu;
  const double* __restrict__ Kf = F.Kf + (int64_t)b * T * nu * nx;
  const double* __restrict__ AclG = F.Acl + (int64_t)b * T * nx * nx;
  const double* __restrict__ Hi = F.Hinv + (int64_t)b * T * nu * nu;
  const double* __restrict__ HB = F.HB + (int64_t)b * T * nu * nx;
  const double rtr = v.rtrust[b];
  const double rinv = (engine == NRTO_FULLADMM) ? 1.0 : 1.0 / rho;
  double* sS = sm;                                    // [(T+1) nx]
  double* ring = sS + (T + 1) * nx;                   // [kQPRing][nx nx]
  uint64_t* qbar = reinterpret_cast<uint64_t*>(ring + kQPRing * nx * nx);   // [kQPRing]
  int16_t* flg = reinterpret_cast<int16_t*>(qbar + kQPRing);                  // [6][T+1] (pipelined)
  const int nn = nx * nx;
  const int nits = v.prm.qp_iters;
  int it_dbg = 0;

  if (NXM > 0 && tid == 0) {
    for (int q = 0; q < kQPRing; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&qbar[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int r = tid; r < (T + 1) * nx; r += nt) gS[r] = 0.0;
  for (int r = tid; r < T * nu; r += nt) gU[r] = 0.0;
  if (NXM > 0)
    for (int r = tid; r < 6 * (T + 1); r += nt) flg[r] = 0;
  __syncthreads();
  QP_CLK(0);
  if (nits > 0) {                                     // rhs / w / scatter of iteration 0
    qp_rows<true, kRowBatch>(v, bg, ng, tid, nt, grad, g0, p, zl, yl, rp, pt, lam, sS, gR, gS, gU, true,
                  rho, rq, sq, aq, den, beta, rinv);
    __syncthreads();
    QP_CLK(1);
  }
  if constexpr (NXM > 0 && PIPE) {
    // ---- pipelined QP iteration (warp-specialised): warp 0 runs the two
    // Riccati recurrences; warps 1.. run every k-parallel phase BEHIND it, per knot,
    // synchronised by per-knot epoch flags in shared memory (membar.cta + volatile):
    //   fa[k]: a_k, r_u,k ready      (helpers -> warp 0, backward sweep)
    //   fs[k]: s_k ready             (warp 0 -> helpers: kff_k, e_k)
    //   fe[k]: kff_k, e_k ready      (helpers -> warp 0, forward sweep)
    //   fx[p]: dx_p, du~_{p-1} ready (warp 0 -> helpers: rows in knot order)
    // so only one block barrier per QP iteration remains (before the ball).
    const int warp = tid >> 5, lane = tid & 31;
    const int nhw = (nt >> 5) - 1;
    volatile int16_t* fa = flg;
    volatile int16_t* fs = fa + (T + 1);
    volatile int16_t* fe = fs + (T + 1);
    volatile int16_t* fx = fe + (T + 1);
    volatile int16_t* fu = fx + (T + 1);
    volatile int16_t* fk = fu + (T + 1);
    for (int it = 0; it < nits; ++it) {
      it_dbg = it;
      const int16_t ep = (int16_t)(it + 1);
      if (warp == 0) {
        // The two recurrences read Acl_k^T (backward) and Acl_k (forward) as ONE stream of
        // chunks of QP_CHUNK consecutive steps (one bulk copy each, kQPRing / QP_CHUNK
        // slots), continued across the QP iterations of the launch, so the forward
        // sweep's first chunks arrive during the backward tail.
        constexpr int C = QP_CHUNK;
        constexpr int S = kQPRing / C;
        const int NC = (T + C - 1) / C;
        const int ptot = nits * 2 * NC;
        const double* AT = F.AclT + (int64_t)b * T * nn;
        const double* AG = F.Acl + (int64_t)b * T * nn;
        auto chunk = [&](int p, int& lo, int& hi) {
          const int g = p % (2 * NC);
          if (g < NC) { hi = T - 1 - g * C; lo = max(0, hi - C + 1); return true; }
          lo = (g - NC) * C; hi = min(T, lo + C) - 1; return false;
        };
        auto issue = [&](int p) {
          if (lane != 0 || p >= ptot) return;
          int lo, hi;
          const bool bw = chunk(p, lo, hi);
          const int sl = p % S;
          const uint32_t bytes = (uint32_t)((hi - lo + 1) * nn * 8);
          qp_expect_tx(&qbar[sl], bytes);
          qp_bulk(ring + sl * C * nn, (bw ? AT : AG) + (int64_t)lo * nn, bytes, &qbar[sl]);
        };
        if (it == 0)
          for (int p = 0; p < S; ++p) issue(p);
        const int pb = it * 2 * NC;
        // backward recurrence s_k = a_k + Acl_k^T s_{k+1}
        const int ic = lane < nx ? lane : 0;
        qp_spin(&fa[T], ep);
        const double* base = ring;
        int lo = 0, hi = -1;
        long long tb0 = 0, tb1 = 0, tb2 = 0;
        for (int k = T - 1; k >= 0; --k) {
          const int c = (T - 1 - k) / C, p = pb + c;
          const long long q0 = clock64();
          if (k > hi || k < lo) {
            chunk(p, lo, hi);
            qp_wait(&qbar[p % S], (uint32_t)(p / S) & 1u);
            base = ring + (p % S) * C * nn;
          }
          const long long q1 = clock64();
          tb0 += q1 - q0;
          qp_spin(&fa[k], ep);
          const long long q2 = clock64();
          tb1 += q2 - q1;
          const double* Ar = base + (k - lo) * nn + ic * nx;
          const double* sn = sS + (k + 1) * nx;
          double c0 = sS[k * nx + ic], c1 = 0.0;
#pragma unroll
          for (int r = 0; r < NXM; r += 2)
            if (r < nx) {
              const double2 a = *reinterpret_cast<const double2*>(Ar + r);
              const double2 x2 = *reinterpret_cast<const double2*>(sn + r);
              c0 = fma(a.x, x2.x, c0);
              c1 = fma(a.y, x2.y, c1);
            }
          __syncwarp();
          if (lane < nx) sS[k * nx + lane] = c0 + c1;
          __syncwarp();
          if (lane == 0) qp_publish(&fs[k], ep);
          if (k == lo) issue(p + S);
          tb2 += clock64() - q2;
        }
        if (b == 0 && tid == 0 && it_dbg < 2) {
          g_qp_clk[it_dbg * 32 + 12] = tb0; g_qp_clk[it_dbg * 32 + 13] = tb1; g_qp_clk[it_dbg * 32 + 14] = tb2;
        }
        QP_CLK(4);
        // forward recurrence dx_{k+1} = Acl_k dx_k + e_k, e_k in shared slot k+1 (overwritten
        // by dx_{k+1})
        for (int k = lane; k < T; k += 32) qp_spin(&fe[k], ep);   // every e_k (e_0 comes last)
        if (lane < nx) sS[lane] = 0.0;                     // dx_0 = 0 (s_0 is not read by anyone)
        __syncwarp();
        lo = 0; hi = -1;
        long long tq0 = 0, tq1 = 0, tq2 = 0;
        for (int k = 0; k < T; ++k) {
          const int c = k / C, p = pb + NC + c;
          const long long q1 = clock64();
          if (k > hi || k < lo) {
            chunk(p, lo, hi);
            qp_wait(&qbar[p % S], (uint32_t)(p / S) & 1u);
            base = ring + (p % S) * C * nn;
          }
          const long long q2 = clock64();
          tq1 += q2 - q1;
          const double* Ar = base + (k - lo) * nn + ic * nx;
          const double* xk = sS + k * nx;
          double c0 = sS[(k + 1) * nx + ic], c1 = 0.0;
#pragma unroll
          for (int r = 0; r < NXM; r += 2)
            if (r < nx) {
              const double2 a = *reinterpret_cast<const double2*>(Ar + r);
              const double2 x2 = *reinterpret_cast<const double2*>(xk + r);
              c0 = fma(a.x, x2.x, c0);
              c1 = fma(a.y, x2.y, c1);
            }
          __syncwarp();
          if (lane < nx) sS[(k + 1) * nx + lane] = c0 + c1;
          __syncwarp();
          if (lane == 0) qp_publish(&fx[k + 1], ep);
          if (k == hi) issue(p + S);
          tq2 += clock64() - q2;
        }
        if (b == 0 && tid == 0 && it_dbg < 2) {
          g_qp_clk[it_dbg * 32 + 16] = tq0; g_qp_clk[it_dbg * 32 + 17] = tq1; g_qp_clk[it_dbg * 32 + 18] = tq2;
        }
        QP_CLK(7);
      } else {
        // helpers, knot k by warp (k mod nhw): a_k, r_u,k (descending, ahead of warp 0)
        for (int k = T - (warp - 1); k >= 0; k -= nhw) {
          double ru = 0.0;                               // r_u,k (recomputed by the kff helper)
          if (k < T && lane < nu) {
            const int r = k * nu + lane;
            ru = sq * du[r] + __ldcg(gU + r) + cu2[r];   // cu2 = -2 R_u u_hat (setup)
          }
          double acc = 0.0;
          if (lane < nx && k > 0) {
            const int r = k * nx + lane;
            acc = __ldcg(gS + r) + rq * zb[r] - yb[r];
          }
          if (k < T) {
            const double* Kk = Kf + (int64_t)k * nu * nx + (lane < nx ? lane : 0);
#pragma unroll
            for (int m = 0; m < (NUM > 0 ? NUM : 8); ++m) {
              const double rm = __shfl_sync(0xffffffffu, ru, m);
              if (m < nu && lane < nx) acc -= Kk[m * nx] * rm;
            }
          }
          if (lane < nx) sS[k * nx + lane] = acc;       // a_k (k < T), s_T
          __syncwarp();
          if (lane == 0) qp_publish(&fa[k], ep);
        }
        // kff_k = H^-1 r_u,k + H^-1 B_k^T s_{k+1}, e_k = B_k kff_k (descending, behind warp 0).
        // Lane (m, part) = (lane / 4, lane % 4) sums part of the NUM + NXM terms of kff[m];
        // the constants of a warp's next knot are loaded while it waits for the current one.
        {
          constexpr int NT = NUM + NXM;                  // terms per kff row
          constexpr int NP = (NT + 3) / 4;               // terms per lane
          const int m = lane >> 2, part = lane & 3;
          const bool mok = m < nu;
          double hv[NP], bv[NUM], pr[3];
          auto load = [&](int k) {
#pragma unroll
            for (int u = 0; u < NP; ++u) {
              const int t = part * NP + u;
              hv[u] = 0.0;
              if (mok && t < NT && k >= 0)
                hv[u] = (t < NUM) ? Hi[(int64_t)k * nu * nu + m * nu + t]
                                  : HB[(int64_t)k * nu * nx + m * nx + (t - NUM)];
            }
#pragma unroll
            for (int q = 0; q < NUM; ++q)
              bv[q] = (lane < nx && k >= 0) ? Bm[(int64_t)k * nx * nu + lane * nu + q] : 0.0;
            if (lane < nu && k >= 0) {
              const int r = k * nu + lane;
              pr[0] = du[r]; pr[1] = __ldcg(gU + r); pr[2] = cu2[r];
            }
          };
          int k = T - 1 - (warp - 1);
          load(k);
          for (; k >= 0; k -= nhw) {
            double cur_h[NP], cur_b[NUM], cur_p[3];
#pragma unroll
            for (int u = 0; u < NP; ++u) cur_h[u] = hv[u];
#pragma unroll
            for (int q = 0; q < NUM; ++q) cur_b[q] = bv[q];
            cur_p[0] = pr[0]; cur_p[1] = pr[1]; cur_p[2] = pr[2];
            load(k - nhw);                               // next knot of this warp
            const double ru = (lane < nu) ? sq * cur_p[0] + cur_p[1] + cur_p[2] : 0.0;
            qp_spin(k + 1 == T ? &fa[T] : &fs[k + 1], ep);
            const double* sk = sS + (k + 1) * nx;
            double acc = 0.0;
#pragma unroll
            for (int u = 0; u < NP; ++u) {
              const int t = part * NP + u;
              // every lane executes the same shuffle (uniform call site, full mask)
              const double xr = __shfl_sync(0xffffffffu, ru, (t < NUM) ? t : 0);
              if (t < NT) acc = fma(cur_h[u], (t < NUM) ? xr : sk[t - NUM], acc);
            }
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);   // kff[m] in lanes 4m..4m+3
            double e = 0.0;
#pragma unroll
            for (int q = 0; q < NUM; ++q) {
              const double kq = __shfl_sync(0xffffffffu, acc, 4 * q);
              e = fma(cur_b[q], kq, e);
            }
            // e_k goes to shared slot k+1 (s_{k+1} is dead once warp 0 has published s_k)
            qp_spin(&fs[k], ep);
            if (lane < nx) sS[(k + 1) * nx + lane] = e;
            __syncwarp();
            if (lane == 0) qp_publish(&fe[k], ep);
            // kff_k (read by warp 1 in the forward phase) and the cleared scatter targets
            // of the next QP iteration go to global memory; one fence per warp below
            if (mok && part == 0) gK[k * nu + m] = acc;
            if (lane < nu) gU[k * nu + lane] = 0.0;
            if (lane < nx) {
              gS[k * nx + lane] = 0.0;
              if (k == T - 1) gS[T * nx + lane] = 0.0;
            }
          }
          __threadfence_block();
          __syncwarp();
          if (lane == 0)
            for (int kk = T - 1 - (warp - 1); kk >= 0; kk -= nhw) qp_publish(&fk[kk], ep);
        }
        if (warp == 1) {
          // du~_k = kff_k - Kf_k dx_k and du_k (relaxed), 4 knots per publication (fu)
          const int c = lane / nu, m = lane - c * nu;
          double nbp = 0.0;
          for (int k0 = 0; k0 < T; k0 += 4) {
            const int k = k0 + c;
            qp_spin(&fx[min(k0 + 3, T - 1)], ep);
            if (c < 4 && k < T) qp_spin(&fk[k], ep);
            if (c < 4 && k < T) {
              const double* Kk = Kf + (int64_t)k * nu * nx + m * nx;
              const double* xk = sS + k * nx;
              const double dd = __ldcg(gK + k * nu + m) -
                                dotn<NXM>(nx, [&](int q) { return Kk[q]; }, [&](int q) { return xk[q]; }, 0.0);
              gR[k * nu + m] = dd;
              du[k * nu + m] = aq * dd + (1.0 - aq) * du[k * nu + m];
            }
            __threadfence_block();                       // global du~ before fu
            __syncwarp();
            if (lane < 4 && k0 + lane < T) qp_publish(&fu[k0 + lane], ep);
            // trust-region ball partial sum of the knots whose dx is final (zb, yb then sit
            // in this SM's L1 for the update after the barrier)
            const int r1 = (k0 + 4 >= T ? T + 1 : k0 + 4) * nx;
            if (k0 + 4 >= T) qp_spin(&fx[T], ep);
            for (int r = k0 * nx + lane; r < r1; r += 32) {
              const double zh = aq * sS[r] + (1.0 - aq) * zb[r];
              const double w = zh + yb[r] * irq;
              nbp += w * w;
            }
          }
          nbp = warp_sum(nbp);
          if (lane == 0) red[31] = nbp;
        } else {
          // rows in knot order, each as soon as dx_k (fx) / du~_k (fu) is published
          const bool more = it + 1 < nits;
          qp_rows_pipe<kRowBatch>(v, bg, ng, tid - 64, nt - 64, grad, g0, p, zl, yl, rp, sS, gR, gS, gU,
                                  more, fx, fu, ep, rho, rq, sq, aq, den, beta);
        }
      }
      __syncthreads();
      QP_CLK(9);
      {                                                 // trust-region ball (norm by warp 1)
        const double nb = sqrt(red[31]);
        const double scl = (nb > rtr) ? rtr / nb : 1.0;
        for (int r = tid; r < (T + 1) * nx; r += nt) {
          const double zh = aq * sS[r] + (1.0 - aq) * zb[r];
          const double zn = scl * (zh + yb[r] * irq);
          yb[r] += rq * (zh - zn);
          zb[r] = zn;
        }
      }
      __syncthreads();
      QP_CLK(10);
    }
  } else {
  for (int it = 0; it < nits; ++it) {
    it_dbg = it;
    for (int r = tid; r < T * nu; r += nt) {          // r_u (consumes and clears U)
      const double acc = sq * du[r] + gU[r] + cu2[r];  // cu2 = -2 R_u u_hat (setup)
      gU[r] = 0.0;
      gR[r] = acc;
    }
    __syncthreads();
    QP_CLK(2);
    for (int r = tid; r < (T + 1) * nx; r += nt) {    // r_x and a_k (consumes and clears S)
      const int k = r / nx, i = r % nx;
      double acc = (k > 0) ? gS[r] + rq * zb[r] - yb[r] : 0.0;
      gS[r] = 0.0;
      if (k < T) {
        const double* Kk = Kf + (int64_t)k * nu * nx + i;
        const double* rk = gR + k * nu;
        acc -= dotn<NUM>(nu, [&](int m) { return Kk[m * nx]; }, [&](int m) { return rk[m]; }, 0.0);
      }
      sS[r] = acc;        // a_k (k < T), s_T; the recurrence overwrites a_k by s_k
    }
    __syncthreads();
    QP_CLK(3);
    if (tid < 32) {                                   // backward recurrence
      if constexpr (NXM > 0) {
        // s_k[i] = a_k[i] + <column i of Acl_k, s_{k+1}>: Acl_k arrives by one bulk copy
        // per step into a kQPRing-slot ring (mbarrier; the same array as the forward
        // sweep, so the QP streams Acl once, not Acl and its transpose), column reads
        // conflict-free across lanes, s_{k+1} by broadcast LDS.128
        const double* AT = F.Acl + (int64_t)b * T * nn;
        // ring position = running copy count n (2T per QP iteration): slot n % R,
        // parity (n / R) & 1 -- computed, not carried, to keep it out of local memory
        const int n0 = it * 2 * T;
        if (tid == 0)
          for (int pf = 0; pf < kQPRing && pf < T; ++pf) {
            const int sl = (n0 + pf) & (kQPRing - 1);
            qp_expect_tx(&qbar[sl], nn * 8);
            qp_bulk(ring + sl * nn, AT + (int64_t)(T - 1 - pf) * nn, nn * 8, &qbar[sl]);
          }
        const int ic = tid < nx ? tid : 0;
        for (int k = T - 1; k >= 0; --k) {
          const int n = n0 + (T - 1 - k), rslot = n & (kQPRing - 1);
          qp_wait(&qbar[rslot], (uint32_t)(n / kQPRing) & 1u);
          const double* Ac = ring + rslot * nn + ic;
          const double* sn = sS + (k + 1) * nx;
          double c0 = sS[k * nx + ic], c1 = 0.0;
#pragma unroll
          for (int r = 0; r < NXM; r += 2)
            if (r < nx) {
              const double2 x2 = *reinterpret_cast<const double2*>(sn + r);
              c0 = fma(Ac[r * nx], x2.x, c0);
              c1 = fma(Ac[(r + 1) * nx], x2.y, c1);
            }
          __syncwarp();
          if (tid < nx) sS[k * nx + tid] = c0 + c1;
          __syncwarp();
          const int kn = k - kQPRing;
          if (tid == 0 && kn >= 0) {
            qp_expect_tx(&qbar[rslot], nn * 8);
            qp_bulk(ring + rslot * nn, AT + (int64_t)kn * nn, nn * 8, &qbar[rslot]);
          }
        }
      } else {
      for (int pf = 0; pf < kQPRing; ++pf) {
        const int k = T - 1 - pf;
        if (k >= 0) for (int e = tid; e < nn; e += 32) cpa8(ring + pf * nn + e, AclG + (int64_t)k * nn + e);
        cpa_commit();
      }
      double s = (tid < nx) ? sS[T * nx + tid] : 0.0;
      const int ic = tid < nx ? tid : 0;
      for (int k = T - 1, slot = 0; k >= 0; --k, slot = (slot + 1) % kQPRing) {
        cpa_wait<kQPRing - 1>();
        __syncwarp();
        const double* Ak = ring + slot * nn + ic;
        const double* sn = sS + (k + 1) * nx;       // s_{k+1} (broadcast reads)
        s = dotn<NXM>(nx, [&](int r) { return Ak[r * nx]; }, [&](int r) { return sn[r]; },
                      sS[k * nx + ic]);
        if (tid < nx) sS[k * nx + tid] = s;
        __syncwarp();
        const int kn = k - kQPRing;
        if (kn >= 0) for (int e = tid; e < nn; e += 32) cpa8(ring + slot * nn + e, AclG + (int64_t)kn * nn + e);
        cpa_commit();
      }
      cpa_wait<0>();
      }
    }
    __syncthreads();
    QP_CLK(4);
    for (int r = tid; r < T * nu; r += nt) {          // kff_k
      const int k = r / nu, m = r % nu;
      const double* H = Hi + (int64_t)k * nu * nu + m * nu;
      const double* hb = HB + (int64_t)k * nu * nx + m * nx;
      const double* rk = gR + k * nu;
      const double* sk = sS + (k + 1) * nx;
      double acc = dotn<NUM>(nu, [&](int q) { return H[q]; }, [&](int q) { return rk[q]; }, 0.0);
      acc = dotn<NXM>(nx, [&](int q) { return hb[q]; }, [&](int q) { return sk[q]; }, acc);
      gK[r] = acc;
    }
    __syncthreads();
    QP_CLK(5);
    for (int r = tid; r < T * nx; r += nt) {          // e_k = B_k kff_k
      const int k = r / nx, i = r % nx;
      const double* Bk = Bm + (int64_t)k * nx * nu + i * nu;
      const double* kk = gK + k * nu;
      const double acc = dotn<NUM>(nu, [&](int m) { return Bk[m]; }, [&](int m) { return kk[m]; }, 0.0);
      sS[r + nx] = acc;   // e_k at slot k+1; the forward recurrence overwrites it by dx_{k+1}
    }
    __syncthreads();
    QP_CLK(6);
    if (tid < 32) {                                   // forward recurrence
      if constexpr (NXM > 0) {
        // dx_{k+1}[i] = e_k[i] + <Acl_k row i, dx_k>
        const double* AG = F.Acl + (int64_t)b * T * nn;
        const int n0 = it * 2 * T + T;
        if (tid == 0)
          for (int pf = 0; pf < kQPRing && pf < T; ++pf) {
            const int sl = (n0 + pf) & (kQPRing - 1);
            qp_expect_tx(&qbar[sl], nn * 8);
            qp_bulk(ring + sl * nn, AG + (int64_t)pf * nn, nn * 8, &qbar[sl]);
          }
        const int ic = tid < nx ? tid : 0;
        if (tid < nx) sS[tid] = 0.0;
        __syncwarp();
        for (int k = 0; k < T; ++k) {
          const int n = n0 + k, rslot = n & (kQPRing - 1);
          qp_wait(&qbar[rslot], (uint32_t)(n / kQPRing) & 1u);
          const double* Ar = ring + rslot * nn + ic * nx;
          const double* xk = sS + k * nx;
          double c0 = sS[(k + 1) * nx + ic], c1 = 0.0;
#pragma unroll
          for (int r = 0; r < NXM; r += 2)
            if (r < nx) {
              const double2 a = *reinterpret_cast<const double2*>(Ar + r);
              const double2 x2 = *reinterpret_cast<const double2*>(xk + r);
              c0 = fma(a.x, x2.x, c0);
              c1 = fma(a.y, x2.y, c1);
            }
          __syncwarp();
          if (tid < nx) sS[(k + 1) * nx + tid] = c0 + c1;
          __syncwarp();
          const int kn = k + kQPRing;
          if (tid == 0 && kn < T) {
            qp_expect_tx(&qbar[rslot], nn * 8);
            qp_bulk(ring + rslot * nn, AG + (int64_t)kn * nn, nn * 8, &qbar[rslot]);
          }
        }
      } else {
      for (int pf = 0; pf < kQPRing; ++pf) {
        if (pf < T) for (int e = tid; e < nn; e += 32) cpa8(ring + pf * nn + e, AclG + (int64_t)pf * nn + e);
        cpa_commit();
      }
      double x = 0.0;
      const int ic = tid < nx ? tid : 0;
      if (tid < nx) sS[tid] = 0.0;
      for (int k = 0, slot = 0; k < T; ++k, slot = (slot + 1) % kQPRing) {
        cpa_wait<kQPRing - 1>();
        __syncwarp();
        const double* Ak = ring + slot * nn + ic * nx;
        const double* xk = sS + k * nx;             // dx_k (broadcast reads)
        x = dotn<NXM>(nx, [&](int r) { return Ak[r]; }, [&](int r) { return xk[r]; },
                      sS[(k + 1) * nx + ic]);
        if (tid < nx) sS[(k + 1) * nx + tid] = x;
        __syncwarp();
        const int kn = k + kQPRing;
        if (kn < T) for (int e = tid; e < nn; e += 32) cpa8(ring + slot * nn + e, AclG + (int64_t)kn * nn + e);
        cpa_commit();
      }
      cpa_wait<0>();
      }
    }
    __syncthreads();
    QP_CLK(7);
    for (int r = tid; r < T * nu; r += nt) {          // du~_k
      const int k = r / nu, m = r % nu;
      const double* Kk = Kf + (int64_t)k * nu * nx + m * nx;
      const double* xk = sS + k * nx;
      gR[r] = gK[r] - dotn<NXM>(nx, [&](int q) { return Kk[q]; }, [&](int q) { return xk[q]; }, 0.0);
    }
    __syncthreads();
    QP_CLK(8);
    const bool more = it + 1 < nits;
    qp_rows<false, kRowBatch>(v, bg, ng, tid, nt, grad, g0, p, zl, yl, rp, pt, lam, sS, gR, gS, gU, more,
                   rho, rq, sq, aq, den, beta, rinv);
    for (int r = tid; r < T * nu; r += nt) du[r] = aq * gR[r] + (1.0 - aq) * du[r];
    __syncthreads();
    QP_CLK(9);
    double nb = 0.0;                                  // trust-region ball
    for (int r = tid; r < (T + 1) * nx; r += nt) {
      const double zh = aq * sS[r] + (1.0 - aq) * zb[r];
      sS[r] = zh;
      const double w = zh + yb[r] * irq;
      nb += w * w;
    }
    nb = sqrt(block_sum(nb, red));
    const double scl = (nb > rtr) ? rtr / nb : 1.0;
    for (int r = tid; r < (T + 1) * nx; r += nt) {
      const double zh = sS[r];
      const double zn = scl * (zh + yb[r] * irq);
      yb[r] += rq * (zh - zn);
      zb[r] = zn;
    }
    __syncthreads();
    QP_CLK(10);
  }
  }
  double ap = 0.0, ad = 0.0;
  double* tin = v.tin + bg;
  double* ptp = v.ptprev + bg;
  for (int j = tid; j < ng; j += nt) {
    const double dp = p[j] - pt[j];
    if (engine == NRTO_FULLADMM) {
      lam[j] += dp;
      tin[j] = p[j] + lam[j];
    } else {
      lam[j] += rho * dp;
    }
    ap += dp * dp;
    const double dd = pt[j] - ptp[j];
    ad += dd * dd;
    ptp[j] = pt[j];
  }
  ap = block_sum(ap, red);
  ad = block_sum(ad, red);
  if (tid == 0) {
    const double rpv = sqrt(ap), rdv = rho * sqrt(ad);
    v.r_p[b] = rpv;
    v.r_d[b] = rdv;
    record_hist(v, b, l, rpv, rdv, engine);
    v.iters[b] = l;
    if (!isfinite(rpv) || !isfinite(rdv)) {
      v.status[b] = NRTO_DIVERGED;
      v.active[b] = 0;
    } else if (!v.prm.fixed_iters && (l % v.prm.check_every) == 0 && rpv <= v.prm.eps_p &&
               rdv <= v.prm.eps_d) {
      v.status[b] = NRTO_CONVERGED;
      v.active[b] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// Chunked-scan QP for small batches (parallel-in-time
// Riccati).  Same OSQP iteration as qp_instance (R1, F4), but the two linear
// recurrences of the Riccati x-step,
//   s_k = a_k + Acl_k^T s_{k+1}   (backward)     dx_{k+1} = Acl_k dx_k + e_k   (forward),
// are not run as 2T dependent steps on one warp.  The horizon is cut into C
// chunks of M steps; each warp runs its chunk's recurrence from a zero boundary
// (the last / first chunk from the exact s_T / dx_0 = 0), one warp chains the C
// chunk boundaries with the transfer matrices of setup (k_scan_factors),
//   s_lo = s~_lo + PhiB_lo s_{hi+1},     dx_{hi+1} = x~_{hi+1} + PhiF_hi dx_lo,
// and every thread fixes up the interior steps in parallel.  Depth per sweep
// M + C + 1 instead of T (T = 100: 10 + 10 + 1).  Everything k-parallel (a_k,
// kff_k, e_k, du~_k, the rows, the ball) runs on all 512 threads between block
// barriers; Acl of the horizon is staged in shared memory when it fits.
void scan_plan(int T, int& M, int& C) {
  int m = (int)std::ceil(std::sqrt((double)T));
  int c = (T + m - 1) / m;
  while (c > 16) { ++m; c = (T + m - 1) / m; }    // one warp per chunk (512 threads)
  M = m; C = c;
}

__global__ void k_scan_factors(Dev v, int eng) {
  extern __shared__ double sm[];
  const Dims d = v.d;
  const int nx = d.nx, T = d.T, M = v.scanM, C = v.scanC, nn = nx * nx;
  const int b = blockIdx.x / C, c = blockIdx.x % C;
  const int lo = c * M, hi = min(T, (c + 1) * M) - 1;
  const EngineFactors& F = eng == 0 ? v.fa : v.dr;
  const double* Acl = F.Acl + (int64_t)b * T * nn;
  double* PB = F.PhiB + (int64_t)b * T * nn;
  double* PF = F.PhiF + (int64_t)b * T * nn;
  const int tid = threadIdx.x, i = tid / nx, j = tid % nx;
  double* P = sm;
  if (tid < nn) { P[tid] = Acl[(int64_t)hi * nn + j * nx + i]; PB[(int64_t)hi * nn + tid] = P[tid]; }
  __syncthreads();
  for (int k = hi - 1; k >= lo; --k) {            // PhiB_k = Acl_k^T PhiB_{k+1}
    double acc = 0.0;
    if (tid < nn)
      for (int r = 0; r < nx; ++r) acc += Acl[(int64_t)k * nn + r * nx + i] * P[r * nx + j];
    __syncthreads();
    if (tid < nn) { P[tid] = acc; PB[(int64_t)k * nn + tid] = acc; }
    __syncthreads();
  }
  if (tid < nn) { P[tid] = Acl[(int64_t)lo * nn + tid]; PF[(int64_t)lo * nn + tid] = P[tid]; }
  __syncthreads();
  for (int k = lo + 1; k <= hi; ++k) {            // PhiF_k = Acl_k PhiF_{k-1}
    double acc = 0.0;
    if (tid < nn)
      for (int r = 0; r < nx; ++r) acc += Acl[(int64_t)k * nn + i * nx + r] * P[r * nx + j];
    __syncthreads();
    if (tid < nn) { P[tid] = acc; PF[(int64_t)k * nn + tid] = acc; }
    __syncthreads();
  }
}

cudaError_t launch_scan_factors(nrto_handle_s* h, int engine, cudaStream_t st) {
  const Dev& v = h->dev;
  const int nn = v.d.nx * v.d.nx;
  k_scan_factors<<<v.d.B * v.scanC, (nn + 31) / 32 * 32, nn * sizeof(double), st>>>(v, engine);
  h->launches++;
  return cudaGetLastError();
}

// One step of a warp recurrence: lane i < nx returns base_i + sum_r Mat(i, r) x_r,
// x in shared memory (broadcast reads; LDS.128 pairs when n_x is a compile-time
// even number), four independent FMA chains.
template <int NXM, class MF>
__device__ __forceinline__ double scan_step(int nx, int lane, double base, const double* x, MF mat) {
  double c0 = base, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  const int ic = lane < nx ? lane : 0;
  if constexpr (NXM > 0 && (NXM % 2) == 0) {
#pragma unroll
    for (int r = 0; r < NXM; r += 2) {
      const double2 xx = *reinterpret_cast<const double2*>(x + r);
      if ((r >> 1) & 1) { c2 = fma(mat(ic, r), xx.x, c2); c3 = fma(mat(ic, r + 1), xx.y, c3); }
      else { c0 = fma(mat(ic, r), xx.x, c0); c1 = fma(mat(ic, r + 1), xx.y, c1); }
    }
  } else {
    constexpr int NR = NXM > 0 ? NXM : 32;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (r >= nx) break;
      const double t = mat(ic, r);
      switch (r & 3) {
        case 0: c0 = fma(t, x[r], c0); break;
        case 1: c1 = fma(t, x[r], c1); break;
        case 2: c2 = fma(t, x[r], c2); break;
        default: c3 = fma(t, x[r], c3); break;
      }
    }
  }
  return (c0 + c1) + (c2 + c3);
}

// Shared-memory staging of the scan QP's per-step constants (bit mask, staged in
// this priority order while they fit): 1 Acl (the recurrences), 2 Kf, 4 H^-1 and
// H^-1 B^T, 8 B, 16 the transfer matrices PhiB / PhiF (short chunks), 32 the mutable
// QP vectors (p, z, y, the ball pair, du, the knot accumulators) for the launch.
constexpr int kScanStageBits = 6;
static size_t scan_stage_doubles(const Dims& d, int bit) {
  const size_t T = d.T, nx = d.nx, nu = d.nu, ng = d.ng;
  switch (bit) {
    case 0: return T * nx * nx;
    case 1: return T * nu * nx;
    case 2: return T * nu * nu + T * nu * nx;
    case 3: return T * nx * nu;
    case 4: return 2 * T * nx * nx;
    default: return 4 * ng + 3 * (T + 1) * nx + 2 * T * nu;   // resident mutable vectors
  }
}
static size_t scan_smem(const Dims& d, int C, int smask) {
  size_t n = (size_t)(d.T + 1) * d.nx + (size_t)d.T * d.nx + 2 * (size_t)d.T * d.nu +
             2 * (size_t)C * d.nx * d.nx;
  for (int b = 0; b < kScanStageBits; ++b)
    if (smask & (1 << b)) n += scan_stage_doubles(d, b);
  return n * sizeof(double);
}

// debug phase clocks of the scan QP (instance 0, QP iterations 0-1): g_qp_clk[it*32 + ph]
#define SCAN_CLK(ph) \
  do { if (b == 0 && tid == 0 && it < 2) g_qp_clk[it * 32 + (ph)] = clock64(); } while (0)
template <int NXM, int NUM>
__device__ __forceinline__ void qp_scan_run(const Dev& v, int engine, int l, int smask, int b, double* sm,
                                            double* red) {
  const Dims d = v.d;
  const int nx = NXM > 0 ? NXM : d.nx, nu = NUM > 0 ? NUM : d.nu, T = d.T, ng = d.ng;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int M = v.scanM, C = v.scanC, nn = nx * nx;
  if (!v.active[b]) return;
  const EngineFactors& F = engine == NRTO_FULLADMM ? v.fa : v.dr;
  const double rho = engine == NRTO_FULLADMM ? v.prm.rho : v.prm.rho_admm;
  const double rq = v.prm.rho_qp, sq = v.prm.sigma_qp, aq = v.prm.alpha_qp;
  const double den = rho + sq + rq, beta = rq / den, irq = 1.0 / rq;
  const int64_t bg = (int64_t)b * ng;
  const double* __restrict__ grad = v.grad + bg * nx;
  const double* __restrict__ g0 = v.g0 + bg;
  double* const p_g = v.p + bg; double* const zl_g = v.zl + bg; double* const yl_g = v.yl + bg;
  double* p = p_g; double* zl = zl_g; double* yl = yl_g;
  double* rp = v.rp + bg;
  const double* pt = v.pt + bg; double* lam = v.lamp + bg;
  double* const zb_g = v.zb + (int64_t)b * (T + 1) * nx; double* const yb_g = v.yb + (int64_t)b * (T + 1) * nx;
  double* const du_g = v.du + (int64_t)b * T * nu;
  double* zb = zb_g; double* yb = yb_g; double* du = du_g;
  double* gS = v.rx + (int64_t)b * (T + 1) * nx;      // S_k = sum_{state j@k} w_j grad_j (atomic)
  double* gU = v.dut + (int64_t)b * T * nu;           // U_k = sum_{ctrl j@k} w_j h'_j   (atomic)
  const double* __restrict__ cu2 = v.cu2 + (int64_t)b * T * nu;
  const double* KfG = F.Kf + (int64_t)b * T * nu * nx;
  const double* AclG = F.Acl + (int64_t)b * T * nn;
  const double* HiG = F.Hinv + (int64_t)b * T * nu * nu;
  const double* HBG = F.HB + (int64_t)b * T * nu * nx;
  const double* BmG = v.Bm + (int64_t)b * T * nx * nu;
  const double* PBg = F.PhiB + (int64_t)b * T * nn;
  const double* PFg = F.PhiF + (int64_t)b * T * nn;
  const double rtr = v.rtrust[b];
  const double rinv = (engine == NRTO_FULLADMM) ? 1.0 : 1.0 / rho;
  double* sS = sm;                          // [(T+1) nx]  s~/s, then dx~/dx, then z^_ball
  double* sA = sS + (T + 1) * nx;           // [T nx]      a_k, then e_k
  double* sR = sA + T * nx;                 // [T nu]      r_u,k, then du~_k
  double* sK = sR + T * nu;                 // [T nu]      kff_k
  double* sPb = sK + T * nu;                // [C][nx][nx] PhiB at chunk starts
  double* sPf = sPb + C * nn;               // [C][nx][nx] PhiF at chunk ends
  // staged per-step constants (smask), in this order after sPf
  double* nxt = sPf + C * nn;
  auto stage = [&](int bit, const double* g, int64_t n) -> const double* {
    if (!(smask & (1 << bit))) return g;
    double* dst = nxt;
    nxt += n;
    for (int64_t r = tid; r < n; r += nt) dst[r] = g[r];
    return dst;
  };
  const double* __restrict__ Acl = stage(0, AclG, (int64_t)T * nn);
  const double* __restrict__ Kf = stage(1, KfG, (int64_t)T * nu * nx);
  const double* __restrict__ Hi = stage(2, HiG, (int64_t)T * nu * nu);
  const double* __restrict__ HB = (smask & 4) ? stage(2, HBG, (int64_t)T * nu * nx) : HBG;
  const double* __restrict__ Bm = stage(3, BmG, (int64_t)T * nx * nu);
  const double* __restrict__ PB = stage(4, PBg, (int64_t)T * nn);
  const double* __restrict__ PF = (smask & 16) ? stage(4, PFg, (int64_t)T * nn) : PFg;
  // interior steps: long chunks re-run the chunk from its exact boundary (M more
  // dependent steps, shared-memory operands only); short chunks add PhiB_k s_{hi+1} /
  // PhiF_k dx_lo in one parallel phase (one round of transfer-matrix loads)
  const bool rescan = M >= 8;
  // bit 32: the QP's mutable vectors live in shared memory for the launch (copied in
  // here, out before the tail); the knot accumulators S, U then take shared atomics
  const bool res = (smask & 32) != 0;
  if (res) {
    auto take = [&](int64_t n) { double* q = nxt; nxt += n; return q; };
    p = take(ng); zl = take(ng); yl = take(ng); rp = take(ng);
    zb = take((int64_t)(T + 1) * nx); yb = take((int64_t)(T + 1) * nx); gS = take((int64_t)(T + 1) * nx);
    du = take((int64_t)T * nu); gU = take((int64_t)T * nu);
    for (int r = tid; r < ng; r += nt) { p[r] = p_g[r]; zl[r] = zl_g[r]; yl[r] = yl_g[r]; }
    for (int r = tid; r < (T + 1) * nx; r += nt) { zb[r] = zb_g[r]; yb[r] = yb_g[r]; }
    for (int r = tid; r < T * nu; r += nt) du[r] = du_g[r];
  }
  auto ldacc = [&](const double* q) { return res ? *q : __ldcg(q); };
  for (int r = tid; r < C * nn; r += nt) {
    const int c = r / nn, e = r - c * nn;
    sPb[r] = PBg[(int64_t)(c * M) * nn + e];
    sPf[r] = PFg[(int64_t)(min(T, (c + 1) * M) - 1) * nn + e];
  }
  for (int r = tid; r < (T + 1) * nx; r += nt) gS[r] = 0.0;
  for (int r = tid; r < T * nu; r += nt) gU[r] = 0.0;
  __syncthreads();
  const int nits = v.prm.qp_iters;
  if (nits > 0) {                                     // rhs / w / scatter of iteration 0
    qp_rows<true, kRowBatch>(v, bg, ng, tid, nt, grad, g0, p, zl, yl, rp, pt, lam, sS, sR, gS, gU, true,
                             rho, rq, sq, aq, den, beta, rinv);
    __syncthreads();
  }
  for (int it = 0; it < nits; ++it) {
    SCAN_CLK(0);
    for (int r = tid; r < T * nu; r += nt) {          // r_u (consumes and clears U)
      sR[r] = sq * du[r] + ldacc(gU + r) + cu2[r];    // cu2 = -2 R_u u_hat (setup)
      gU[r] = 0.0;
    }
    __syncthreads(); SCAN_CLK(1);
    for (int r = tid; r < (T + 1) * nx; r += nt) {    // r_x and a_k (consumes and clears S)
      const int k = r / nx, i = r - k * nx;
      double acc = (k > 0) ? ldacc(gS + r) + rq * zb[r] - yb[r] : 0.0;
      gS[r] = 0.0;
      if (k < T) {
        const double* Kk = Kf + (int64_t)k * nu * nx + i;
        const double* rk = sR + k * nu;
        acc -= dotn<NUM>(nu, [&](int m) { return Kk[m * nx]; }, [&](int m) { return rk[m]; }, 0.0);
      }
      if (k < T) sA[r] = acc;                         // a_k
      else sS[r] = acc;                               // s_T
    }
    __syncthreads(); SCAN_CLK(2);
    if (warp < C) {                                   // chunk-local backward recurrences
      const int lo = warp * M, hi = min(T, (warp + 1) * M) - 1;
      for (int k = hi; k >= lo; --k) {
        const double* Ak = Acl + (size_t)k * nn;
        const double base = lane < nx ? sA[k * nx + lane] : 0.0;
        // s~_{hi+1} = 0 for all but the last chunk (which starts from the exact s_T)
        const double x = (k == hi && warp != C - 1)
                             ? base
                             : scan_step<NXM>(nx, lane, base, sS + (k + 1) * nx,
                                               [&](int i, int r) { return Ak[r * nx + i]; });
        __syncwarp();
        if (lane < nx) sS[k * nx + lane] = x;
        __syncwarp();
      }
    }
    __syncthreads(); SCAN_CLK(3);
    if (warp == 0) {                                  // chunk boundaries, last to first
      for (int c = C - 2; c >= 0; --c) {
        const double* P = sPb + c * nn;
        const double base = lane < nx ? sS[c * M * nx + lane] : 0.0;
        const double x = scan_step<NXM>(nx, lane, base, sS + (c + 1) * M * nx,
                                         [&](int i, int r) { return P[i * nx + r]; });
        __syncwarp();
        if (lane < nx) sS[c * M * nx + lane] = x;
        __syncwarp();
      }
    }
    __syncthreads(); SCAN_CLK(4);
    if (!rescan) {
      for (int r = tid; r < T * nx; r += nt) {        // interior fix-up s_k += PhiB_k s_{hi+1}
        const int k = r / nx, i = r - k * nx, c = k / M;
        if (c == C - 1 || k == c * M) continue;
        const double* Pk = PB + (int64_t)k * nn + i * nx;
        const double* sn = sS + (c + 1) * M * nx;
        sS[r] += dotn<NXM>(nx, [&](int q) { return Pk[q]; }, [&](int q) { return sn[q]; }, 0.0);
      }
    } else if (warp < C - 1) {                        // interior: re-run each chunk from its
      const int lo = warp * M, hi = min(T, (warp + 1) * M) - 1;   // exact boundary s_{hi+1}
      for (int k = hi; k > lo; --k) {
        const double* Ak = Acl + (size_t)k * nn;
        const double base = lane < nx ? sA[k * nx + lane] : 0.0;
        const double x = scan_step<NXM>(nx, lane, base, sS + (k + 1) * nx,
                                        [&](int i, int r) { return Ak[r * nx + i]; });
        __syncwarp();
        if (lane < nx) sS[k * nx + lane] = x;
        __syncwarp();
      }
    }
    __syncthreads(); SCAN_CLK(5);
    for (int r = tid; r < T * nu; r += nt) {          // kff_k = H^-1 r_u,k + H^-1 B_k^T s_{k+1}
      const int k = r / nu, m = r - k * nu;
      const double* H = Hi + (int64_t)k * nu * nu + m * nu;
      const double* hb = HB + (int64_t)k * nu * nx + m * nx;
      const double* rk = sR + k * nu;
      const double* sk = sS + (k + 1) * nx;
      double acc = dotn<NUM>(nu, [&](int q) { return H[q]; }, [&](int q) { return rk[q]; }, 0.0);
      acc = dotn<NXM>(nx, [&](int q) { return hb[q]; }, [&](int q) { return sk[q]; }, acc);
      sK[r] = acc;
    }
    __syncthreads(); SCAN_CLK(6);
    for (int r = tid; r < T * nx; r += nt) {          // e_k = B_k kff_k
      const int k = r / nx, i = r - k * nx;
      const double* Bk = Bm + (int64_t)k * nx * nu + i * nu;
      const double* kk = sK + k * nu;
      sA[r] = dotn<NUM>(nu, [&](int m) { return Bk[m]; }, [&](int m) { return kk[m]; }, 0.0);
    }
    __syncthreads(); SCAN_CLK(7);
    if (warp < C) {                                   // chunk-local forward recurrences
      const int lo = warp * M, hi = min(T, (warp + 1) * M) - 1;
      if (warp == 0 && lane < nx) sS[lane] = 0.0;     // dx_0 = 0
      for (int k = lo; k <= hi; ++k) {
        const double* Ak = Acl + (size_t)k * nn;
        const double base = lane < nx ? sA[k * nx + lane] : 0.0;
        // x~_lo = 0 (slot lo belongs to the previous chunk's warp)
        const double x = (k == lo) ? base
                                   : scan_step<NXM>(nx, lane, base, sS + k * nx,
                                                     [&](int i, int r) { return Ak[i * nx + r]; });
        if (lane < nx) sS[(k + 1) * nx + lane] = x;
        __syncwarp();
      }
    }
    __syncthreads(); SCAN_CLK(8);
    if (warp == 0) {                                  // chunk boundaries, first to last
      for (int c = 1; c < C; ++c) {
        const int hi = min(T, (c + 1) * M) - 1;
        const double* P = sPf + c * nn;
        const double base = lane < nx ? sS[(hi + 1) * nx + lane] : 0.0;
        const double x = scan_step<NXM>(nx, lane, base, sS + c * M * nx,
                                         [&](int i, int r) { return P[i * nx + r]; });
        __syncwarp();
        if (lane < nx) sS[(hi + 1) * nx + lane] = x;
        __syncwarp();
      }
    }
    __syncthreads(); SCAN_CLK(9);
    if (!rescan) {
      for (int r = tid; r < T * nx; r += nt) {        // interior fix-up dx_{k+1} += PhiF_k dx_lo
        const int k = r / nx, i = r - k * nx, c = k / M;
        const int hi = min(T, (c + 1) * M) - 1;
        if (c == 0 || k == hi) continue;
        const double* Pk = PF + (int64_t)k * nn + i * nx;
        const double* xl = sS + c * M * nx;
        sS[r + nx] += dotn<NXM>(nx, [&](int q) { return Pk[q]; }, [&](int q) { return xl[q]; }, 0.0);
      }
    } else if (warp >= 1 && warp < C) {               // interior: re-run each chunk from its
      const int lo = warp * M, hi = min(T, (warp + 1) * M) - 1;   // exact boundary dx_lo
      for (int k = lo; k < hi; ++k) {
        const double* Ak = Acl + (size_t)k * nn;
        const double base = lane < nx ? sA[k * nx + lane] : 0.0;
        const double x = scan_step<NXM>(nx, lane, base, sS + k * nx,
                                        [&](int i, int r) { return Ak[i * nx + r]; });
        if (lane < nx) sS[(k + 1) * nx + lane] = x;
        __syncwarp();
      }
    }
    __syncthreads(); SCAN_CLK(10);
    for (int r = tid; r < T * nu; r += nt) {          // du~_k = kff_k - Kf_k dx_k ; relaxed du
      const int k = r / nu, m = r - k * nu;
      const double* Kk = Kf + (int64_t)k * nu * nx + m * nx;
      const double* xk = sS + k * nx;
      const double dd = sK[r] - dotn<NXM>(nx, [&](int q) { return Kk[q]; }, [&](int q) { return xk[q]; }, 0.0);
      sR[r] = dd;
      du[r] = aq * dd + (1.0 - aq) * du[r];
    }
    __syncthreads(); SCAN_CLK(11);
    const bool more = it + 1 < nits;
    qp_rows<false, kRowBatch>(v, bg, ng, tid, nt, grad, g0, p, zl, yl, rp, pt, lam, sS, sR, gS, gU, more,
                              rho, rq, sq, aq, den, beta, rinv);
    __syncthreads(); SCAN_CLK(12);
    double nb = 0.0;                                  // trust-region ball
    for (int r = tid; r < (T + 1) * nx; r += nt) {
      const double zh = aq * sS[r] + (1.0 - aq) * zb[r];
      sS[r] = zh;
      const double w = zh + yb[r] * irq;
      nb += w * w;
    }
    nb = sqrt(block_sum(nb, red));
    const double scl = (nb > rtr) ? rtr / nb : 1.0;
    for (int r = tid; r < (T + 1) * nx; r += nt) {
      const double zh = sS[r];
      const double zn = scl * (zh + yb[r] * irq);
      yb[r] += rq * (zh - zn);
      zb[r] = zn;
    }
    __syncthreads(); SCAN_CLK(13);
  }
  if (res) {                                          // resident vectors back to global
    for (int r = tid; r < ng; r += nt) { p_g[r] = p[r]; zl_g[r] = zl[r]; yl_g[r] = yl[r]; }
    for (int r = tid; r < (T + 1) * nx; r += nt) { zb_g[r] = zb[r]; yb_g[r] = yb[r]; }
    for (int r = tid; r < T * nu; r += nt) du_g[r] = du[r];
  }
  double ap = 0.0, ad = 0.0;
  double* tin = v.tin + bg;
  double* ptp = v.ptprev + bg;
  for (int j = tid; j < ng; j += nt) {
    const double dp = p[j] - pt[j];
    if (engine == NRTO_FULLADMM) {
      lam[j] += dp;
      tin[j] = p[j] + lam[j];
    } else {
      lam[j] += rho * dp;
    }
    ap += dp * dp;
    const double dd = pt[j] - ptp[j];
    ad += dd * dd;
    ptp[j] = pt[j];
  }
  ap = block_sum(ap, red);
  ad = block_sum(ad, red);
  if (tid == 0) {
    const double rpv = sqrt(ap), rdv = rho * sqrt(ad);
    v.r_p[b] = rpv;
    v.r_d[b] = rdv;
    record_hist(v, b, l, rpv, rdv, engine);
    v.iters[b] = l;
    if (!isfinite(rpv) || !isfinite(rdv)) {
      v.status[b] = NRTO_DIVERGED;
      v.active[b] = 0;
    } else if (!v.prm.fixed_iters && (l % v.prm.check_every) == 0 && rpv <= v.prm.eps_p &&
               rdv <= v.prm.eps_d) {
      v.status[b] = NRTO_CONVERGED;
      v.active[b] = 0;
    }
  }
}

template <int NXM, int NUM>
__global__ void __launch_bounds__(512, 1) k_qp_scan(Dev v, int engine, int l, int smask) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  qp_scan_run<NXM, NUM>(v, engine, l, smask, blockIdx.x, sm, red);
}

// ---------------------------------------------------------------------------
// Whole FullADMM loop of one small instance per CTA (SURVEY §8f NEXT-3(ii) for the
// c1-class sizes, Algorithm 1): every outer iteration runs the generic
// cone pass (13) with the pending dual update (16), the adjoint S7, the gain
// update (14b) and the chunked-scan QP (14a) + duals / residuals back to back with
// block barriers, instead of four kernel launches per iteration.  Same per-element
// arithmetic as k_fa_pass, k_adjoint (cone-list order), k_fa_gain (warp-level
// chain) and k_qp_scan; per-instance termination (R11, R12) ends the CTA's loop.
template <int NXM, int NUM>
__global__ void __launch_bounds__(512, 1) k_fa_small(Dev v, int L, int smask) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  const Dims d = v.d;
  const int nx = NXM > 0 ? NXM : d.nx, nu = NUM > 0 ? NUM : d.nu, T = d.T, ng = d.ng;
  const int NA = nu * nx;
  const int b = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const double st = sqrt(v.tau[b]);
  const double rho = v.prm.rho;
  for (int l = 1; l <= L; ++l) {
    if (!v.active[b]) break;                          // set by the QP tail (barrier below)
    // ---- (13) + pending (16): y = D b + b_hat + (1 - s) y, projection per cone
    for (int j = warp; j < ng; j += nw) {
      const ConeGeom g = cone_geom(v, j);
      const int64_t ij = (int64_t)b * ng + j;
      const double omsp = 1.0 - v.s[ij];
      double* Y = v.Y + (int64_t)b * d.E + g.off;
      const double* bh = v.bhat + (int64_t)b * d.E + g.off;
      const double* Bd = v.Bd + (int64_t)b * d.EB + g.offB;
      const double* Dm = v.D + (int64_t)b * T * nx * nu;
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
      double s;
      const double tp = soc_case(v.tin[ij], sqrt(n2), &s);
      if (lane == 0) { v.s[ij] = s; v.pt[ij] = tp; }
      if (v.case_cnt && l <= v.hist_L && lane == 0) {
        unsigned long long* cc = v.case_cnt + (int64_t)(l - 1) * 3;
        atomicAdd(cc + (s == 1.0 ? 0 : (s == 0.0 ? 1 : 2)), 1ULL);
      }
    }
    __syncthreads();
    // ---- S7: Z_k = sum_j s_j b_{j,k} y_{j,k}^T (cones with a block at k, list order)
    for (int r = tid; r < T * NA; r += nt) {
      const int k = r / NA, o = r - k * NA, m = o / nx, i = o - m * nx;
      const double* yb = v.Y + (int64_t)b * d.E;
      const double* Bd = v.Bd + (int64_t)b * d.EB;
      double acc = 0.0;
      for (int c = v.kptr[k]; c < v.kptr[k + 1]; ++c) {
        const int j = v.kcone[c];
        const int kb = (v.kind[j] == 0) ? k : 0;
        acc += Bd[v.offB[j] + kb * d.nup + m] * yb[v.off[j] + kb * nx + i] * v.s[(int64_t)b * ng + j];
      }
      v.Z[((int64_t)b * T + k) * NA + o] = acc;
    }
    __syncthreads();
    // ---- (14b): R = 2 W K + rho sqrt(tau) (Z - Zb) Psi_k, K = chain, C, D (warp per step)
    for (int k = warp; k < T; k += nw) {
      const int64_t bk = (int64_t)b * T + k;
      double* sR = sm + (size_t)warp * 3 * NA;
      double* sX = sR + NA;
      double* sK = sX + NA;
      const double* Pk = v.Psi + ((int64_t)b * (T + 1) + k) * nx * nx;
      const double* Wk = v.W + bk * nu * nu;
      double* Kb = v.K + (int64_t)b * d.NK + (int64_t)k * NA;
      for (int r = lane; r < NA; r += 32) {
        sX[r] = v.Z[bk * NA + r] - v.Zb[bk * NA + r];
        const int m = r / nx, i = r % nx;
        sK[r] = Kb[i * nu + m];
      }
      __syncwarp();
      for (int r = lane; r < NA; r += 32) {
        const int m = r / nx, i = r % nx;
        double gp = 0.0, wk = 0.0;
        for (int q = 0; q < nx; ++q) gp += sX[m * nx + q] * Pk[q * nx + i];
        for (int q = 0; q < nu; ++q) wk += Wk[m * nu + q] * sK[q * nx + i];
        sR[r] = 2.0 * wk + rho * st * gp;
      }
      __syncwarp();
      chain_solve_w<NXM, NUM>(v.fa.V + bk * nu * nu, v.U + bk * nx * nx, v.fa.den + bk * NA, sR, sX,
                               nu, nx, lane);
      for (int r = lane; r < NA; r += 32) {
        const int m = r / nx, i = r % nx;
        Kb[i * nu + m] = sR[r];
      }
      for (int r = lane; r < NA; r += 32) {
        const int i = r / nu, m = r % nu;
        double acc = 0.0;
        for (int q = 0; q < nx; ++q) acc += Pk[i * nx + q] * sR[m * nx + q];
        const double c = st * acc;
        const int64_t idx = bk * NA + r;
        const double cold = v.Ccur[idx];
        v.Cprev[idx] = cold;
        v.Ccur[idx] = c;
        v.D[idx] = 2.0 * c - cold;
      }
      __syncwarp();
    }
    __syncthreads();
    // ---- (14a) QP + (16) lam_p + residuals + termination
    qp_scan_run<NXM, NUM>(v, NRTO_FULLADMM, l, smask, b, sm, red);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Grid-wide QP for ONE large instance (SURVEY §8f NEXT-3(iii) at c4 scale: a
// quadcopter with T = 800 and 166 k rows took 50 ms per QP launch on one CTA).
// Same OSQP iteration and chunked-scan recurrences as qp_scan_run (R1, R26), but
// every k-parallel phase and the row phase run on the whole grid (cooperative
// launch, grid barriers), each chunk's recurrence on its own CTA with the chunk's
// Acl in shared memory, the boundary chains on CTA 0.  Cross-CTA vectors go
// through L2 (ld.global.cg); the row phase reads dx and du~ from a shared-memory
// copy.  Ten grid barriers per QP iteration.
__device__ __forceinline__ unsigned long long qg_ld_acquire(const unsigned long long* p) {
  unsigned long long x;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
  return x;
}
__device__ __forceinline__ void qg_barrier(unsigned long long* ctr, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    while (qg_ld_acquire(ctr) < target) {
    }
  }
  __syncthreads();
}

bool qp_grid_plan(const Dims& d, int nsm, int& M, int& C) {
  static const int env = [] { const char* e = getenv("NRTO_QP_GRID"); return e ? atoi(e) : -1; }();
  if (d.B != 1 || env == 0 || d.T < 8) return false;
  const size_t base = ((size_t)(d.T + 1) * d.nx + (size_t)d.T * d.nx + 2 * (size_t)d.T * d.nu) * 8;
  // large: many rows, or the one-CTA scan QP's vectors alone exceed its shared memory
  if (env != 1 && d.ng < 16384 && base <= 150 * 1024) return false;
  int m = (int)std::ceil(std::sqrt((double)d.T));
  int c = (d.T + m - 1) / m;
  while (c > nsm) { ++m; c = (d.T + m - 1) / m; }
  M = m; C = c;
  return true;
}

static size_t qg_smem(const Dims& d, int M, int C) {
  const size_t nn = (size_t)d.nx * d.nx;
  return ((size_t)M * nn + 2 * (size_t)C * nn + (size_t)M * d.nx + (size_t)(M + 1) * d.nx +
          (size_t)(d.T + 1) * d.nx + (size_t)d.T * d.nu) * sizeof(double);
}

template <int NXM, int NUM>
__global__ void __launch_bounds__(512, 1) k_qp_grid(Dev v, int engine, int l) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ double bcast;
  const Dims d = v.d;
  const int nx = NXM > 0 ? NXM : d.nx, nu = NUM > 0 ? NUM : d.nu, T = d.T, ng = d.ng;
  const int b = 0, tid = threadIdx.x, nt = blockDim.x, G = gridDim.x, cta = blockIdx.x;
  const int gtid = cta * nt + tid, gnt = G * nt;
  const int warp = tid >> 5, lane = tid & 31;
  const int M = v.scanM, C = v.scanC, nn = nx * nx;
  if (!v.active[b]) return;                          // uniform over the grid
  const EngineFactors& F = engine == NRTO_FULLADMM ? v.fa : v.dr;
  const double rho = engine == NRTO_FULLADMM ? v.prm.rho : v.prm.rho_admm;
  const double rq = v.prm.rho_qp, sq = v.prm.sigma_qp, aq = v.prm.alpha_qp;
  const double den = rho + sq + rq, beta = rq / den, irq = 1.0 / rq;
  const double rinv = (engine == NRTO_FULLADMM) ? 1.0 : 1.0 / rho;
  const double* __restrict__ grad = v.grad;
  const double* __restrict__ g0 = v.g0;
  double* p = v.p; double* zl = v.zl; double* yl = v.yl; double* rp = v.rp;
  const double* pt = v.pt; double* lam = v.lamp;
  double* zb = v.zb; double* yb = v.yb; double* du = v.du;
  double* gS = v.rx; double* gU = v.dut; double* gR = v.ru; double* gK = v.kff;
  double* gdx = v.dxt; double* gs = v.qg_s; double* ga = v.qg_a;
  const double* __restrict__ cu2 = v.cu2;
  const double* __restrict__ Bm = v.Bm;
  const double* __restrict__ Kf = F.Kf;
  const double* __restrict__ Acl = F.Acl;
  const double* __restrict__ Hi = F.Hinv;
  const double* __restrict__ HB = F.HB;
  const double rtr = v.rtrust[b];
  // shared memory: my chunk's Acl, the boundary transfer matrices (CTA 0), chunk
  // vectors, and the row phase's copies of dx and du~
  double* sAc = sm;                                  // [M][nn]
  double* sPb = sAc + (size_t)M * nn;                // [C][nn]
  double* sPf = sPb + (size_t)C * nn;                // [C][nn]
  double* sVa = sPf + (size_t)C * nn;                // [M][nx]   a_k / e_k of my chunk
  double* sVs = sVa + (size_t)M * nx;                // [M+1][nx] chunk vector
  double* sX = sVs + (size_t)(M + 1) * nx;           // [(T+1)][nx] dx (row phase)
  double* sU = sX + (size_t)(T + 1) * nx;            // [T][nu]     du~ (row phase)
  const int lo = cta * M, hi = min(T, (cta + 1) * M) - 1;
  const bool mine = cta < C;
  if (mine)
    for (int r = tid; r < (hi - lo + 1) * nn; r += nt) sAc[r] = Acl[(int64_t)lo * nn + r];
  if (cta == 0)
    for (int r = tid; r < C * nn; r += nt) {
      const int c = r / nn, e = r - c * nn;
      sPb[r] = F.PhiB[(int64_t)(c * M) * nn + e];
      sPf[r] = F.PhiF[(int64_t)(min(T, (c + 1) * M) - 1) * nn + e];
    }
  unsigned long long nbar = 0;
  auto gsync = [&]() { qg_barrier(v.qg_bar, (++nbar) * (unsigned long long)G); };
  for (int r = gtid; r < (T + 1) * nx; r += gnt) gS[r] = 0.0;
  for (int r = gtid; r < T * nu; r += gnt) gU[r] = 0.0;
  gsync();
  const int nits = v.prm.qp_iters;
  if (nits > 0) {
    qp_rows<true, kRowBatch>(v, 0, ng, gtid, gnt, grad, g0, p, zl, yl, rp, pt, lam, sX, sU, gS, gU, true,
                             rho, rq, sq, aq, den, beta, rinv);
    gsync();
  }
  // one step of a chunk recurrence on warp 0: x_out = base + Mat x_in (x_in in smem)
  auto step = [&](double base, const double* xin, const double* Mt, bool trans) {
    return scan_step<NXM>(nx, lane, base, xin, [&](int i, int r) { return trans ? Mt[r * nx + i] : Mt[i * nx + r]; });
  };
  for (int it = 0; it < nits; ++it) {
    // A: r_u (to gR) and a_k (to ga), s_T (to gs); S consumed and cleared
    for (int r = gtid; r < T * nu; r += gnt) gR[r] = sq * __ldcg(du + r) + __ldcg(gU + r) + cu2[r];
    for (int r = gtid; r < (T + 1) * nx; r += gnt) {
      const int k = r / nx, i = r - k * nx;
      double acc = (k > 0) ? __ldcg(gS + r) + rq * zb[r] - yb[r] : 0.0;
      gS[r] = 0.0;
      if (k < T) {
        for (int m = 0; m < nu; ++m) {
          const int q = k * nu + m;
          const double ru = sq * __ldcg(du + q) + __ldcg(gU + q) + cu2[q];
          acc -= Kf[(int64_t)k * nu * nx + m * nx + i] * ru;
        }
        ga[r] = acc;
      } else {
        gs[r] = acc;
      }
    }
    gsync();
    // B1: chunk-local backward recurrences (the last chunk from s_T: exact)
    if (mine) {
      for (int r = tid; r < (hi - lo + 1) * nx; r += nt) sVa[r] = __ldcg(ga + (int64_t)lo * nx + r);
      if (tid < nx) sVs[(hi + 1 - lo) * nx + tid] = (cta == C - 1) ? __ldcg(gs + (int64_t)T * nx + tid) : 0.0;
      __syncthreads();
      if (warp == 0) {
        for (int k = hi; k >= lo; --k) {
          const double base = lane < nx ? sVa[(k - lo) * nx + lane] : 0.0;
          const double x = step(base, sVs + (k + 1 - lo) * nx, sAc + (size_t)(k - lo) * nn, true);
          __syncwarp();
          if (lane < nx) sVs[(k - lo) * nx + lane] = x;
          __syncwarp();
        }
        if (lane < nx) {
          if (cta == C - 1)
            for (int k = lo; k <= hi; ++k) gs[(int64_t)k * nx + lane] = sVs[(k - lo) * nx + lane];
          else
            gs[(int64_t)lo * nx + lane] = sVs[lane];
        }
      }
    }
    gsync();
    // B2: chunk starts, last to first (CTA 0)
    if (cta == 0 && warp == 0) {
      double* xv = sVs;                               // [2][nx] ping-pong
      if (lane < nx) xv[lane] = __ldcg(gs + (int64_t)(C - 1) * M * nx + lane);
      __syncwarp();
      for (int c = C - 2; c >= 0; --c) {
        const double base = lane < nx ? __ldcg(gs + (int64_t)c * M * nx + lane) : 0.0;
        const double x = step(base, xv, sPb + (size_t)c * nn, false);
        __syncwarp();
        if (lane < nx) { xv[lane] = x; gs[(int64_t)c * M * nx + lane] = x; }
        __syncwarp();
      }
    }
    gsync();
    // B3: re-run each chunk's interior from its exact boundary s_{hi+1}
    if (mine && cta < C - 1) {
      if (tid < nx) sVs[(hi + 1 - lo) * nx + tid] = __ldcg(gs + (int64_t)(hi + 1) * nx + tid);
      __syncthreads();
      if (warp == 0) {
        for (int k = hi; k > lo; --k) {
          const double base = lane < nx ? sVa[(k - lo) * nx + lane] : 0.0;
          const double x = step(base, sVs + (k + 1 - lo) * nx, sAc + (size_t)(k - lo) * nn, true);
          __syncwarp();
          if (lane < nx) { sVs[(k - lo) * nx + lane] = x; gs[(int64_t)k * nx + lane] = x; }
          __syncwarp();
        }
      }
    }
    gsync();
    // C: kff_k = H^-1 r_u,k + H^-1 B_k^T s_{k+1}, e_k = B_k kff_k (thread per k); U cleared
    for (int k = gtid; k < T; k += gnt) {
      double kf[NUM > 0 ? NUM : 32];
      for (int m = 0; m < nu; ++m) {
        double acc = 0.0;
        for (int q = 0; q < nu; ++q) acc += Hi[((int64_t)k * nu + m) * nu + q] * __ldcg(gR + k * nu + q);
        for (int i = 0; i < nx; ++i) acc += HB[((int64_t)k * nu + m) * nx + i] * __ldcg(gs + (int64_t)(k + 1) * nx + i);
        kf[m] = acc;
        gK[k * nu + m] = acc;
        gU[k * nu + m] = 0.0;
      }
      for (int i = 0; i < nx; ++i) {
        double acc = 0.0;
        for (int m = 0; m < nu; ++m) acc += Bm[((int64_t)k * nx + i) * nu + m] * kf[m];
        ga[(int64_t)k * nx + i] = acc;
      }
    }
    gsync();
    // D1: chunk-local forward recurrences (chunk 0 from dx_0 = 0: exact)
    if (mine) {
      for (int r = tid; r < (hi - lo + 1) * nx; r += nt) sVa[r] = __ldcg(ga + (int64_t)lo * nx + r);
      if (tid < nx) sVs[tid] = 0.0;
      __syncthreads();
      if (warp == 0) {
        for (int k = lo; k <= hi; ++k) {
          const double base = lane < nx ? sVa[(k - lo) * nx + lane] : 0.0;
          const double x = (k == lo) ? base : step(base, sVs + (k - lo) * nx, sAc + (size_t)(k - lo) * nn, false);
          if (lane < nx) sVs[(k + 1 - lo) * nx + lane] = x;
          __syncwarp();
        }
        if (lane < nx) {
          if (cta == 0)
            for (int k = 0; k <= hi + 1; ++k) gdx[(int64_t)k * nx + lane] = sVs[k * nx + lane];
          else
            gdx[(int64_t)(hi + 1) * nx + lane] = sVs[(hi + 1 - lo) * nx + lane];
        }
      }
    }
    gsync();
    // D2: chunk ends, first to last (CTA 0)
    if (cta == 0 && warp == 0) {
      double* xv = sVs;
      if (lane < nx) xv[lane] = __ldcg(gdx + (int64_t)min(T, M) * nx + lane);
      __syncwarp();
      for (int c = 1; c < C; ++c) {
        const int h2 = min(T, (c + 1) * M) - 1;
        const double base = lane < nx ? __ldcg(gdx + (int64_t)(h2 + 1) * nx + lane) : 0.0;
        const double x = step(base, xv, sPf + (size_t)c * nn, false);
        __syncwarp();
        if (lane < nx) { xv[lane] = x; gdx[(int64_t)(h2 + 1) * nx + lane] = x; }
        __syncwarp();
      }
    }
    gsync();
    // D3: re-run each chunk's interior from its exact boundary dx_lo
    if (mine && cta > 0) {
      if (tid < nx) sVs[tid] = __ldcg(gdx + (int64_t)lo * nx + tid);
      __syncthreads();
      if (warp == 0) {
        for (int k = lo; k < hi; ++k) {
          const double base = lane < nx ? sVa[(k - lo) * nx + lane] : 0.0;
          const double x = step(base, sVs + (k - lo) * nx, sAc + (size_t)(k - lo) * nn, false);
          if (lane < nx) { sVs[(k + 1 - lo) * nx + lane] = x; gdx[(int64_t)(k + 1) * nx + lane] = x; }
          __syncwarp();
        }
      }
    }
    gsync();
    // E: du~_k = kff_k - Kf_k dx_k, relaxed du
    for (int r = gtid; r < T * nu; r += gnt) {
      const int k = r / nu, m = r - k * nu;
      double acc = __ldcg(gK + r);
      for (int q = 0; q < nx; ++q) acc -= Kf[(int64_t)k * nu * nx + m * nx + q] * __ldcg(gdx + (int64_t)k * nx + q);
      gR[r] = acc;
      du[r] = aq * acc + (1.0 - aq) * __ldcg(du + r);
    }
    gsync();
    // F: rows (gather B du~, update p, z, y, scatter the next w) on a shared-memory copy
    //    of dx and du~; trust-region ball partial sums
    for (int r = tid; r < (T + 1) * nx; r += nt) sX[r] = __ldcg(gdx + r);
    for (int r = tid; r < T * nu; r += nt) sU[r] = __ldcg(gR + r);
    __syncthreads();
    const bool more = it + 1 < nits;
    qp_rows<false, kRowBatch>(v, 0, ng, gtid, gnt, grad, g0, p, zl, yl, rp, pt, lam, sX, sU, gS, gU, more,
                              rho, rq, sq, aq, den, beta, rinv);
    double nbp = 0.0;
    for (int r = gtid; r < (T + 1) * nx; r += gnt) {
      const double zh = aq * sX[r] + (1.0 - aq) * zb[r];
      const double w = zh + yb[r] * irq;
      nbp += w * w;
    }
    nbp = block_sum(nbp, red);
    if (tid == 0) v.qg_part[cta] = nbp;
    gsync();
    // G: ball scale from the CTA partials (fixed order), projection of the ball pair
    if (warp == 0) {
      double a = 0.0;
      for (int q = lane; q < G; q += 32) a += __ldcg(v.qg_part + q);
      a = warp_sum(a);
      if (lane == 0) bcast = a;
    }
    __syncthreads();
    {
      const double nb = sqrt(bcast);
      const double scl = (nb > rtr) ? rtr / nb : 1.0;
      for (int r = gtid; r < (T + 1) * nx; r += gnt) {
        const double zh = aq * sX[r] + (1.0 - aq) * zb[r];
        const double zn = scl * (zh + yb[r] * irq);
        yb[r] += rq * (zh - zn);
        zb[r] = zn;
      }
    }
    __syncthreads();
  }
  gsync();                                            // rows (p) of every CTA done
  // dual update + residuals of the outer iteration (per-CTA partials, fixed order)
  double ap = 0.0, ad = 0.0;
  for (int j = gtid; j < ng; j += gnt) {
    const double pj = __ldcg(p + j);
    const double dp = pj - pt[j];
    if (engine == NRTO_FULLADMM) {
      lam[j] += dp;
      v.tin[j] = pj + lam[j];
    } else {
      lam[j] += rho * dp;
    }
    ap += dp * dp;
    const double dd = pt[j] - v.ptprev[j];
    ad += dd * dd;
    v.ptprev[j] = pt[j];
  }
  ap = block_sum(ap, red);
  ad = block_sum(ad, red);
  if (tid == 0) { v.qg_part[cta] = ap; v.qg_part[1024 + cta] = ad; }
  gsync();
  if (cta == 0 && warp == 0) {
    double a1 = 0.0, a2 = 0.0;
    for (int q = lane; q < G; q += 32) { a1 += __ldcg(v.qg_part + q); a2 += __ldcg(v.qg_part + 1024 + q); }
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    if (lane == 0) {
      const double rpv = sqrt(a1), rdv = rho * sqrt(a2);
      v.r_p[b] = rpv;
      v.r_d[b] = rdv;
      record_hist(v, b, l, rpv, rdv, engine);
      v.iters[b] = l;
      if (!isfinite(rpv) || !isfinite(rdv)) {
        v.status[b] = NRTO_DIVERGED;
        v.active[b] = 0;
      } else if (!v.prm.fixed_iters && (l % v.prm.check_every) == 0 && rpv <= v.prm.eps_p &&
                 rdv <= v.prm.eps_d) {
        v.status[b] = NRTO_CONVERGED;
        v.active[b] = 0;
      }
    }
  }
}

int qp_grid_size(const nrto_handle_s* h) {
  const Dev& v = h->dev;
  if (!v.qpgrid) return 0;
  const size_t smem = qg_smem(v.d, v.scanM, v.scanC);
  if (smem > 220 * 1024) return 0;
  void* kern = (v.d.nx == 12 && v.d.nu == 4) ? (void*)k_qp_grid<12, 4>
             : (v.d.nx == 14 && v.d.nu == 7) ? (void*)k_qp_grid<14, 7> : (void*)k_qp_grid<0, 0>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 512, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    return 0;
  }
  const int G = std::min(v.nsm * occ, 1024);
  return G >= v.scanC ? G : 0;
}

static cudaError_t launch_qp_grid(nrto_handle_s* h, int engine, int l, cudaStream_t st) {
  const Dev& v = h->dev;
  cudaError_t e = cudaMemsetAsync(v.qg_bar, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(h->qp_grid);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = qg_smem(v.d, v.scanM, v.scanC);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (v.d.nx == 12 && v.d.nu == 4) e = cudaLaunchKernelEx(&cfg, k_qp_grid<12, 4>, v, engine, l);
  else if (v.d.nx == 14 && v.d.nu == 7) e = cudaLaunchKernelEx(&cfg, k_qp_grid<14, 7>, v, engine, l);
  else e = cudaLaunchKernelEx(&cfg, k_qp_grid<0, 0>, v, engine, l);
  h->launches++;
  return e;
}

// Chunked-scan QP usable for this launch (grid 0 / >= B: one CTA per instance):
// returns its staging mask (-1: not usable).
static int scan_stage(const nrto_handle_s* h, int grid) {
  const Dev& v = h->dev;
  static const int env = [] { const char* e = getenv("NRTO_QP_SCAN"); return e ? atoi(e) : 1; }();
  static const int menv = [] { const char* e = getenv("NRTO_QP_SCAN_STAGE"); return e ? atoi(e) : -1; }();
  if (!env || v.scanC <= 0 || v.qpgrid || !v.fa.PhiB || v.d.B > kScanMaxBatch) return -1;
  if (grid > 0 && grid < v.d.B) return -1;
  const size_t lim = 220 * 1024;
  if (scan_smem(v.d, v.scanC, 0) > lim) return -1;
  if (menv >= 0) return scan_smem(v.d, v.scanC, menv) <= lim ? menv : 0;
  // staged data up to ~120 KB: beyond that the L1 cache, which shares the 256 KB
  // with shared memory, serves the per-step constants better (c3: Acl alone is
  // 157 KB; measured 573 -> 522 us per FullADMM iteration unstaged)
  const size_t cap = std::max(scan_smem(v.d, v.scanC, 0), (size_t)120 * 1024);
  int mask = 0;
  const int order[kScanStageBits] = {0, 5, 1, 2, 3, 4};
  for (int q = 0; q < kScanStageBits; ++q) {
    const int b = order[q];
    if (b == 4 && v.scanM >= 8) continue;          // long chunks re-scan: no transfer matrices
    if (scan_smem(v.d, v.scanC, mask | (1 << b)) <= std::min(lim, cap)) mask |= 1 << b;
  }
  return mask;
}

static cudaError_t launch_qp_scan(nrto_handle_s* h, int engine, int l, int smask, cudaStream_t st) {
  const Dims& d = h->dev.d;
  const size_t smem = scan_smem(d, h->dev.scanC, smask);
  void* kern;
  if (d.nx == 14 && d.nu == 7) kern = (void*)k_qp_scan<14, 7>;
  else if (d.nx == 12 && d.nu == 4) kern = (void*)k_qp_scan<12, 4>;
  else if (d.nx == 3 && d.nu == 2) kern = (void*)k_qp_scan<3, 2>;
  else kern = (void*)k_qp_scan<0, 0>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (d.nx == 14 && d.nu == 7) k_qp_scan<14, 7><<<d.B, 512, smem, st>>>(h->dev, engine, l, smask);
  else if (d.nx == 12 && d.nu == 4) k_qp_scan<12, 4><<<d.B, 512, smem, st>>>(h->dev, engine, l, smask);
  else if (d.nx == 3 && d.nu == 2) k_qp_scan<3, 2><<<d.B, 512, smem, st>>>(h->dev, engine, l, smask);
  else k_qp_scan<0, 0><<<d.B, 512, smem, st>>>(h->dev, engine, l, smask);
  h->launches++;
  return cudaGetLastError();
}

// One CTA per instance (grid = B, all resident: in-order schedule) or a
// persistent grid looping over instances (overlapped schedule: one QP CTA per SM
// beside the cone pass, so the QP never holds more than that share of the SMs).
template <int NXM, int NUM, bool PIPE>
__global__ void __launch_bounds__(QP_THREADS, QP_MINB) k_qp_sparse(Dev v, int engine, int l) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  for (int b = blockIdx.x; b < v.d.B; b += gridDim.x) {
    qp_instance<NXM, NUM, PIPE>(v, engine, l, b, sm, red);
    __syncthreads();
  }
}

// Setup: compressed rows of the constraint gradients (state rows: n_x entries,
// control rows: the first n_u) as packed records {knot, kind | nz << 8, idx0..3,
// idx4..7} + values gval[row][8]; nnz > kRowNZ keeps the dense row (nz = 255).
__global__ void k_sparse_rows(Dev v) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)v.d.B * v.d.ng) return;
  const int j = (int)(id % v.d.ng);
  const int kind = v.kind[j];
  const int n = (kind == 0) ? v.d.nx : v.d.nu;
  const double* g = v.grad + id * v.d.nx;
  int nz = 0;
  for (int i = 0; i < n; ++i) nz += (g[i] != 0.0);
  uint32_t w0 = 0, w1 = 0;
  if (nz > kRowNZ) {
    nz = 255;
  } else {
    int s = 0;
    for (int i = 0; i < n; ++i)
      if (g[i] != 0.0) {
        v.gval[id * kRowNZ + s] = g[i];
        if (s < 4) w0 |= (uint32_t)i << (8 * s); else w1 |= (uint32_t)i << (8 * (s - 4));
        ++s;
      }
    for (; s < kRowNZ; ++s) v.gval[id * kRowNZ + s] = 0.0;
  }
  v.rowpk[id] = make_int4(v.knot[j], kind | (nz << 8), (int)w0, (int)w1);
}

// Setup: c_u,k = -2 R_u,k u_hat_k, the constant part of the QP's r_u (it does not
// change across QP iterations or outer iterations of one setup).
__global__ void k_qp_cu(Dev v) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nu = v.d.nu;
  if (id >= (int64_t)v.d.B * v.d.T * nu) return;
  const int64_t bk = id / nu;
  const int m = (int)(id % nu);
  const double* Rm = v.Ru + (bk * nu + m) * nu;
  const double* uk = v.uhat + bk * nu;
  double ru = 0.0;
  for (int q = 0; q < nu; ++q) ru += Rm[q] * uk[q];
  v.cu2[id] = -2.0 * ru;
}

cudaError_t launch_sparse_rows(nrto_handle_s* h, cudaStream_t st) {
  {
    const int64_t m = (int64_t)h->dev.d.B * h->dev.d.T * h->dev.d.nu;
    if (m > 0) { k_qp_cu<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(h->dev); h->launches++; }
  }
  const int64_t n = (int64_t)h->dev.d.B * h->dev.d.ng;
  if (n > 0) {
    k_sparse_rows<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(h->dev);
    h->launches++;
  }
  return cudaGetLastError();
}

bool fa_small_ok(const nrto_handle_s* h) {
  const Dev& v = h->dev;
  static const int env = [] { const char* e = getenv("NRTO_FA_SMALL"); return e ? atoi(e) : 1; }();
  if (!env || v.fused != 0 || v.d.B > kScanMaxBatch || v.d.nx > 32) return false;
  const int sm = scan_stage(h, 0);
  if (sm < 0) return false;
  return std::max(scan_smem(v.d, v.scanC, sm), (size_t)16 * 3 * v.d.nu * v.d.nx * sizeof(double)) <= 220 * 1024;
}

cudaError_t launch_fa_small(nrto_handle_s* h, int L, cudaStream_t st) {
  const Dims& d = h->dev.d;
  const int smask = scan_stage(h, 0);
  const size_t smem = std::max(scan_smem(d, h->dev.scanC, smask), (size_t)16 * 3 * d.nu * d.nx * sizeof(double));
  void* kern = (d.nx == 3 && d.nu == 2) ? (void*)k_fa_small<3, 2> : (void*)k_fa_small<0, 0>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (d.nx == 3 && d.nu == 2) k_fa_small<3, 2><<<d.B, 512, smem, st>>>(h->dev, L, smask);
  else k_fa_small<0, 0><<<d.B, 512, smem, st>>>(h->dev, L, smask);
  h->launches++;
  return cudaGetLastError();
}

cudaError_t launch_qp_sparse(nrto_handle_s* h, int engine, int l, cudaStream_t st, int grid) {
  const Dims& d = h->dev.d;
  if (h->dev.qpgrid && (grid == 0 || grid >= d.B)) return launch_qp_grid(h, engine, l, st);
  { const int sa = scan_stage(h, grid); if (sa >= 0) return launch_qp_scan(h, engine, l, sa, st); }
  const size_t smem = ((size_t)(d.T + 1) * d.nx + (size_t)kQPRing * d.nx * d.nx + kQPRing) * sizeof(double) +
                      (size_t)6 * (d.T + 1) * sizeof(int16_t);
  if (smem > 48 * 1024 || h->dev.prm.qp_iters > 32000) return launch_qp(h, engine, l, st);
  if (d.nx <= 127) {
    const int g = (grid > 0 && grid < d.B) ? grid : d.B;
    // warp-specialised pipelined iteration (PIPE) or the phase-synchronous one with
    // the bulk-copy recurrence ring; NRTO_QP_PIPE: 0 never, 1 always, 2 (default) only
    // for in-order launches (one CTA per instance) -- beside the cone pass the pipelined
    // variant's spinning helper warps take issue slots from the pass
    static const int pipe_env = [] { const char* e = getenv("NRTO_QP_PIPE"); return e ? atoi(e) : 2; }();
    const bool pipe = pipe_env == 1 || (pipe_env == 2 && g >= d.B);
    if (d.nx == 14 && d.nu == 7) {
      if (pipe) k_qp_sparse<14, 7, true><<<g, QP_THREADS, smem, st>>>(h->dev, engine, l);
      else k_qp_sparse<14, 7, false><<<g, QP_THREADS, smem, st>>>(h->dev, engine, l);
    } else if (d.nx == 12 && d.nu == 4) {
      if (pipe) k_qp_sparse<12, 4, true><<<g, QP_THREADS, smem, st>>>(h->dev, engine, l);
      else k_qp_sparse<12, 4, false><<<g, QP_THREADS, smem, st>>>(h->dev, engine, l);
    } else {
      k_qp_sparse<0, 0, false><<<g, QP_THREADS, smem, st>>>(h->dev, engine, l);
    }
    h->launches++;
    return cudaGetLastError();
  }
  return launch_qp(h, engine, l, st);
}

static size_t qp_smem(const Dims& d, int stageA) {
  return ((size_t)(d.T + 1) * d.nx + (size_t)d.T * d.nx + 2 * (size_t)d.T * d.nu +
          (stageA ? (size_t)d.T * d.nx * d.nx : 0)) * sizeof(double);
}

cudaError_t launch_qp(nrto_handle_s* h, int engine, int l, cudaStream_t st) {
  const Dims& d = h->dev.d;
  if (h->dev.qpgrid) return launch_qp_grid(h, engine, l, st);
  { const int sa = scan_stage(h, 0); if (sa >= 0) return launch_qp_scan(h, engine, l, sa, st); }
  const size_t lim = 200 * 1024;
  int stageA = qp_smem(d, 1) <= lim;
  if (stageA || qp_smem(d, 0) <= lim) {
    const size_t smem = qp_smem(d, stageA);
    cudaFuncSetAttribute(k_qp_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // threads: enough for the widest phase (rows, (T+1) n_x state entries), at most
    // 1024 -- tiny instances (c1) synchronise 2 warps instead of 32 per phase
    int nth = std::max(d.ng, (d.T + 1) * d.nx);
    nth = std::min(1024, std::max(64, (nth + 31) / 32 * 32));
    k_qp_staged<<<d.B, nth, smem, st>>>(h->dev, engine, l, stageA);
  } else {
    k_qp<<<d.B, 128, 0, st>>>(h->dev, engine, l);
  }
  h->launches++;
  return cudaGetLastError();
}

__global__ void k_reset_inst(Dev v, int engine) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= v.d.B) return;
  v.status[b] = NRTO_MAX_ITERS;
  v.iters[b] = 0;
  v.active[b] = 1;
  v.dr_active[b] = 1;
  v.r_p[b] = INFINITY;
  v.r_d[b] = INFINITY;
  v.rdr[b] = INFINITY;
}

__global__ void k_dr_arm(Dev v) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < v.d.B) v.dr_active[b] = v.active[b];
  if (b == 0 && v.drbar) *v.drbar = 0ULL;    // grid barrier of the persistent DR loop
}

static cudaError_t zero(nrto_handle_s* h, double* p, int64_t n, cudaStream_t st) {
  return cudaMemsetAsync(p, 0, n * sizeof(double), st);
}

cudaError_t launch_fa_reset(nrto_handle_s* h, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  const int64_t B = d.B;
  // TMA path: every y^1 block is written before it is read (no history at l = 1),
  // so the B E-double state array is not cleared (8.7 GB at the bench batch)
  // (max_iter = 0 runs no pass: the outputs nu / lam_nu are then built from Y = 0)
  if (v.fused != 2 || v.prm.max_iter == 0) zero(h, v.Y, B * d.E, st);
  zero(h, v.s, B * d.ng, st); zero(h, v.tin, B * d.ng, st); zero(h, v.pt, B * d.ng, st);
  zero(h, v.ptprev, B * d.ng, st); zero(h, v.p, B * d.ng, st); zero(h, v.lamp, B * d.ng, st);
  zero(h, v.K, B * d.NK, st);
  zero(h, v.Ccur, B * d.T * d.nx * d.nu, st); zero(h, v.Cprev, B * d.T * d.nx * d.nu, st);
  zero(h, v.D, B * d.T * d.nx * d.nu, st);
  zero(h, v.du, B * d.T * d.nu, st); zero(h, v.zl, B * d.ng, st); zero(h, v.yl, B * d.ng, st);
  zero(h, v.zb, B * (d.T + 1) * d.nx, st); zero(h, v.yb, B * (d.T + 1) * d.nx, st);
  cudaMemsetAsync(v.ncorr, 0, B * sizeof(int32_t), st);
  if (v.fused == 2) {
    cudaMemcpyAsync(v.G, v.G0, B * d.T * d.nu * d.nu * sizeof(double), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(v.H, v.H0, B * d.T * d.nu * d.nx * sizeof(double), cudaMemcpyDeviceToDevice, st);
  }
  k_reset_inst<<<(d.B + 127) / 128, 128, 0, st>>>(v, NRTO_FULLADMM);
  h->launches++;
  h->dr_fresh = 1;   // Y / Z now hold FullADMM state
  return cudaGetLastError();
}

cudaError_t launch_dr_reset(nrto_handle_s* h, int full, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  const int64_t B = d.B;
  if (full) {          // DR warm state (chi~, s~) and Z = adjoint(eta~ = 0)
    zero(h, v.Y, B * d.E, st); zero(h, v.tt, B * d.ng, st); zero(h, v.pit, B * d.ng, st);
    zero(h, v.Kt, B * d.NK, st); zero(h, v.Z, B * d.T * d.nu * d.nx, st);
  }
  zero(h, v.pt, B * d.ng, st); zero(h, v.ptprev, B * d.ng, st); zero(h, v.p, B * d.ng, st);
  zero(h, v.lamp, B * d.ng, st); zero(h, v.K, B * d.NK, st);
  zero(h, v.Ccur, B * d.T * d.nx * d.nu, st); zero(h, v.Cprev, B * d.T * d.nx * d.nu, st);
  zero(h, v.s, B * d.ng, st);
  zero(h, v.du, B * d.T * d.nu, st); zero(h, v.zl, B * d.ng, st); zero(h, v.yl, B * d.ng, st);
  zero(h, v.zb, B * (d.T + 1) * d.nx, st); zero(h, v.yb, B * (d.T + 1) * d.nx, st);
  k_reset_inst<<<(d.B + 127) / 128, 128, 0, st>>>(v, NRTO_DR);
  h->launches++;
  return cudaGetLastError();
}

cudaError_t launch_dr_arm(nrto_handle_s* h, cudaStream_t st) {
  k_dr_arm<<<(h->dev.d.B + 127) / 128, 128, 0, st>>>(h->dev);
  h->launches++;
  return cudaGetLastError();
}

}  // namespace nrto

extern "C" int nrto_debug_qp_clocks(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, nrto::g_qp_clk, sizeof(long long) * 64);
}
