// Setup kernels S0-S2: build the ragged SOC data, the per-step
// gain chains and the QP Riccati factors on the device.
#include "common.cuh"

namespace nrto {

__device__ int g_setup_err;   // 0 ok, 1 W' not SPD, 2 H_uu not SPD

// ---------------------------------------------------------------------------
// S0: costate sweep per cone.  State cone j at knot K:
//   c_{j,K} = grad_j,  b_{j,k} = B_k^T c_{j,k+1},  c_{j,k} = A_k^T c_{j,k+1},
//   b_hat_{j,k} = sqrt(tau) Psi_k c_{j,k}   (k = K..0).
// Control cone (R14): b_{j,k} = h'_j at its own step, b_hat = 0.
// One warp per (instance, cone); lane i holds c_i (n_x <= 32).
__global__ void k_costate(Dev v) {
  const Dims d = v.d;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gw >= (int64_t)d.B * d.ng) return;
  const int lane = threadIdx.x & 31;
  const int b = (int)(gw / d.ng), j = (int)(gw % d.ng);
  const int nx = d.nx, nu = d.nu;
  const double* grad = v.grad + ((int64_t)b * d.ng + j) * nx;
  double* bh = v.bhat + (int64_t)b * d.E + v.off[j];
  double* Bd = v.Bd + (int64_t)b * d.EB + v.offB[j];
  if (v.kind[j] != 0) {
    if (lane < d.nup) Bd[lane] = (lane < nu) ? grad[lane] : 0.0;
    if (lane < nx) bh[lane] = 0.0;
    return;
  }
  const int K = v.knot[j];
  const double st = sqrt(v.tau[b]);
  const double* A = v.A + (int64_t)b * d.T * nx * nx;
  const double* B = v.Bm + (int64_t)b * d.T * nx * nu;
  const double* Psi = v.Psi + (int64_t)b * (d.T + 1) * nx * nx;
  double c = (lane < nx) ? grad[lane] : 0.0;
  for (int k = K; k >= 0; --k) {
    if (k < K) {
      const double* Bk = B + (int64_t)k * nx * nu;
      const double* Ak = A + (int64_t)k * nx * nx;
      double bm = 0.0, cn = 0.0;
      for (int r = 0; r < nx; ++r) {
        const double cr = __shfl_sync(0xffffffffu, c, r);
        if (lane < nu) bm += Bk[r * nu + lane] * cr;   // (B_k^T c)_m
        if (lane < nx) cn += Ak[r * nx + lane] * cr;   // (A_k^T c)_i
      }
      if (lane < d.nup) Bd[k * d.nup + lane] = (lane < nu) ? bm : 0.0;
      c = cn;
    }
    const double* Pk = Psi + (int64_t)k * nx * nx;
    double bhv = 0.0;
    for (int r = 0; r < nx; ++r) {
      const double cr = __shfl_sync(0xffffffffu, c, r);
      if (lane < nx) bhv += Pk[lane * nx + r] * cr;
    }
    if (lane < nx) bh[k * nx + lane] = st * bhv;
  }
}

// S0b: Lambda_k = sum_j b_{j,k} b_{j,k}^T, Zb_k = sum_j b_{j,k} b_hat_{j,k}^T over
// the cones with a b-block at step k (fixed order -> deterministic).
__global__ void k_lam_zb(Dev v) {
  const Dims d = v.d;
  const int b = blockIdx.x / d.T, k = blockIdx.x % d.T;
  const int nx = d.nx, nu = d.nu;
  const int nout = nu * nu + nu * nx;
  const double* bhat = v.bhat + (int64_t)b * d.E;
  const double* Bd = v.Bd + (int64_t)b * d.EB;
  for (int o = threadIdx.x; o < nout; o += blockDim.x) {
    double acc = 0.0;
    const bool isLam = o < nu * nu;
    const int m = isLam ? o / nu : (o - nu * nu) / nx;
    const int q = isLam ? o % nu : (o - nu * nu) % nx;
    for (int c = v.kptr[k]; c < v.kptr[k + 1]; ++c) {
      const int j = v.kcone[c];
      const bool st = v.kind[j] == 0;
      const int kb = st ? k : 0;
      const double bm = Bd[v.offB[j] + kb * d.nup + m];
      if (isLam) acc += bm * Bd[v.offB[j] + kb * d.nup + q];
      else if (st) acc += bm * bhat[v.off[j] + kb * nx + q];
    }
    if (isLam) v.Lam[((int64_t)b * d.T + k) * nu * nu + o] = acc;
    else v.Zb[((int64_t)b * d.T + k) * nu * nx + (o - nu * nu)] = acc;
  }
}

// ---------------------------------------------------------------------------
// Cyclic Jacobi eigen-decomposition of a symmetric n x n matrix in shared
// memory, one warp: A <- diag(eigenvalues), V <- eigenvectors (columns).
__device__ void warp_jacobi(double* A, double* V, int n) {
  const int lane = threadIdx.x & 31;
  for (int r = lane; r < n * n; r += 32) V[r] = (r / n == r % n) ? 1.0 : 0.0;
  __syncwarp();
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int r = lane; r < n * n; r += 32) {
      const double a = A[r];
      if (r / n == r % n) dia += a * a; else off += a * a;
    }
    off = warp_sum(off); dia = warp_sum(dia);
    if (off <= 1e-30 * dia || off == 0.0) break;   // off-diagonal at 1e-15 of the diagonal
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (apq == 0.0) continue;
        const double app = A[p * n + p], aqq = A[q * n + q];
        const double th = (aqq - app) / (2.0 * apq);
        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        __syncwarp();
        if (lane < n) {                       // A <- A P (columns p, q)
          const double arp = A[lane * n + p], arq = A[lane * n + q];
          A[lane * n + p] = c * arp - s * arq;
          A[lane * n + q] = s * arp + c * arq;
          const double vrp = V[lane * n + p], vrq = V[lane * n + q];
          V[lane * n + p] = c * vrp - s * vrq;
          V[lane * n + q] = s * vrp + c * vrq;
        }
        __syncwarp();
        if (lane < n) {                       // A <- P^T A (rows p, q)
          const double apr = A[p * n + lane], aqr = A[q * n + lane];
          A[p * n + lane] = c * apr - s * aqr;
          A[q * n + lane] = s * apr + c * aqr;
        }
        __syncwarp();
      }
    }
  }
  __syncwarp();
}

// S1: per (instance, step k) gain chain of SURVEY F2.  The k-th diagonal block
// of Q_v + c sum_j A_hat_j^T A_hat_j is 2 (I (x) W'_k) + c tau
// (Sigma_k (x) Lambda_k) with Sigma_k = Psi_k^T Psi_k; its solve is the exact
// chain K = V [(V^T R U) ./ (2 + c tau sigma_a lambda_b)] U^T with
// Lambda V = W' V diag(sigma), V^T W' V = I, Sigma = U diag(lambda) U^T.
// Engine FullADMM: W' = W, c = rho.  DR (F3): W' = W + sigma_dr/2, c = r_s.
// psame[b][k] = (Psi_k bit-identical to Psi_{k-1}), one warp per (instance, step).
__global__ void k_psi_same(Dev v) {
  const Dims d = v.d;
  const int nn = d.nx * d.nx, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gw >= (int64_t)d.B * d.T) return;
  const int b = (int)(gw / d.T), k = (int)(gw % d.T);
  int same = k > 0;
  if (k > 0) {
    const double* Pk = v.Psi + ((int64_t)b * (d.T + 1) + k) * nn;
    for (int r = lane; r < nn; r += 32) same &= (Pk[r - nn] == Pk[r]);
  }
  same = __all_sync(0xffffffffu, same);
  if (lane == 0) v.psame[gw] = same;
}

__global__ void k_chain(Dev v) {
  extern __shared__ double sm[];
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu;
  const int wpb = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int per = 2 * nx * nx + 4 * nu * nu + nx + nu;
  double* S = sm + (threadIdx.x >> 5) * per;
  double* Uq = S + nx * nx;
  double* M = Uq + nx * nx;
  double* Q = M + nu * nu;
  double* L = Q + nu * nu;
  double* Li = L + nu * nu;
  double* lam = Li + nu * nu;
  double* sig = lam + nx;
  if (gw >= (int64_t)d.B * d.T) return;
  const int b = (int)(gw / d.T), k = (int)(gw % d.T);
  const int64_t bk = (int64_t)b * d.T + k;
  const double* Pk = v.Psi + ((int64_t)b * (d.T + 1) + k) * nx * nx;
  // Sigma_k depends on Psi_k only: the warp for the first step of a run of
  // bit-identical Psi blocks (S = blkdiag(S_0, S_d, ..., S_d)) does the
  // eigen-decomposition; the others wait for it in k_chain_copy.
  int k0 = k;                                   // start of the run (k_psi_same flags)
  while (k0 > 0 && v.psame[(int64_t)b * d.T + k0]) --k0;
  v.Urep[bk] = k0;
  if (k0 == k) {
    for (int r = lane; r < nx * nx; r += 32) {   // Sigma = Psi^T Psi
      const int i = r / nx, c = r % nx;
      double acc = 0.0;
      for (int q = 0; q < nx; ++q) acc += Pk[q * nx + i] * Pk[q * nx + c];
      S[r] = acc;
    }
    __syncwarp();
    warp_jacobi(S, Uq, nx);
    for (int r = lane; r < nx; r += 32) v.Ulam[bk * nx + r] = S[r * nx + r];
    for (int r = lane; r < nx * nx; r += 32) v.U[bk * nx * nx + r] = Uq[r];
  }
  __syncwarp();
}

// S1b: generalized eigen-chain of (Lambda_k, W'_k) per engine, with the
// Sigma_k eigenpairs of step Urep[k] (identical Psi blocks share them).
__global__ void k_chain2(Dev v, int engmask) {
  extern __shared__ double sm[];
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu;
  const int wpb = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int per = 4 * nu * nu + nx + nu;
  double* M = sm + (threadIdx.x >> 5) * per;
  double* Q = M + nu * nu;
  double* L = Q + nu * nu;
  double* Li = L + nu * nu;
  double* lam = Li + nu * nu;
  double* sig = lam + nx;
  if (gw >= (int64_t)d.B * d.T) return;
  const int b = (int)(gw / d.T), k = (int)(gw % d.T);
  const int64_t bk = (int64_t)b * d.T + k;
  const int64_t bk0 = (int64_t)b * d.T + v.Urep[bk];
  if (bk0 != bk)
    for (int r = lane; r < nx * nx; r += 32) v.U[bk * nx * nx + r] = v.U[bk0 * nx * nx + r];
  for (int r = lane; r < nx; r += 32) lam[r] = v.Ulam[bk0 * nx + r];
  __syncwarp();
  const double tau = v.tau[b];
  for (int eng = 0; eng < 2; ++eng) {
    if (!((engmask >> eng) & 1)) continue;
    const EngineFactors& F = eng == 0 ? v.fa : v.dr;
    const double shift = eng == 0 ? 0.0 : 0.5 * v.prm.sigma_dr;
    const double coef = eng == 0 ? v.prm.rho : v.prm.r_s;
    const double* Wk = v.W + bk * nu * nu;
    if (lane == 0) {                           // Cholesky W' = L L^T, then L^{-1}
      for (int r = 0; r < nu * nu; ++r) L[r] = 0.0;
      for (int c = 0; c < nu; ++c) {
        double dg = Wk[c * nu + c] + shift;
        for (int q = 0; q < c; ++q) dg -= L[c * nu + q] * L[c * nu + q];
        if (!(dg > 0.0)) { atomicExch(&g_setup_err, 1); dg = 1.0; }
        const double lc = sqrt(dg);
        L[c * nu + c] = lc;
        for (int r = c + 1; r < nu; ++r) {
          double a = Wk[r * nu + c];
          for (int q = 0; q < c; ++q) a -= L[r * nu + q] * L[c * nu + q];
          L[r * nu + c] = a / lc;
        }
      }
      for (int r = 0; r < nu * nu; ++r) Li[r] = 0.0;
      for (int c = 0; c < nu; ++c) {           // forward substitution L Li = I
        for (int r = c; r < nu; ++r) {
          double a = (r == c) ? 1.0 : 0.0;
          for (int q = c; q < r; ++q) a -= L[r * nu + q] * Li[q * nu + c];
          Li[r * nu + c] = a / L[r * nu + r];
        }
      }
    }
    __syncwarp();
    const double* Lk = v.Lam + bk * nu * nu;
    for (int r = lane; r < nu * nu; r += 32) {   // Q := Li Lambda
      const int i = r / nu, c = r % nu;
      double acc = 0.0;
      for (int q = 0; q < nu; ++q) acc += Li[i * nu + q] * Lk[q * nu + c];
      Q[r] = acc;
    }
    __syncwarp();
    for (int r = lane; r < nu * nu; r += 32) {   // M := (Li Lambda) Li^T
      const int i = r / nu, c = r % nu;
      double acc = 0.0;
      for (int q = 0; q < nu; ++q) acc += Q[i * nu + q] * Li[c * nu + q];
      M[r] = acc;
    }
    __syncwarp();
    for (int r = lane; r < nu * nu; r += 32) {   // symmetrise
      const int i = r / nu, c = r % nu;
      if (i < c) { const double a = 0.5 * (M[r] + M[c * nu + i]); M[r] = a; M[c * nu + i] = a; }
    }
    __syncwarp();
    warp_jacobi(M, Q, nu);
    for (int r = lane; r < nu; r += 32) sig[r] = M[r * nu + r];
    __syncwarp();
    for (int r = lane; r < nu * nu; r += 32) {   // V = L^{-T} Q
      const int i = r / nu, c = r % nu;
      double acc = 0.0;
      for (int q = 0; q < nu; ++q) acc += Li[q * nu + i] * Q[q * nu + c];
      F.V[bk * nu * nu + r] = acc;
    }
    for (int r = lane; r < nu * nx; r += 32) {
      const int a = r / nx, c = r % nx;
      F.den[bk * nu * nx + r] = 1.0 / (2.0 + coef * tau * sig[a] * lam[c]);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// S2: Riccati factorisation of the QP x-step (DESIGN R1):
//   P_T = Qt_T;  H_uu = Rt_k + B^T P B;  H_ux = B^T P A;  Kf = H_uu^{-1} H_ux;
//   P_k = Qt_k + A^T P A - H_ux^T Kf   (k = T-1..1)
// with Qt_k = rho_q I + c sum_{state j@k} g g^T, Rt_k = 2 R_u + sigma_q I +
// c sum_{ctrl j@k} h h^T, c = rho_q (rho+sigma_q)/(rho+sigma_q+rho_q).
// One CTA per (instance, engine).
__global__ void k_riccati(Dev v, int eng) {
  extern __shared__ double sm[];
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu;
  const int b = blockIdx.x;
  const EngineFactors& F = eng == 0 ? v.fa : v.dr;
  const double rho = eng == 0 ? v.prm.rho : v.prm.rho_admm;
  const double rq = v.prm.rho_qp, sq = v.prm.sigma_qp;
  const double cc = rq * (rho + sq) / (rho + sq + rq);
  double* P = sm;                 // nx*nx
  double* PA = P + nx * nx;       // nx*nx
  double* PB = PA + nx * nx;      // nx*nu
  double* Huu = PB + nx * nu;     // nu*nu
  double* Hux = Huu + nu * nu;    // nu*nx
  double* Hi = Hux + nu * nx;     // nu*nu
  double* L = Hi + nu * nu;       // nu*nu
  double* Kf = L + nu * nu;       // nu*nx
  const int tid = threadIdx.x, nt = blockDim.x;
  const double* grad = v.grad + (int64_t)b * d.ng * nx;
  // P = Qt_T
  for (int r = tid; r < nx * nx; r += nt) {
    const int i = r / nx, c = r % nx;
    double acc = (i == c) ? rq : 0.0;
    for (int q = v.sptr[d.T]; q < v.sptr[d.T + 1]; ++q) {
      const int j = v.srow[q];
      acc += cc * grad[j * nx + i] * grad[j * nx + c];
    }
    P[r] = acc;
  }
  __syncthreads();
  for (int k = d.T - 1; k >= 0; --k) {
    const double* A = v.A + ((int64_t)b * d.T + k) * nx * nx;
    const double* B = v.Bm + ((int64_t)b * d.T + k) * nx * nu;
    const double* Ru = v.Ru + ((int64_t)b * d.T + k) * nu * nu;
    for (int r = tid; r < nx * nx; r += nt) {       // PA = P A
      const int i = r / nx, c = r % nx;
      double acc = 0.0;
      for (int q = 0; q < nx; ++q) acc += P[i * nx + q] * A[q * nx + c];
      PA[r] = acc;
    }
    for (int r = tid; r < nx * nu; r += nt) {       // PB = P B
      const int i = r / nu, c = r % nu;
      double acc = 0.0;
      for (int q = 0; q < nx; ++q) acc += P[i * nx + q] * B[q * nu + c];
      PB[r] = acc;
    }
    __syncthreads();
    for (int r = tid; r < nu * nu; r += nt) {       // Huu = Rt + B^T P B
      const int i = r / nu, c = r % nu;
      double acc = 2.0 * Ru[r] + ((i == c) ? sq : 0.0);
      for (int q = v.cptr[k]; q < v.cptr[k + 1]; ++q) {
        const int j = v.crow[q];
        acc += cc * grad[j * nx + i] * grad[j * nx + c];
      }
      for (int q = 0; q < nx; ++q) acc += B[q * nu + i] * PB[q * nu + c];
      Huu[r] = acc;
    }
    for (int r = tid; r < nu * nx; r += nt) {       // Hux = B^T P A
      const int i = r / nx, c = r % nx;
      double acc = 0.0;
      for (int q = 0; q < nx; ++q) acc += B[q * nu + i] * PA[q * nx + c];
      Hux[r] = acc;
    }
    __syncthreads();
    if (tid == 0) {                                 // Huu^{-1} via Cholesky
      for (int r = 0; r < nu * nu; ++r) L[r] = 0.0;
      for (int c = 0; c < nu; ++c) {
        double dg = 0.5 * (Huu[c * nu + c] + Huu[c * nu + c]);
        for (int q = 0; q < c; ++q) dg -= L[c * nu + q] * L[c * nu + q];
        if (!(dg > 0.0)) { atomicExch(&g_setup_err, 2); dg = 1.0; }
        const double lc = sqrt(dg);
        L[c * nu + c] = lc;
        for (int r = c + 1; r < nu; ++r) {
          double a = 0.5 * (Huu[r * nu + c] + Huu[c * nu + r]);
          for (int q = 0; q < c; ++q) a -= L[r * nu + q] * L[c * nu + q];
          L[r * nu + c] = a / lc;
        }
      }
      for (int c = 0; c < nu; ++c) {               // solve L L^T x = e_c
        double* x = Hi + c * nu;                    // column c stored as row c (symmetric)
        for (int r = 0; r < nu; ++r) {
          double a = (r == c) ? 1.0 : 0.0;
          for (int q = 0; q < r; ++q) a -= L[r * nu + q] * x[q];
          x[r] = a / L[r * nu + r];
        }
        for (int r = nu - 1; r >= 0; --r) {
          double a = x[r];
          for (int q = r + 1; q < nu; ++q) a -= L[q * nu + r] * x[q];
          x[r] = a / L[r * nu + r];
        }
      }
    }
    __syncthreads();
    const int64_t bk = (int64_t)b * d.T + k;
    for (int r = tid; r < nu * nx; r += nt) {       // Kf = Hi Hux ; HB = Hi B^T
      const int i = r / nx, c = r % nx;
      double acc = 0.0, hb = 0.0;
      for (int q = 0; q < nu; ++q) {
        acc += Hi[i * nu + q] * Hux[q * nx + c];
        hb += Hi[i * nu + q] * B[c * nu + q];
      }
      Kf[r] = acc;
      F.Kf[bk * nu * nx + r] = acc;
      F.HB[bk * nu * nx + r] = hb;
    }
    for (int r = tid; r < nu * nu; r += nt) F.Hinv[bk * nu * nu + r] = Hi[r];
    __syncthreads();
    for (int r = tid; r < nx * nx; r += nt) {       // Acl = A - B Kf
      const int i = r / nx, c = r % nx;
      double acc = A[r];
      for (int q = 0; q < nu; ++q) acc -= B[i * nu + q] * Kf[q * nx + c];
      F.Acl[bk * nx * nx + r] = acc;
      F.AclT[bk * nx * nx + c * nx + i] = acc;
    }
    if (k >= 1) {                                   // P = Qt_k + A^T P A - Hux^T Kf
      __syncthreads();
      for (int r = tid; r < nx * nx; r += nt) {
        const int i = r / nx, c = r % nx;
        double acc = (i == c) ? rq : 0.0;
        for (int q = v.sptr[k]; q < v.sptr[k + 1]; ++q) {
          const int j = v.srow[q];
          acc += cc * grad[j * nx + i] * grad[j * nx + c];
        }
        for (int q = 0; q < nx; ++q) acc += A[q * nx + i] * PA[q * nx + c];
        for (int q = 0; q < nu; ++q) acc -= Hux[q * nx + i] * Kf[q * nx + c];
        P[r] = acc;                                  // PA / Kf not read after this
      }
      __syncthreads();
      for (int r = tid; r < nx * nx; r += nt) {     // symmetrise
        const int i = r / nx, c = r % nx;
        if (i < c) { const double a = 0.5 * (P[r] + P[c * nx + i]); P[r] = a; P[c * nx + i] = a; }
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_setup(nrto_handle_s* h, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  int zero = 0;
  cudaMemcpyToSymbolAsync(g_setup_err, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, st);
  if (d.nx <= 16 && d.nu <= 8) {              // tensor-core S0 / S0b
    cudaError_t e = launch_setup_mma(h, st);
    if (e != cudaSuccess) return e;
  } else {
    if ((int64_t)d.B * d.ng > 0) {
      const int64_t warps = (int64_t)d.B * d.ng;
      k_costate<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(v);
      h->launches++;
    }
    k_lam_zb<<<d.B * d.T, 128, 0, st>>>(v);
    h->launches++;
  }
  const int per = 2 * d.nx * d.nx + 4 * d.nu * d.nu + d.nx + d.nu;
  const int wpb = 4;
  const int64_t nw = (int64_t)d.B * d.T;
  k_psi_same<<<(unsigned)((nw + 7) / 8), 256, 0, st>>>(v);
  h->launches++;
  k_chain<<<(unsigned)((nw + wpb - 1) / wpb), 32 * wpb, wpb * per * sizeof(double), st>>>(v);
  h->launches++;
  h->dr_ready = 0;
  cudaError_t e = launch_sparse_rows(h, st);
  if (e != cudaSuccess) return e;
  return launch_engine_factors(h, NRTO_FULLADMM, st);
}

// Per-engine S1b/S2 factors: FullADMM at setup, DR lazily on its first solve.
cudaError_t launch_engine_factors(nrto_handle_s* h, int engine, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  if (engine != NRTO_FULLADMM) {       // fresh error flag for the lazily built DR factors
    int zero = 0;
    cudaMemcpyToSymbolAsync(g_setup_err, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, st);
  }
  const int wpb = 4;
  const int64_t nw = (int64_t)d.B * d.T;
  k_chain2<<<(unsigned)((nw + wpb - 1) / wpb), 32 * wpb,
             wpb * (4 * d.nu * d.nu + d.nx + d.nu) * sizeof(double), st>>>(v, 1 << engine);
  h->launches++;
  const int rs = 3 * d.nx * d.nx + 2 * d.nx * d.nu + 3 * d.nu * d.nu + 2 * d.nu * d.nx;
  k_riccati<<<d.B, 128, rs * sizeof(double), st>>>(v, engine);
  h->launches++;
  if (v.scanC > 0) return launch_scan_factors(h, engine, st);
  return cudaGetLastError();
}

int read_setup_error(cudaStream_t st) {
  int e = 0;
  cudaMemcpyFromSymbolAsync(&e, g_setup_err, sizeof(int), 0, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return e;
}

}  // namespace nrto
