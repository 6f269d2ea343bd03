// General uncertainty set: zeta = Gamma z, z^T S z <= tau with
// Gamma in R^{(T+1) n_x x n_z} and a dense S.  Then
//   A_hat_j k_v + b_hat_j = W (A_bar_j k_v + c_j),   W = sqrt(tau) Psi Gamma^T  (n_z x NX),
// with the RAW ragged vectors v_j = [K_k^T b_{j,k} + c_{j,k}]_k (c_{j,k} = Phi(k_j,k)^T grad g_j,
// F1 without Psi), so every cone row is a dense n_z vector and the gain system
//   M^{-1} = Q_v + rho sum_j A_hat_j^T A_hat_j,
//   (sum_j A_hat_j^T A_hat_j)[(k,i,m),(k',i',m')] = G[(k,i),(k',i')] Lam[(k,m),(k',m')],
//   G = W^T W,  Lam = sum_j b_bar_j b_bar_j^T  (b_bar_j = [b_{j,0}; ...; b_{j,T-1}]),
// couples every time step (no F2 block structure).  This path forms M^{-1} densely and
// factors it once per setup (Cholesky, own kernel); per FullADMM iteration it runs
//   forward:  V (ragged -> dense rows) ; a = V W^T          (GEMM n_g x NX x n_z)
//   Block-1:  lam += a - nu (pending (16) of l-1) ; y = a + lam ; SOC projection (13)
//   Block-2:  the QP (14a) kernels of the block-diagonal path (they do not see Psi, Gamma)
//   (14b):    U = (nu - b_hat) W (GEMM n_g x n_z x NX) ; rhs = Q_v k + rho A_bar^T U ;
//             k = M rhs by the Cholesky factor
// The block-diagonal machinery (costate sweeps, b_{j,k}, QP Riccati factors) is reused by
// running the regular setup with Psi_k = I and tau = 1, which makes its ragged "b_hat"
// array the raw costates c_{j,k}.
#include "common.cuh"
#include <algorithm>
#include <cmath>

namespace nrto {

__device__ int g_gen_err;   // 1: Cholesky pivot <= 0 (M^{-1} not SPD)

// C[b] (M x N) = alpha * A[b] (M x K) * op(B[b]);  op = B^T (B is N x K, TB = 1) or
// B (K x N, TB = 0).  Row-major, leading dims = row lengths.  16 x 16 tiles, FP64 FMA.
template <int TB>
__global__ void k_dgemm(const double* __restrict__ A, const double* __restrict__ B, double* C,
                        int M, int N, int K, int64_t sA, int64_t sB, int64_t sC, double alpha) {
  __shared__ double As[16][17], Bs[16][17];
  const int b = blockIdx.z;
  const double* Ab = A + b * sA;
  const double* Bb = B + b * sB;
  const int r = blockIdx.y * 16 + threadIdx.y, c = blockIdx.x * 16 + threadIdx.x;
  double acc = 0.0;
  for (int k0 = 0; k0 < K; k0 += 16) {
    const int ka = k0 + threadIdx.x, kb = k0 + threadIdx.y;
    As[threadIdx.y][threadIdx.x] = (r < M && ka < K) ? Ab[(int64_t)r * K + ka] : 0.0;
    const int cb = blockIdx.x * 16 + threadIdx.x;
    if (TB) Bs[threadIdx.y][threadIdx.x] = (cb < N && kb < K) ? Bb[(int64_t)cb * K + kb] : 0.0;
    else Bs[threadIdx.y][threadIdx.x] = (cb < N && kb < K) ? Bb[(int64_t)kb * N + cb] : 0.0;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = fma(As[threadIdx.y][q], Bs[q][threadIdx.x], acc);
    __syncthreads();
  }
  if (r < M && c < N) C[b * sC + (int64_t)r * N + c] = alpha * acc;
}

// C[b] (M x N) = A[b]^T (A: K x M) * B[b] (K x N)
__global__ void k_dgemm_tn(const double* __restrict__ A, const double* __restrict__ B, double* C,
                           int M, int N, int K, int64_t sA, int64_t sB, int64_t sC) {
  __shared__ double As[16][17], Bs[16][17];
  const int b = blockIdx.z;
  const double* Ab = A + b * sA;
  const double* Bb = B + b * sB;
  const int r = blockIdx.y * 16 + threadIdx.y, c = blockIdx.x * 16 + threadIdx.x;
  double acc = 0.0;
  for (int k0 = 0; k0 < K; k0 += 16) {
    const int ka = k0 + threadIdx.x, kb = k0 + threadIdx.y;
    const int ra = blockIdx.y * 16 + threadIdx.y;
    As[threadIdx.y][threadIdx.x] = (ra < M && ka < K) ? Ab[(int64_t)ka * M + ra] : 0.0;
    Bs[threadIdx.y][threadIdx.x] = (c < N && kb < K) ? Bb[(int64_t)kb * N + c] : 0.0;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = fma(As[threadIdx.y][q], Bs[q][threadIdx.x], acc);
    __syncthreads();
  }
  if (r < M && c < N) C[b * sC + (int64_t)r * N + c] = acc;
}

static cudaError_t dgemm(int tb, const double* A, const double* B, double* C, int M, int N, int K,
                         int64_t sA, int64_t sB, int64_t sC, int batch, double alpha, cudaStream_t st) {
  if (M <= 0 || N <= 0 || batch <= 0) return cudaSuccess;
  dim3 grid((N + 15) / 16, (M + 15) / 16, batch), blk(16, 16);
  if (tb) k_dgemm<1><<<grid, blk, 0, st>>>(A, B, C, M, N, K, sA, sB, sC, alpha);
  else k_dgemm<0><<<grid, blk, 0, st>>>(A, B, C, M, N, K, sA, sB, sC, alpha);
  return cudaGetLastError();
}

// Dense rows of the raw costates c_j (NX, zero tail) and of b_bar_j (T n_u, zero tail)
// from the ragged arrays of the regular setup (Psi = I, tau = 1: bhat = c, Bd = b).
__global__ void k_gen_expand(Dev v, double* Cf, double* Bf) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const Dims d = v.d;
  const int NX = (d.T + 1) * d.nx, NU = d.T * d.nu;
  if (id >= (int64_t)d.B * d.ng) return;
  const int b = (int)(id / d.ng), j = (int)(id % d.ng);
  const int kj = v.knot[j];
  double* cr = Cf + id * NX;
  double* br = Bf + id * NU;
  for (int x = 0; x < NX; ++x) cr[x] = 0.0;
  for (int x = 0; x < NU; ++x) br[x] = 0.0;
  const double* bh = v.bhat + (int64_t)b * d.E + v.off[j];
  const double* bd = v.Bd + (int64_t)b * d.EB + v.offB[j];
  if (v.kind[j] == 0) {
    for (int x = 0; x < (kj + 1) * d.nx; ++x) cr[x] = bh[x];
    for (int k = 0; k < kj; ++k)
      for (int m = 0; m < d.nu; ++m) br[k * d.nu + m] = bd[k * d.nup + m];
  } else {
    for (int m = 0; m < d.nu; ++m) br[kj * d.nu + m] = bd[m];
  }
}

// M^{-1}[(k,i,m),(k',i',m')] = rho G[(k,i),(k',i')] Lam[(k,m),(k',m')] + [k=k', i=i'] 2 W_k[m][m']
__global__ void k_gen_minv(Dev v, const double* G, const double* Lam, double* Mi, double rho) {
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, NK = d.NK, NX = (d.T + 1) * nx, NU = d.T * nu;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)d.B * NK * NK) return;
  const int b = (int)(id / ((int64_t)NK * NK));
  const int64_t rc = id % ((int64_t)NK * NK);
  const int r = (int)(rc / NK), c = (int)(rc % NK);
  const int k = r / (nx * nu), i = (r % (nx * nu)) / nu, m = r % nu;
  const int k2 = c / (nx * nu), i2 = (c % (nx * nu)) / nu, m2 = c % nu;
  double val = rho * G[(int64_t)b * NX * NX + (int64_t)(k * nx + i) * NX + (k2 * nx + i2)] *
               Lam[(int64_t)b * NU * NU + (int64_t)(k * nu + m) * NU + (k2 * nu + m2)];
  if (k == k2 && i == i2) val += 2.0 * v.W[((int64_t)b * d.T + k) * nu * nu + m * nu + m2];
  Mi[id] = val;
}

// In-place lower Cholesky of one NK x NK matrix per CTA (right-looking, column by column).
__global__ void k_gen_chol(double* Mi, int n) {
  double* A = Mi + (int64_t)blockIdx.x * n * n;
  __shared__ double piv;
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      const double djj = A[(int64_t)j * n + j];
      if (!(djj > 0.0)) g_gen_err = 1;
      piv = sqrt(fmax(djj, 1e-300));
      A[(int64_t)j * n + j] = piv;
    }
    __syncthreads();
    const double p = piv;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) A[(int64_t)i * n + j] /= p;
    __syncthreads();
    // trailing update of the lower triangle: A[i][c] -= L[i][j] L[c][j], j < c <= i
    const int64_t m = n - j - 1;
    for (int64_t t = threadIdx.x; t < m * (m + 1) / 2; t += blockDim.x) {
      // t -> (ii, cc) with 0 <= cc <= ii < m
      const int64_t ii = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
      int64_t i0 = ii;
      while (i0 * (i0 + 1) / 2 > t) --i0;
      while ((i0 + 1) * (i0 + 2) / 2 <= t) ++i0;
      const int64_t cc = t - i0 * (i0 + 1) / 2;
      const int64_t i = j + 1 + i0, c = j + 1 + cc;
      A[i * n + c] -= A[i * n + j] * A[c * n + j];
    }
    __syncthreads();
  }
}

// V[j] = A_bar_j k_v + c_j as a dense NX row: block k < k_j: K_k^T b_{j,k} + c_{j,k};
// block k_j: c_{j,k_j} = grad g_j; control rows: block k_j = K_k^T h'_j.
__global__ void k_gen_v(Dev v, const double* __restrict__ Cf, double* Vf) {
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, NX = (d.T + 1) * nx;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)d.B * d.ng * NX) return;
  const int64_t bj = id / NX;
  const int x = (int)(id % NX);
  const int b = (int)(bj / d.ng), j = (int)(bj % d.ng);
  if (!v.active[b]) return;
  const int k = x / nx, i = x % nx;
  const int kj = v.knot[j];
  double val = Cf[id];
  const bool ctrl = v.kind[j] != 0;
  if ((!ctrl && k < kj) || (ctrl && k == kj)) {
    const double* bb = v.Bd + (int64_t)b * d.EB + v.offB[j] + (ctrl ? 0 : (int64_t)k * d.nup);
    const double* Kk = v.K + (int64_t)b * d.NK + (int64_t)k * nu * nx;   // vec: [i*nu + m] = K[m][i]
    for (int m = 0; m < nu; ++m) val += Kk[i * nu + m] * bb[m];
  }
  Vf[id] = val;
}

// Block-1 (13) on dense n_z rows, with the pending dual update (16) of iteration l-1:
// lam += a - nu (l > 1); y = a + lam; (p~, nu) = Pi(t, y), t = p + lam_p.  Warp per cone.
__global__ void k_gen_project(Dev v, const double* __restrict__ Aa, double* lam, double* nu, int nz,
                              int first) {
  const Dims d = v.d;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (int64_t)d.B * d.ng) return;
  const int b = (int)(w / d.ng);
  if (!v.active[b]) return;
  const int lane = threadIdx.x & 31;
  const double* a = Aa + w * nz;
  double* l = lam + w * nz;
  double* n = nu + w * nz;
  double n2 = 0.0;
  for (int z = lane; z < nz; z += 32) {
    const double lz = first ? 0.0 : l[z] + a[z] - n[z];
    l[z] = lz;
    const double y = a[z] + lz;
    n[z] = y;
    n2 += y * y;
  }
  n2 = warp_sum(n2);
  double s;
  const double tp = soc_case(v.tin[w], sqrt(n2), &s);
  for (int z = lane; z < nz; z += 32) n[z] *= s;
  if (lane == 0) {
    v.s[w] = s;
    v.pt[w] = tp;
  }
  count_case(v, s);
}

// W[b] *= sqrt(tau_b)
__global__ void k_gen_scale(double* W, const double* __restrict__ tau, int64_t per, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) W[i] *= sqrt(tau[i / per]);
}

// nu - b_hat (dense n_z rows)
__global__ void k_gen_sub(const double* __restrict__ nu, const double* __restrict__ Bh, double* out,
                          int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = nu[i] - Bh[i];
}

// rhs of (14b): Q_v k + rho A_bar^T U, U = (nu - b_hat) W  (rows NX):
// rhs[(k,i,m)] = 2 (W_k K_k)[m][i] + rho sum_{j with a b-block at k} b_{j,k}[m] U[j][(k,i)]
__global__ void k_gen_rhs(Dev v, const double* __restrict__ U, double* rhs, double rho) {
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, NX = (d.T + 1) * nx;
  const int b = blockIdx.x / d.T, k = blockIdx.x % d.T;
  if (!v.active[b]) return;
  const double* Kk = v.K + (int64_t)b * d.NK + (int64_t)k * nu * nx;
  const double* Wk = v.W + ((int64_t)b * d.T + k) * nu * nu;
  for (int o = threadIdx.x; o < nu * nx; o += blockDim.x) {
    const int i = o / nu, m = o % nu;
    double acc = 0.0;
    for (int q = v.kptr[k]; q < v.kptr[k + 1]; ++q) {
      const int j = v.kcone[q];
      const bool ctrl = v.kind[j] != 0;
      const double bm = v.Bd[(int64_t)b * d.EB + v.offB[j] + (ctrl ? 0 : (int64_t)k * d.nup) + m];
      acc += bm * U[((int64_t)b * d.ng + j) * NX + k * nx + i];
    }
    double wk = 0.0;
    for (int q = 0; q < nu; ++q) wk += Wk[m * nu + q] * Kk[i * nu + q];
    rhs[(int64_t)b * d.NK + (int64_t)k * nu * nx + o] = 2.0 * wk + rho * acc;
  }
}

// k_v = M rhs with M^{-1} = L L^T (one CTA per instance: forward, then backward substitution)
__global__ void k_gen_solve(Dev v, const double* __restrict__ L, const double* __restrict__ rhs) {
  const int b = blockIdx.x;
  if (!v.active[b]) return;
  const int n = v.d.NK;
  const double* Lb = L + (int64_t)b * n * n;
  extern __shared__ double x[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = rhs[(int64_t)b * n + i];
  __syncthreads();
  for (int j = 0; j < n; ++j) {                  // L y = rhs
    if (threadIdx.x == 0) x[j] /= Lb[(int64_t)j * n + j];
    __syncthreads();
    const double xj = x[j];
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) x[i] -= Lb[(int64_t)i * n + j] * xj;
    __syncthreads();
  }
  for (int j = n - 1; j >= 0; --j) {             // L^T k = y
    if (threadIdx.x == 0) x[j] /= Lb[(int64_t)j * n + j];
    __syncthreads();
    const double xj = x[j];
    for (int i = threadIdx.x; i < j; i += blockDim.x) x[i] -= Lb[(int64_t)j * n + i] * xj;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) v.K[(int64_t)b * n + i] = x[i];
}

// finish: lam^L = lam + a(k^L) - nu^L, margin_cone = p~ - ||a(k^L)||
__global__ void k_gen_finish(Dev v, const double* __restrict__ Aa, double* lam, const double* nu, int nz,
                             double* mcone) {
  const Dims d = v.d;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (int64_t)d.B * d.ng) return;
  const int lane = threadIdx.x & 31;
  const double* a = Aa + w * nz;
  double n2 = 0.0;
  for (int z = lane; z < nz; z += 32) {
    lam[w * nz + z] += a[z] - nu[w * nz + z];
    n2 += a[z] * a[z];
  }
  n2 = warp_sum(n2);
  if (lane == 0 && mcone) mcone[w] = v.pt[w] - sqrt(n2);
}

// ---------------------------------------------------------------------------
cudaError_t gen_setup(nrto_handle_s* h, const double* Gamma, const double* Psi, int nz, bool host,
                      cudaStream_t st, int* spd_err) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  GenState& g = h->gen;
  const int NX = (d.T + 1) * d.nx, NU = d.T * d.nu, NK = d.NK;
  const int64_t B = d.B;
  auto al = [&](double** p, int64_t n) -> cudaError_t {
    cudaError_t e = cudaMalloc((void**)p, (size_t)std::max<int64_t>(n, 1) * sizeof(double));
    if (e == cudaSuccess) g.allocs[g.nallocs++] = *p;
    return e;
  };
  cudaError_t e = cudaSuccess;
  g.nz = nz;
  double *Gm = nullptr, *Ps = nullptr, *Cf = nullptr, *Bf = nullptr, *GG = nullptr, *Lam = nullptr;
  if (e == cudaSuccess) e = al(&g.W, B * nz * NX);
  if (e == cudaSuccess) e = al(&g.Bh, B * d.ng * nz);
  if (e == cudaSuccess) e = al(&g.L, B * (int64_t)NK * NK);
  if (e == cudaSuccess) e = al(&g.lam, B * d.ng * nz);
  if (e == cudaSuccess) e = al(&g.nu, B * d.ng * nz);
  if (e == cudaSuccess) e = al(&g.a, B * d.ng * nz);
  if (e == cudaSuccess) e = al(&g.V, B * d.ng * NX);
  if (e == cudaSuccess) e = al(&g.Cf, B * d.ng * NX);
  if (e == cudaSuccess) e = al(&g.rhs, B * NK);
  if (e != cudaSuccess) return e;
  Cf = g.Cf;
  // scratch for setup only
  e = cudaMalloc((void**)&Gm, (size_t)std::max<int64_t>(B * NX * nz, 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc((void**)&Ps, (size_t)std::max<int64_t>(B * nz * nz, 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc((void**)&Bf, (size_t)std::max<int64_t>(B * d.ng * NU, 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc((void**)&GG, (size_t)std::max<int64_t>(B * NX * NX, 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc((void**)&Lam, (size_t)std::max<int64_t>(B * NU * NU, 1) * 8);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(Gm, Gamma, (size_t)B * NX * nz * 8, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(Ps, Psi, (size_t)B * nz * nz * 8, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st);
  // W = sqrt(tau) Psi Gamma^T
  if (e == cudaSuccess)
    e = dgemm(1, Ps, Gm, g.W, nz, NX, nz, (int64_t)nz * nz, (int64_t)NX * nz, (int64_t)nz * NX, d.B, 1.0, st);
  if (e == cudaSuccess) {
    const int64_t n = B * nz * NX;
    k_gen_scale<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g.W, g.tau, (int64_t)nz * NX, n);
    h->launches++;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && (int64_t)B * d.ng > 0) {
    k_gen_expand<<<(unsigned)((B * d.ng + 127) / 128), 128, 0, st>>>(v, Cf, Bf);
    h->launches++;
    e = cudaGetLastError();
  }
  // b_hat = C W^T ; G = W^T W ; Lam = Bf^T Bf
  if (e == cudaSuccess) e = dgemm(1, Cf, g.W, g.Bh, d.ng, nz, NX, (int64_t)d.ng * NX, (int64_t)nz * NX,
                                 (int64_t)d.ng * nz, d.B, 1.0, st);
  if (e == cudaSuccess) {
    dim3 grid((NX + 15) / 16, (NX + 15) / 16, d.B), blk(16, 16);
    k_dgemm_tn<<<grid, blk, 0, st>>>(g.W, g.W, GG, NX, NX, nz, (int64_t)nz * NX, (int64_t)nz * NX, (int64_t)NX * NX);
    h->launches++;
    dim3 grid2((NU + 15) / 16, (NU + 15) / 16, d.B);
    k_dgemm_tn<<<grid2, blk, 0, st>>>(Bf, Bf, Lam, NU, NU, d.ng, (int64_t)d.ng * NU, (int64_t)d.ng * NU, (int64_t)NU * NU);
    h->launches++;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    int zero = 0;
    cudaMemcpyToSymbolAsync(g_gen_err, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, st);
    const int64_t n = B * (int64_t)NK * NK;
    k_gen_minv<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(v, GG, Lam, g.L, v.prm.rho);
    k_gen_chol<<<d.B, 1024, 0, st>>>(g.L, NK);
    h->launches += 2;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    int err = 0;
    e = cudaMemcpyFromSymbolAsync(&err, g_gen_err, sizeof(int), 0, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    *spd_err = err;
  }
  cudaFree(Gm); cudaFree(Ps); cudaFree(Bf); cudaFree(GG); cudaFree(Lam);
  return e;
}

cudaError_t gen_reset(nrto_handle_s* h, cudaStream_t st) {
  GenState& g = h->gen;
  const Dims& d = h->dev.d;
  const int64_t n = (int64_t)d.B * d.ng * g.nz;
  cudaError_t e = cudaMemsetAsync(g.lam, 0, (size_t)std::max<int64_t>(n, 1) * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(g.nu, 0, (size_t)std::max<int64_t>(n, 1) * 8, st);
  return e;
}

// one FullADMM outer iteration l on the general set (in-order)
cudaError_t gen_iteration(nrto_handle_s* h, int l, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  GenState& g = h->gen;
  const int NX = (d.T + 1) * d.nx, nz = g.nz;
  v.iter = l;
  const int64_t nvx = (int64_t)d.B * d.ng * NX;
  cudaError_t e = cudaSuccess;
  if (nvx > 0) {
    k_gen_v<<<(unsigned)((nvx + 255) / 256), 256, 0, st>>>(v, g.Cf, g.V);   // a(k^{l-1})
    h->launches++;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = dgemm(1, g.V, g.W, g.a, d.ng, nz, NX, (int64_t)d.ng * NX, (int64_t)nz * NX,
                                 (int64_t)d.ng * nz, d.B, 1.0, st);
  if (e == cudaSuccess && (int64_t)d.B * d.ng > 0) {
    k_gen_project<<<(unsigned)(((int64_t)d.B * d.ng + 7) / 8), 256, 0, st>>>(v, g.a, g.lam, g.nu, nz, l == 1);
    h->launches++;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    const bool wide = d.ng >= 512 || d.B >= v.nsm;
    e = wide ? launch_qp_sparse(h, NRTO_FULLADMM, l, st) : launch_qp(h, NRTO_FULLADMM, l, st);
  }
  // (14b): U = (nu - b_hat) W  -> rhs -> k
  const int64_t nzz = (int64_t)d.B * d.ng * nz;
  if (e == cudaSuccess && nzz > 0) {
    k_gen_sub<<<(unsigned)((nzz + 255) / 256), 256, 0, st>>>(g.nu, g.Bh, g.a, nzz);   // a <- nu - b_hat
    h->launches++;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = dgemm(0, g.a, g.W, g.V, d.ng, NX, nz, (int64_t)d.ng * nz, (int64_t)nz * NX,
                                 (int64_t)d.ng * NX, d.B, 1.0, st);
  if (e == cudaSuccess) {
    k_gen_rhs<<<d.B * d.T, 128, 0, st>>>(v, g.V, g.rhs, v.prm.rho);
    k_gen_solve<<<d.B, 256, (size_t)d.NK * 8, st>>>(v, g.L, g.rhs);
    h->launches += 2;
    e = cudaGetLastError();
  }
  return e;
}

cudaError_t gen_finish(nrto_handle_s* h, double* mcone, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  GenState& g = h->gen;
  const int NX = (d.T + 1) * d.nx, nz = g.nz;
  const int64_t nvx = (int64_t)d.B * d.ng * NX;
  int32_t* act = v.active;
  cudaError_t e = cudaSuccess;
  // a(k^L) for every instance (frozen ones included): temporarily mark all active
  int32_t* ones = nullptr;
  e = cudaMalloc((void**)&ones, (size_t)std::max(d.B, 1) * 4);
  if (e != cudaSuccess) return e;
  std::vector<int32_t> h1(d.B, 1);
  e = cudaMemcpyAsync(ones, h1.data(), (size_t)d.B * 4, cudaMemcpyHostToDevice, st);
  v.active = ones;
  if (e == cudaSuccess && nvx > 0) {
    k_gen_v<<<(unsigned)((nvx + 255) / 256), 256, 0, st>>>(v, g.Cf, g.V);
    h->launches++;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = dgemm(1, g.V, g.W, g.a, d.ng, nz, NX, (int64_t)d.ng * NX, (int64_t)nz * NX,
                                 (int64_t)d.ng * nz, d.B, 1.0, st);
  if (e == cudaSuccess && (int64_t)d.B * d.ng > 0) {
    k_gen_finish<<<(unsigned)(((int64_t)d.B * d.ng + 7) / 8), 256, 0, st>>>(v, g.a, g.lam, g.nu, nz, mcone);
    h->launches++;
    e = cudaGetLastError();
  }
  v.active = act;
  cudaStreamSynchronize(st);
  cudaFree(ones);
  return e;
}

void gen_free(nrto_handle_s* h) {
  for (int i = 0; i < h->gen.nallocs; ++i) cudaFree(h->gen.allocs[i]);
  h->gen.nallocs = 0;
}

}  // namespace nrto

// Debug copy of internal general-set arrays to caller memory (not part of nrto.h):
// which = 0 W [B][n_z][NX], 1 b_hat [B][n_g][n_z], 2 L [B][NK][NK], 3 ragged costates
// (v.bhat) [B][E], 4 ragged b rows (v.Bd) [B][EB], 5 dense M^-1 rebuilt into dst.
extern "C" int nrto_debug_gen_copy(nrto_handle h, int which, double* dst, int64_t n) {
  using namespace nrto;
  const GenState& g = h->gen;
  const Dev& v = h->dev;
  const double* src = nullptr;
  int64_t avail = 0;
  const int64_t B = v.d.B, NX = (int64_t)(v.d.T + 1) * v.d.nx, NK = v.d.NK;
  switch (which) {
    case 0: src = g.W; avail = B * g.nz * NX; break;
    case 1: src = g.Bh; avail = B * v.d.ng * g.nz; break;
    case 2: src = g.L; avail = B * NK * NK; break;
    case 3: src = v.bhat; avail = B * v.d.E; break;
    case 4: src = v.Bd; avail = B * v.d.EB; break;
    default: return -1;
  }
  if (!src || n > avail) return -2;
  cudaDeviceSynchronize();
  return (int)cudaMemcpy(dst, src, (size_t)n * 8, cudaMemcpyDeviceToHost);
}
