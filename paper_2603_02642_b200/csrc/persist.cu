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

// Shared-memory doubles of k_dr_loop (host and device agree on this).
__host__ __device__ inline int64_t dr_loop_smem_doubles(const Dims& d, int Ec, int EBc, int ncmax) {
  const int NA = d.nu * d.nx, NN = d.nx * d.nx, NG = d.nu * d.nu;
  const int ngrp = 256 / NA > 0 ? 256 / NA : 1;
  const int64_t g = (int64_t)NA * (5 + ngrp) + 2 * NN + NG;
  const int64_t p = (int64_t)d.T * NA + 2 * (int64_t)Ec + EBc + ncmax;
  return (g > p ? g : p) + 8 * ncmax;   // + cone records (int64 offsets, ints)
}

template <int NUM>
__global__ void __launch_bounds__(256) k_dr_loop(Dev v, int ndr, int ncmax) {
  extern __shared__ double sm[];
  __shared__ int sact[32];      // DR-active per instance (same in every CTA)
  __shared__ int sran[32];      // instance ran the previous pass
  const Dims d = v.d;
  const int nx = d.nx, nu = NUM > 0 ? NUM : d.nu, T = d.T, Q = v.drQ, B = d.B;
  const int NA = nu * nx, NN = nx * nx, NG = nu * nu;
  const int tid = threadIdx.x, nt = blockDim.x, G = gridDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const double sg = v.prm.sigma_dr, rs = v.prm.r_s, al = v.prm.alpha_dr, rho = v.prm.rho_admm;
  unsigned long long nbar = 0;
  if (tid < B) { sact[tid] = v.active[tid] && v.dr_active[tid]; sran[tid] = 0; }
  __syncthreads();
  for (int m = 1;; ++m) {
    // ---- head: r_dr of pass m-1 and the stop test, identically in every CTA
    if (m > 1) {
      if (tid < B) sran[tid] = sact[tid];
      __syncthreads();
      for (int b = warp; b < B; b += nw) {
        if (!sran[b]) continue;
        double a = 0.0;
        for (int q = lane; q < Q; q += 32) a += __ldcg(v.drrq + (int64_t)b * Q + q);
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
    int any = 0;
    for (int b = 0; b < B; ++b) any |= sact[b];
    const bool run = any && m <= ndr;
    // ---- phase G: adjoint of eta~^{m-1} per step (stored to Z for the warm start
    //      of the next call) and, while running, the affine prox (11a)
    for (int task = blockIdx.x; task < B * T; task += G) {
      const int b = task / T, k = task % T;
      const bool need_z = m > 1 && sran[b];
      const bool gain = run && sact[b];
      if (!need_z && !gain) continue;
      const int64_t bk = (int64_t)b * T + k;
      const int ngrp = nt / NA > 0 ? nt / NA : 1;
      double* sZ = sm;
      double* sR = sZ + NA;
      double* sX = sR + NA;
      double* sKt = sX + NA;
      double* sden = sKt + NA;
      double* sP = sden + NA;
      double* sU = sP + NN;
      double* sV = sU + NN;
      double* sZg = sV + NG;       // [ngrp][NA]
      if (m == 1) {
        for (int r = tid; r < NA; r += nt) sZ[r] = __ldcg(v.Z + bk * NA + r);
      } else {
        const int g = tid / NA, o = tid - g * NA;
        if (g < ngrp) {
          double acc = 0.0;
          for (int q = g; q < Q; q += ngrp) {
            const int klo = __ldg(v.drkr + 2 * q), khi = __ldg(v.drkr + 2 * q + 1);
            if (k >= klo && k < khi) acc += __ldcg(v.drZpart + (((int64_t)b * Q + q) * T + k) * NA + o);
          }
          sZg[g * NA + o] = acc;
        }
        __syncthreads();
        for (int r = tid; r < NA; r += nt) {
          double z = 0.0;
          for (int g2 = 0; g2 < ngrp; ++g2) z += sZg[g2 * NA + r];
          sZ[r] = z;
          v.Z[bk * NA + r] = z;
        }
      }
      if (!gain) { __syncthreads(); continue; }
      const int kr = __ldg(v.Urep + bk);
      const double st = sqrt(__ldg(v.tau + b));
      double* Kt = v.Kt + (int64_t)b * d.NK + (int64_t)k * nu * nx;
      const double* Pk = v.Psi + ((int64_t)b * (T + 1) + kr) * NN;
      const double* Uk = v.U + ((int64_t)b * T + kr) * NN;
      for (int r = tid; r < NA; r += nt) {
        sKt[r] = __ldcg(Kt + r);
        sden[r] = __ldg(v.dr.den + bk * NA + r);
      }
      for (int r = tid; r < NN; r += nt) { sP[r] = __ldg(Pk + r); sU[r] = __ldg(Uk + r); }
      for (int r = tid; r < NG; r += nt) sV[r] = __ldg(v.dr.V + bk * NG + r);
      __syncthreads();
      for (int r = tid; r < NA; r += nt) sX[r] = sZ[r] - __ldg(v.Zb + bk * NA + r);
      __syncthreads();
      for (int r = tid; r < NA; r += nt) {
        const int mm = r / nx, i = r % nx;
        double gp = 0.0;
        for (int q = 0; q < nx; ++q) gp += sX[mm * nx + q] * sP[q * nx + i];
        sR[r] = sg * sKt[i * nu + mm] + rs * st * gp;
      }
      __syncthreads();
      chain_solve<0, NUM>(sV, sU, sden, sR, sX, nu, nx, tid, nt);
      double* Ko = v.K + (int64_t)b * d.NK + (int64_t)k * nu * nx;
      for (int r = tid; r < NA; r += nt) {
        const int mm = r / nx, i = r % nx;
        Ko[i * nu + mm] = sR[r];
        Kt[i * nu + mm] = sKt[i * nu + mm] + al * (sR[r] - sKt[i * nu + mm]);
      }
      for (int r = tid; r < NA; r += nt) {
        const int i = r / nu, mm = r % nu;
        double acc = 0.0;
        for (int q = 0; q < nx; ++q) acc += sP[i * nx + q] * sR[mm * nx + q];
        v.Ccur[bk * NA + r] = st * acc;
      }
      __syncthreads();
    }
    if (!run) break;
    grid_barrier(v.drbar, (++nbar) * (unsigned long long)G);
    // ---- phase P: cone steps of every chunk, chunk adjoint partials
    for (int item = blockIdx.x; item < B * Q; item += G) {
      const int b = item / Q, q = item % Q;
      if (!sact[b]) continue;
      const int j0 = __ldg(v.drchunk + q), j1 = __ldg(v.drchunk + q + 1), nc = j1 - j0;
      const int klo = __ldg(v.drkr + 2 * q), khi = __ldg(v.drkr + 2 * q + 1);
      int64_t* cof = reinterpret_cast<int64_t*>(sm);          // [ncmax] eta~ offsets (chunk-local)
      int64_t* cofB = cof + ncmax;                            // [ncmax] b-row offsets
      int* cinf = reinterpret_cast<int*>(cofB + ncmax);       // [ncmax][4] kind, knot, klo, nbB
      double* sd2 = sm + 6 * ncmax;                           // [ncmax]
      double* sC = sd2 + ncmax;                               // [(khi - klo)][nx][nu]
      double* sB = sC + (int64_t)T * NA;                      // [EBc]
      double* sA = sB + v.drEBc;                              // [Ec]
      double* sY = sA + v.drEc;                               // [Ec]
      const int64_t off0 = __ldg(v.off + j0), offB0 = __ldg(v.offB + j0);
      const int64_t nB = __ldg(v.offB + j1) - offB0;
      for (int c = tid; c < nc; c += nt) {
        const int j = j0 + c, kd = __ldg(v.kind + j), kn = __ldg(v.knot + j);
        cof[c] = __ldg(v.off + j) - off0;
        cofB[c] = __ldg(v.offB + j) - offB0;
        cinf[4 * c + 0] = kd; cinf[4 * c + 1] = kn;
        cinf[4 * c + 2] = kd == 0 ? 0 : kn; cinf[4 * c + 3] = kd == 0 ? kn : 1;
      }
      const double* Cg = v.Ccur + ((int64_t)b * T + klo) * NA;
      for (int r = tid; r < (khi - klo) * NA; r += nt) sC[r] = __ldcg(Cg + r);
      const double* Bdg = v.Bd + (int64_t)b * d.EB + offB0;
      for (int64_t r = tid; r < nB; r += nt) sB[r] = __ldg(Bdg + r);
      __syncthreads();
      for (int c = warp; c < nc; c += nw) {
        const int kd = cinf[4 * c], kn = cinf[4 * c + 1], cklo = cinf[4 * c + 2], nbB = cinf[4 * c + 3];
        const int L = kd == 0 ? (kn + 1) * nx : nx;
        const int64_t ij = (int64_t)b * d.ng + j0 + c;
        const int64_t eo = (int64_t)b * d.E + off0 + cof[c];
        double* Y = v.Y + eo;
        const double* bh = v.bhat + eo;
        const double* br0 = sB + cofB[c];
        double* ca = sA + cof[c];
        double* cy = sY + cof[c];
        const double pit = __ldcg(v.pit + ij), tt = __ldcg(v.tt + ij);
        const double pi = (sg * pit + rho * __ldcg(v.p + ij) + __ldcg(v.lamp + ij) + rs * tt) / (rho + sg + rs);
        double n2 = 0.0;
#pragma unroll 2
        for (int e = lane; e < L; e += 32) {
          const int kb = e / nx, i = e - kb * nx;
          double a = (kd == 0) ? __ldg(bh + e) : 0.0;
          if (kb < nbB) {
            const double* Cr = sC + ((cklo + kb - klo) * nx + i) * nu;
            const double* br = br0 + kb * d.nup;
            if constexpr (NUM > 0) {
#pragma unroll
              for (int mm = 0; mm < NUM; ++mm) a += Cr[mm] * br[mm];
            } else {
              for (int mm = 0; mm < nu; ++mm) a += Cr[mm] * br[mm];
            }
          }
          const double et = __ldcg(Y + e);
          ca[e] = a;
          cy[e] = et;
          const double er = 2.0 * a - et;
          n2 += er * er;
        }
        n2 = warp_sum(n2);
        double sc;
        const double tpi = soc_case(2.0 * pi - tt, sqrt(n2), &sc);
        double d2 = 0.0;
        for (int e = lane; e < L; e += 32) {
          const double a = ca[e], et = cy[e];
          const double er = 2.0 * a - et;
          const double en = et + al * (sc * er - a);
          Y[e] = en;
          cy[e] = en;
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
          sd2[c] = d2;
        }
      }
      __syncthreads();
      // chunk partial Z_k^(q) = sum_{j in q} b_{j,k} eta~_{j,k}^T (cone order)
      double* Zq = v.drZpart + ((int64_t)b * Q + q) * T * NA;
      for (int r = tid; r < (khi - klo) * NA; r += nt) {
        const int k = klo + r / NA, o = r % NA, mm = o / nx, i = o % nx;
        double acc = 0.0;
        for (int c = 0; c < nc; ++c) {
          const int cklo = cinf[4 * c + 2], nbB = cinf[4 * c + 3];
          if (k >= cklo && k < cklo + nbB) {
            const int kb = k - cklo;
            acc += sB[cofB[c] + kb * d.nup + mm] * sY[cof[c] + kb * nx + i];
          }
        }
        Zq[(int64_t)k * NA + o] = acc;
      }
      if (tid == 0) {
        double a = 0.0;
        for (int c = 0; c < nc; ++c) a += sd2[c];
        v.drrq[(int64_t)b * Q + q] = a;
      }
      __syncthreads();
    }
    grid_barrier(v.drbar, (++nbar) * (unsigned long long)G);
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
  const int target_q = std::max(1, nsm / d.B);
  auto work = [&](int j) -> int64_t {
    const int64_t L = kind[j] == 0 ? (int64_t)(knot[j] + 1) * d.nx : d.nx;
    const int64_t nb = kind[j] == 0 ? knot[j] : 1;
    return L + nb * d.nup + 32;
  };
  int64_t tot = 0;
  for (int j = 0; j < d.ng; ++j) tot += work(j);
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

size_t dr_loop_smem(const Dev& v) {
  return (size_t)dr_loop_smem_doubles(v.d, v.drEc, v.drEBc, kDrChunkCones) * sizeof(double);
}

// Grid of the cooperative launch (0: cannot be co-resident -> launch-per-phase path).
int dr_loop_grid(const Dev& v) {
  if (v.drQ <= 0) return 0;
  const size_t smem = dr_loop_smem(v);
  if (smem > 200 * 1024) return 0;
  auto kern = v.d.nu == 4 ? (void*)k_dr_loop<4> : (void*)k_dr_loop<0>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    return 0;
  }
  const int want = std::max(v.d.B * v.drQ, v.d.B * v.d.T);
  return std::min(want, occ * v.nsm);
}

cudaError_t launch_dr_loop(nrto_handle_s* h, int ndr, cudaStream_t st) {
  const Dev& v = h->dev;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(h->dr_loop_grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = dr_loop_smem(v);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (v.d.nu == 4)
    e = cudaLaunchKernelEx(&cfg, k_dr_loop<4>, v, ndr, kDrChunkCones);
  else
    e = cudaLaunchKernelEx(&cfg, k_dr_loop<0>, v, ndr, kDrChunkCones);
  h->launches++;
  return e;
}

}  // namespace nrto
