#include <algorithm>
#include <cstdlib>
// Fused FullADMM cone pass (S3 forward map + S4 SOC projection + S5 state
// update + S7 adjoint) in ONE streaming pass over the ragged cone data, with
// both small contractions on the FP64 tensor cores (DMMA m8n8k4).
//
// Work decomposition.  Cones with the same (kind, knot) are grouped into tiles
// of <= 8 (host side, nrto_setup).  A CTA (8 warps) walks a range of tiles of
// one instance; warp w owns the time blocks k == w (mod 8) of every tile, so
// the per-step adjoint accumulator Z_k lives in a warp-private slice of shared
// memory and is never contended.
//
// Per (tile, block k) a warp computes, for the <= 8 cones c of the tile,
//   y_new[c][k][:] = D_k b_{c,k} + b_hat_{c,k} + (1 - s^{l-1}_c) y_old[c][k][:]
// (see k_fa_pass in iter.cu for the derivation) as one DMMA chain
// [8 cones x 4 m] x [4 m x 8 i] (rows = cones, cols = state index i), writes
// y_new, accumulates ||y_new||^2 per cone, and adds the PREDICTED adjoint
//   Z_k += sum_c shat_c b_{c,k} y_new[c][k]^T,   shat_c = [s^{l-1}_c == 1]
// as a second DMMA chain [8 m x 4 cones] x [4 cones x 8 i].  The exact adjoint
// needs s^l_c, known only after the whole cone; cones whose s^l differs from
// shat (case-3 cones and case switches; all cones at l = 1) are appended to a
// correction list and added by k_zcorr with weight s^l - shat.  For cones in
// case 1 at consecutive iterations (the large majority near convergence) the
// prediction is exact, so the pass streams every cone element exactly once:
// algorithmic bytes 8 (2E + E_s + E_B) per instance-iteration.
#include "common.cuh"

namespace nrto {

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

constexpr int kRing = 4;      // tile slots in flight per CTA (norm partials)
constexpr int kTileInts = 12; // kind, knot, nc, klo, cone[8]

// NTI: 8-wide tiles over the state index i (n_x <= 8 NTI);
// NKS: 4-deep k-steps over the control index m (n_u <= 4 NKS).
template <int NTI, int NKS>
__global__ void __launch_bounds__(256, 2)
k_fa_fused(Dev v, const int32_t* __restrict__ tiles, const int32_t* __restrict__ witems) {
  extern __shared__ double sm[];
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, T = d.T;
  constexpr int ZW = 8 * NTI;                        // padded Z row width
  double* Zs = sm;                                   // [T][8][ZW]
  double* ring = Zs + (size_t)T * 8 * ZW;            // [kRing][8 warps][8 cones]
  int* cnt = (int*)(ring + kRing * 64);              // [kRing]
  int* tag = cnt + kRing;                            // [kRing]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int b = witems[4 * blockIdx.x], t0 = witems[4 * blockIdx.x + 1];
  const int t1 = witems[4 * blockIdx.x + 2], sidx = witems[4 * blockIdx.x + 3];
  if (!v.active[b]) return;                          // uniform over the CTA
  for (int r = threadIdx.x; r < T * 8 * ZW; r += blockDim.x) Zs[r] = 0.0;
  if (threadIdx.x < kRing) { cnt[threadIdx.x] = 0; tag[threadIdx.x] = threadIdx.x; }
  __syncthreads();

  const double* __restrict__ bhat = v.bhat + (int64_t)b * d.E;
  const double* __restrict__ Bd = v.Bd + (int64_t)b * d.EB;
  const double* __restrict__ Dm = v.D + (int64_t)b * T * nx * nu;
  double* __restrict__ Y = v.Y + (int64_t)b * d.E;
  const int64_t bg = (int64_t)b * d.ng;
  const bool vec2 = (nx & 1) == 0;

  for (int t = t0; t < t1; ++t) {
    const int* tl = tiles + (int64_t)t * kTileInts;
    const int kind = tl[0], K = tl[1], nc = tl[2], klo = tl[3];
    const int nblk = K - klo + 1;                    // blocks in each cone row
    const int first = klo + ((warp - klo) % 8 + 8) % 8;
    if (first > K) continue;                         // this warp owns no block of the tile
    const int lt = t - t0, slot = lt % kRing;
    // per-lane cone meta: C/A layout cone = g ; A2/B2 layout cones q, q+4
    const bool gv = g < nc;
    const int cg = gv ? tl[4 + g] : 0;
    const int64_t offg = gv ? v.off[cg] : 0, offBg = gv ? v.offB[cg] : 0;
    const double omsp = gv ? 1.0 - v.s[bg + cg] : 0.0;
    int64_t offB2[2];     // the adjoint DMMA contracts over the tile's 8 cones: 2 steps of 4
    double sh2[2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int c2 = q + 4 * ks;
      const bool c2v = c2 < nc;
      const int cc = c2v ? tl[4 + c2] : 0;
      offB2[ks] = c2v ? v.offB[cc] : 0;
      sh2[ks] = c2v ? shat_of(v, v.s[bg + cc]) : 0.0;
    }
    double nrm = 0.0;
    for (int k = first; k <= K; k += 8) {
      const int kb = k - klo;
      const bool hasB = (kind == 0) ? (k < K) : true;
      double c[NTI][2];
      // ---- C init: b_hat + (1 - s) y_old
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) {
        const int i0 = 2 * q + 8 * nt;
        c[nt][0] = 0.0; c[nt][1] = 0.0;
        if (gv && i0 < nx) {
          const int64_t e = offg + (int64_t)kb * nx + i0;
          if (vec2) {
            const double2 yo = *reinterpret_cast<const double2*>(Y + e);
            c[nt][0] = omsp * yo.x; c[nt][1] = omsp * yo.y;
            if (kind == 0) {
              const double2 bh = __ldg(reinterpret_cast<const double2*>(bhat + e));
              c[nt][0] += bh.x; c[nt][1] += bh.y;
            }
          } else {
            c[nt][0] = omsp * Y[e] + (kind == 0 ? __ldg(bhat + e) : 0.0);
            if (i0 + 1 < nx) c[nt][1] = omsp * Y[e + 1] + (kind == 0 ? __ldg(bhat + e + 1) : 0.0);
          }
        }
      }
      if (hasB) {
        // ---- forward map: y += [b_{c,k}]_(c,m) [D_k^T]_(m,i)
        const int kbB = (kind == 0) ? kb : 0;
        double a[NKS];
#pragma unroll
        for (int ks = 0; ks < NKS; ++ks) {
          const int m = q + 4 * ks;
          a[ks] = (gv && m < nu) ? __ldg(Bd + offBg + (int64_t)kbB * d.nup + m) : 0.0;
        }
        const double* Dk = Dm + (int64_t)k * nx * nu;
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt) {
#pragma unroll
          for (int ks = 0; ks < NKS; ++ks) {
            const int m = q + 4 * ks, i = g + 8 * nt;
            const double bb = (m < nu && i < nx) ? __ldg(Dk + i * nu + m) : 0.0;
            dmma(c[nt], a[ks], bb);
          }
        }
      }
      // ---- store y_new, norm partial
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) {
        const int i0 = 2 * q + 8 * nt;
        if (gv && i0 < nx) {
          const int64_t e = offg + (int64_t)kb * nx + i0;
          if (vec2) {
            *reinterpret_cast<double2*>(Y + e) = make_double2(c[nt][0], c[nt][1]);
          } else {
            Y[e] = c[nt][0];
            if (i0 + 1 < nx) Y[e + 1] = c[nt][1];
          }
        }
        nrm += c[nt][0] * c[nt][0] + c[nt][1] * c[nt][1];
      }
      if (hasB) {
        // ---- predicted adjoint: Z_k += [shat_c b_{c,k,m}]_(m,c) [y_{c,k,i}]_(c,i)
        const int kbB = (kind == 0) ? kb : 0;
        double a2[2];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
          a2[ks] = (g < nu && sh2[ks] != 0.0) ? sh2[ks] * __ldg(Bd + offB2[ks] + (int64_t)kbB * d.nup + g) : 0.0;
        double* Zk = Zs + (size_t)k * 8 * ZW;
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt) {
          double z[2] = {Zk[g * ZW + 2 * q + 8 * nt], Zk[g * ZW + 2 * q + 8 * nt + 1]};
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            // B2[row = cone q+4ks][col = i = g + 8nt] lives in lane (q+4ks)*4 + g/2, slot g&1
            const int src = (q + 4 * ks) * 4 + (g >> 1);
            const double v0 = __shfl_sync(0xffffffffu, c[nt][0], src);
            const double v1 = __shfl_sync(0xffffffffu, c[nt][1], src);
            dmma(z, a2[ks], (g & 1) ? v1 : v0);
          }
          Zk[g * ZW + 2 * q + 8 * nt] = z[0];
          Zk[g * ZW + 2 * q + 8 * nt + 1] = z[1];
        }
      }
    }
    // ---- per-cone norm partial of this warp -> ring slot; last warp projects
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 1);
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 2);
    if (lane == 0) {
      while (atomicAdd(&tag[slot], 0) != lt) { __nanosleep(20); }
    }
    __syncwarp();
    if (q == 0) ring[(slot * 8 + warp) * 8 + g] = nrm;
    __threadfence_block();
    __syncwarp();
    int last = 0;
    const int npart = nblk >= 8 ? 8 : nblk;
    if (lane == 0) last = (atomicAdd(&cnt[slot], 1) == npart - 1);
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence_block();
      if (lane < nc) {
        double n2 = 0.0;
        for (int w = 0; w < 8; ++w)
          if (((w - klo) % 8 + 8) % 8 <= K - klo) n2 += ring[(slot * 8 + w) * 8 + lane];
        v.nrm2[bg + tl[4 + lane]] = n2;     // projection decided by k_project
      }
      __syncwarp();
      if (lane == 0) {
        cnt[slot] = 0;
        __threadfence_block();
        atomicExch(&tag[slot], lt + kRing);
      }
    }
  }
  __syncthreads();
  // ---- flush the warp-private Z slices: Zpart[b][sidx][k][m][i]
  double* Zp = v.Zpart + ((int64_t)b * v.nsplit + sidx) * T * nu * nx;
  for (int r = threadIdx.x; r < T * nu * nx; r += blockDim.x) {
    const int k = r / (nu * nx), rem = r % (nu * nx), m = rem / nx, i = rem % nx;
    Zp[r] = Zs[((size_t)k * 8 + m) * ZW + i];
  }
}

// Register-resident variant (T <= 16 KK): 16 warps, warp w owns the blocks
// k == w (mod 16) of every tile, its Z_k slices (KK of them) live in
// registers, the k-loop is fully unrolled so the loads of later blocks are
// hoisted over the DMMA chains of earlier ones.  Shared memory holds only the
// norm ring, leaving L1 to cache the per-step D_k fragments and b rows.
template <int NTI, int NKS, int KK>
__global__ void __launch_bounds__(512, 1)
k_fa_fused_r(Dev v, const int32_t* __restrict__ tiles, const int32_t* __restrict__ witems) {
  constexpr int NW = 16;
  __shared__ double ring[kRing * NW * 8];
  __shared__ int cnt[kRing], tag[kRing];
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, T = d.T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int b = witems[4 * blockIdx.x], t0 = witems[4 * blockIdx.x + 1];
  const int t1 = witems[4 * blockIdx.x + 2], sidx = witems[4 * blockIdx.x + 3];
  if (!v.active[b]) return;
  if (threadIdx.x < kRing) { cnt[threadIdx.x] = 0; tag[threadIdx.x] = threadIdx.x; }
  __syncthreads();
  const double* __restrict__ bhat = v.bhat + (int64_t)b * d.E;
  const double* __restrict__ Bd = v.Bd + (int64_t)b * d.EB;
  const double* __restrict__ Dm = v.D + (int64_t)b * T * nx * nu;
  double* __restrict__ Y = v.Y + (int64_t)b * d.E;
  const int64_t bg = (int64_t)b * d.ng;
  const bool vec2 = (nx & 1) == 0;
  double z[KK][NTI][2];
#pragma unroll
  for (int kk = 0; kk < KK; ++kk)
#pragma unroll
    for (int nt = 0; nt < NTI; ++nt) { z[kk][nt][0] = 0.0; z[kk][nt][1] = 0.0; }

  for (int t = t0; t < t1; ++t) {
    const int* tl = tiles + (int64_t)t * kTileInts;
    const int kind = tl[0], K = tl[1], nc = tl[2], klo = tl[3];
    const int nblk = K - klo + 1;
    const int first = klo + ((warp - klo) % NW + NW) % NW;
    if (first > K) continue;
    const int lt = t - t0, slot = lt % kRing;
    const bool gv = g < nc;
    const int cg = gv ? tl[4 + g] : 0;
    const int64_t offg = gv ? v.off[cg] : 0, offBg = gv ? v.offB[cg] : 0;
    const double omsp = gv ? 1.0 - v.s[bg + cg] : 0.0;
    int64_t offB2[2];
    double sh2[2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int c2 = q + 4 * ks;
      const bool c2v = c2 < nc;
      const int cc = c2v ? tl[4 + c2] : 0;
      offB2[ks] = c2v ? v.offB[cc] : 0;
      sh2[ks] = c2v ? shat_of(v, v.s[bg + cc]) : 0.0;
    }
    double nrm = 0.0;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {     // absolute slot: k = warp + NW kk (Z slice z[kk])
      const int k = warp + NW * kk;
      if (k > K) break;
      if (k < klo) continue;
      const int kb = k - klo;
      const bool hasB = (kind == 0) ? (k < K) : true;
      const int kbB = (kind == 0) ? kb : 0;
      double c[NTI][2];
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) {
        const int i0 = 2 * q + 8 * nt;
        c[nt][0] = 0.0; c[nt][1] = 0.0;
        if (gv && i0 < nx) {
          const int64_t e = offg + (int64_t)kb * nx + i0;
          if (vec2) {
            const double2 yo = __ldcs(reinterpret_cast<const double2*>(Y + e));
            c[nt][0] = omsp * yo.x; c[nt][1] = omsp * yo.y;
            if (kind == 0) {
              const double2 bh = __ldcs(reinterpret_cast<const double2*>(bhat + e));
              c[nt][0] += bh.x; c[nt][1] += bh.y;
            }
          } else {
            c[nt][0] = omsp * Y[e] + (kind == 0 ? __ldg(bhat + e) : 0.0);
            if (i0 + 1 < nx) c[nt][1] = omsp * Y[e + 1] + (kind == 0 ? __ldg(bhat + e + 1) : 0.0);
          }
        }
      }
      double a[NKS], a2[2];
      if (hasB) {
#pragma unroll
        for (int ks = 0; ks < NKS; ++ks) {
          const int m = q + 4 * ks;
          a[ks] = (gv && m < nu) ? __ldg(Bd + offBg + (int64_t)kbB * d.nup + m) : 0.0;
        }
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
          a2[ks] = (g < nu && sh2[ks] != 0.0) ? sh2[ks] * __ldg(Bd + offB2[ks] + (int64_t)kbB * d.nup + g) : 0.0;
        const double* Dk = Dm + (int64_t)k * nx * nu;
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt) {
#pragma unroll
          for (int ks = 0; ks < NKS; ++ks) {
            const int m = q + 4 * ks, i = g + 8 * nt;
            const double bb = (m < nu && i < nx) ? __ldg(Dk + i * nu + m) : 0.0;
            dmma(c[nt], a[ks], bb);
          }
        }
      }
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) {
        const int i0 = 2 * q + 8 * nt;
        if (gv && i0 < nx) {
          const int64_t e = offg + (int64_t)kb * nx + i0;
          if (vec2) {
            __stcs(reinterpret_cast<double2*>(Y + e), make_double2(c[nt][0], c[nt][1]));
          } else {
            Y[e] = c[nt][0];
            if (i0 + 1 < nx) Y[e + 1] = c[nt][1];
          }
        }
        nrm += c[nt][0] * c[nt][0] + c[nt][1] * c[nt][1];
      }
      if (hasB) {
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const int src = (q + 4 * ks) * 4 + (g >> 1);
            const double v0 = __shfl_sync(0xffffffffu, c[nt][0], src);
            const double v1 = __shfl_sync(0xffffffffu, c[nt][1], src);
            dmma(z[kk][nt], a2[ks], (g & 1) ? v1 : v0);
          }
        }
      }
    }
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 1);
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 2);
    if (lane == 0) {
      while (atomicAdd(&tag[slot], 0) != lt) { __nanosleep(20); }
    }
    __syncwarp();
    if (q == 0) ring[(slot * NW + warp) * 8 + g] = nrm;
    __threadfence_block();
    __syncwarp();
    int last = 0;
    const int npart = nblk >= NW ? NW : nblk;
    if (lane == 0) last = (atomicAdd(&cnt[slot], 1) == npart - 1);
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence_block();
      if (lane < nc) {
        double n2 = 0.0;
        for (int w = 0; w < NW; ++w)
          if (((w - klo) % NW + NW) % NW <= K - klo) n2 += ring[(slot * NW + w) * 8 + lane];
        v.nrm2[bg + tl[4 + lane]] = n2;     // projection decided by k_project
      }
      __syncwarp();
      if (lane == 0) {
        cnt[slot] = 0;
        __threadfence_block();
        atomicExch(&tag[slot], lt + kRing);
      }
    }
  }
  // ---- flush this warp's Z slices: Zpart[b][sidx][k][m][i]  (row m = g, col i)
  double* Zp = v.Zpart + ((int64_t)b * v.nsplit + sidx) * T * nu * nx;
#pragma unroll
  for (int kk = 0; kk < KK; ++kk) {
    const int k = warp + NW * kk;
    if (k < T && g < nu) {
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = 2 * q + r + 8 * nt;
          if (i < nx) Zp[((int64_t)k * nu + g) * nx + i] = z[kk][nt][r];
        }
    }
  }
}

// Adjoint over a cone list, S7 / S7': Z_k = sum_{j in list} w_j b_{j,k} y_{j,k}^T.
// Correction of the fused pass (list = mispredicted cones, w = s^l - shat), or
// the dense adjoint (list = all cones, w = scale_j or 1) for the DR engine,
// nrto_gain_update and the generic path.  One CTA per (instance, step k);
// listed cones are staged in chunks of 64 through shared memory (b rows and
// y rows), then each thread owns outputs (m, i).  Requires n_u <= 8.
__global__ void __launch_bounds__(128)
k_zlist(Dev v, const double* __restrict__ y, const int32_t* __restrict__ clist,
        const double* __restrict__ cw, const double* __restrict__ scale,
        const int32_t* __restrict__ ncnt, int nfixed, const int32_t* __restrict__ act,
        double* __restrict__ Zout) {
  __shared__ double sb[64 * 8];
  __shared__ double sy[64 * 32];
  __shared__ double swt[64];
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu;
  const int b = blockIdx.x / d.T, k = blockIdx.x % d.T;
  double* Zo = Zout + ((int64_t)b * d.T + k) * nu * nx;
  if (act && !act[b]) return;
  const int n = ncnt ? ncnt[b] : nfixed;
  const int64_t bg = (int64_t)b * d.ng;
  const double* yb = y + (int64_t)b * d.E;
  const double* Bd = v.Bd + (int64_t)b * d.EB;
  const int tid = threadIdx.x;
  const int o0 = tid, o1 = tid + 128;
  double acc0 = 0.0, acc1 = 0.0;
  for (int base = 0; base < n; base += 64) {
    const int cnt = min(64, n - base);
    __syncthreads();
    for (int r = tid; r < cnt; r += blockDim.x) {
      const int j = clist ? clist[bg + base + r] : base + r;
      const int kind = v.kind[j], knot = v.knot[j];
      const bool has = (kind == 0) ? (knot > k) : (knot == k);
      const double w = cw ? cw[bg + base + r] : (scale ? scale[bg + j] : 1.0);
      swt[r] = has ? w : 0.0;
    }
    for (int r = tid; r < cnt * 8; r += blockDim.x) {
      const int c = r >> 3, mm = r & 7;
      const int j = clist ? clist[bg + base + c] : base + c;
      const int kind = v.kind[j], knot = v.knot[j];
      const bool has = (kind == 0) ? (knot > k) : (knot == k);
      const int kb = (kind == 0) ? k : 0;
      sb[r] = (has && mm < nu) ? Bd[v.offB[j] + (int64_t)kb * d.nup + mm] : 0.0;
    }
    for (int r = tid; r < cnt * 32; r += blockDim.x) {
      const int c = r >> 5, ii = r & 31;
      const int j = clist ? clist[bg + base + c] : base + c;
      const int kind = v.kind[j], knot = v.knot[j];
      const bool has = (kind == 0) ? (knot > k) : (knot == k);
      const int kb = (kind == 0) ? k : 0;
      sy[r] = (has && ii < nx) ? yb[v.off[j] + (int64_t)kb * nx + ii] : 0.0;
    }
    __syncthreads();
    if (o0 < nu * nx) {
      const int m = o0 / nx, i = o0 % nx;
      for (int c = 0; c < cnt; ++c) acc0 += swt[c] * sb[c * 8 + m] * sy[c * 32 + i];
    }
    if (o1 < nu * nx) {
      const int m = o1 / nx, i = o1 % nx;
      for (int c = 0; c < cnt; ++c) acc1 += swt[c] * sb[c * 8 + m] * sy[c * 32 + i];
    }
  }
  if (o0 < nu * nx) Zo[o0] = acc0;
  if (o1 < nu * nx) Zo[o1] = acc1;
}

// DMMA list adjoint: grid (B, ceil(T/16)), 16 warps, warp w owns step
// k = 16 blockIdx.y + w.  The warp walks the cone list 32 entries at a time,
// keeps (ballot) the cones that have a b-block at k, and folds them into
// Z_k with DMMA 8 cones at a time:
//   Z_k[m][i] += sum_c (w_c b_{c,k,m}) y_{c,k,i}   ([8 m x 4 c] x [4 c x 8 i]).
template <int NTI, int NTH = 512, int MINB = 1>
__global__ void __launch_bounds__(NTH, MINB)
k_zlist_mma(Dev v, const double* __restrict__ y, const int32_t* __restrict__ clist,
            const double* __restrict__ cw, const double* __restrict__ scale,
            const int32_t* __restrict__ ncnt, int nfixed, const int32_t* __restrict__ act,
            double* __restrict__ Zout, int lazy, int ghmode, double* __restrict__ dG,
            double* __restrict__ dH) {
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, nup = d.nup;
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int k = blockIdx.y * (blockDim.x >> 5) + warp;
  if (k >= d.T) return;
  if (act && !act[b]) return;
  // lazy y: entries flagged kRecompute were not stored by the pass
  // (s^{l-1} = 1 predicted s^l = 1); their block y_{c,k} = D_k b_{c,k} + b_hat_{c,k}
  // is rebuilt here from D_k and stored.
  // (rows i = g + 8 nt of D_k, read through L1 only by the rare rebuilt entries)
  const double* __restrict__ Dk = v.D + ((int64_t)b * d.T + k) * nx * nu;
  // dense mode (no list, every cone): walk the static per-step cone list
  // kcone[kptr[k] .. kptr[k+1]) -- exactly the cones with a b-block at k
  const bool dense = !clist && nfixed == d.ng;
  const int kp0 = dense ? v.kptr[k] : 0;
  const int n = ncnt ? ncnt[b] : (dense ? v.kptr[k + 1] - kp0 : nfixed);
  // blockIdx.z splits the list (small batches); partial sums are added atomically
  const int nsp = gridDim.z, sp = blockIdx.z;
  const int per = (((n + nsp - 1) / nsp) + 31) & ~31;
  const int lo = sp * per, hi = min(n, lo + per);
  const int64_t bg = (int64_t)b * d.ng;
  const double* yb = y ? y + (int64_t)b * d.E : nullptr;
  const double* Bd = v.Bd + (int64_t)b * d.EB;
  const double* bhb = v.bhat + (int64_t)b * d.E;
  // Z_k += sum_c w_c b_c y_c^T ; with ghmode also (sign s_c = +1 enter, -1 leave)
  // dG_k += sum_c s_c b_c b_c^T and dH_k += sum_c s_c b_c b_hat_c^T (state cones).
  double z[NTI][2], hz[NTI][2], gz[2] = {0.0, 0.0};
#pragma unroll
  for (int nt = 0; nt < NTI; ++nt) { z[nt][0] = z[nt][1] = 0.0; hz[nt][0] = hz[nt][1] = 0.0; }
  bool any = false;                     // this split saw a cone with a block at k
  for (int base = lo; base < hi; base += 32) {
    // lane l inspects entry base + l
    int j = 0, rec = 0, sgn = 0;
    double w = 0.0;
    bool has = false, hasg = false;
    if (base + lane < hi) {
      const int raw = clist ? clist[bg + base + lane] : (dense ? v.kcone[kp0 + base + lane] : base + lane);
      rec = (raw >> 30) & 1;
      sgn = ((raw >> 28) & 1) - ((raw >> 29) & 1);
      j = raw & kListMask;
      const int kind = v.kind[j], knot = v.knot[j];
      const bool blk = (kind == 0) ? (knot > k) : (knot == k);
      if (Zout) {
        w = cw ? cw[bg + base + lane] : (scale ? scale[bg + j] : 1.0);
        has = blk && (w != 0.0);
      }
      if (ghmode == 2) sgn = 1;
      hasg = ghmode && kind == 0 && blk && sgn != 0;
      if (!has) w = 0.0;
      if (!hasg) sgn = 0;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, has || hasg);
    const int nv = __popc(mask);
    any |= nv > 0;
    // per-lane row pointers of valid entries (computed by their owner lanes)
    int64_t yoff = 0, boff = 0;
    if (has || hasg) {
      const int kb = (v.kind[j] == 0) ? k : 0;
      yoff = v.off[j] + (int64_t)kb * nx;
      boff = v.offB[j] + (int64_t)kb * nup;
    }
    for (int g8 = 0; g8 < nv; g8 += 8) {
      // the (g8 + c)-th set bit of mask is cone c of this group
      double a2[2], ag[2], bb[2], bv[2][NTI], bh[2][NTI];
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int c = g8 + q + 4 * ks;                       // A2 / B2 column index
        int src = 0;
        if (c < nv) {                                         // lane of the c-th set bit
          unsigned mm = mask;
          for (int t = 0; t < c; ++t) mm &= mm - 1;
          src = __ffs(mm) - 1;
        }
        const int64_t yo = __shfl_sync(0xffffffffu, yoff, src);
        const int64_t bo = __shfl_sync(0xffffffffu, boff, src);
        const double ww = __shfl_sync(0xffffffffu, w, src);
        const int rc = __shfl_sync(0xffffffffu, rec, src);
        const int sg = __shfl_sync(0xffffffffu, sgn, src);
        const bool cv = c < nv;
        // b_{c,g}: A operand row m = g; also the G B-operand (row c, col m' = g)
        const double bcg = (cv && g < nu) ? Bd[bo + g] : 0.0;
        a2[ks] = ww * bcg;
        ag[ks] = (double)sg * bcg;
        bb[ks] = bcg;
        const bool rb = lazy && cv && rc;
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt) {
          const int i = g + 8 * nt;
          bh[ks][nt] = (cv && (sg != 0 || rb) && i < nx) ? bhb[yo + i] : 0.0;
        }
        if (rb) {
          double bm[8];
#pragma unroll
          for (int m = 0; m < 8; ++m) bm[m] = (m < nu) ? Bd[bo + m] : 0.0;
          double* yw = v.Y + (int64_t)b * d.E + yo;
#pragma unroll
          for (int nt = 0; nt < NTI; ++nt) {
            const int i = g + 8 * nt;
            double acc = 0.0;
            if (i < nx) {
#pragma unroll
              for (int m = 0; m < 8; ++m) acc += (m < nu) ? __ldg(Dk + i * nu + m) * bm[m] : 0.0;
              acc += bh[ks][nt];
              yw[i] = acc;
            }
            bv[ks][nt] = acc;
          }
        } else {
#pragma unroll
          for (int nt = 0; nt < NTI; ++nt) {
            const int i = g + 8 * nt;
            bv[ks][nt] = (cv && ww != 0.0 && i < nx) ? yb[yo + i] : 0.0;
          }
        }
      }
      if (Zout) {
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) dmma(z[nt], a2[ks], bv[ks][nt]);
      }
      if (ghmode) {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          dmma(gz, ag[ks], bb[ks]);
#pragma unroll
          for (int nt = 0; nt < NTI; ++nt) dmma(hz[nt], ag[ks], bh[ks][nt]);
        }
      }
    }
  }
  if (nsp > 1 && !any) return;         // slices pre-zeroed; nothing to add
  if (g < nu) {
    const int64_t bk = (int64_t)b * d.T + k;
    if (Zout) {
      double* Zo = Zout + bk * nu * nx;
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = 2 * q + r + 8 * nt;
          if (i < nx) {
            if (nsp == 1) Zo[g * nx + i] = z[nt][r];
            else atomicAdd(&Zo[g * nx + i], z[nt][r]);
          }
        }
    }
    if (ghmode) {                       // split: pre-zeroed, accumulated
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int m2 = 2 * q + r;
        if (m2 < nu) {
          if (nsp == 1) dG[bk * nu * nu + g * nu + m2] = gz[r];
          else atomicAdd(&dG[bk * nu * nu + g * nu + m2], gz[r]);
        }
      }
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = 2 * q + r + 8 * nt;
          if (i < nx) {
            if (nsp == 1) dH[bk * nu * nx + g * nx + i] = hz[nt][r];
            else atomicAdd(&dH[bk * nu * nx + g * nx + i], hz[nt][r]);
          }
        }
    }
  }
}

// ---------------------------------------------------------------------------
// S0 on tensor cores: costate sweep for a tile of <= 8 state cones with the
// same knot K (rows = cones), one warp per (instance, tile):
//   C_K = [grad_j]; for k = K..0:  b_k = C_{k+1} B_k,  C_k = C_{k+1} A_k,
//   b_hat_k = sqrt(tau) C_k Psi_k^T          (row form of P:846-866)
// as DMMA chains [8 cones x 4 r] x [4 r x 8 cols], contraction over n_x <= 16.
template <int NTI>
__device__ __forceinline__ void c_as_a(const double (&C)[NTI][2], int g, int q, double (&a)[4]) {
  // A operand [row g][col 4ks + q] of the accumulator-layout matrix C
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int col = 4 * ks + q;
    const int nt = col >> 3, src = g * 4 + ((col & 7) >> 1);
    double v0 = 0.0, v1 = 0.0;
#pragma unroll
    for (int t = 0; t < NTI; ++t) {
      const double x0 = __shfl_sync(0xffffffffu, C[t][0], src);
      const double x1 = __shfl_sync(0xffffffffu, C[t][1], src);
      if (t == nt) { v0 = x0; v1 = x1; }
    }
    a[ks] = (nt < NTI) ? ((col & 1) ? v1 : v0) : 0.0;
  }
}

template <int NTI>
__global__ void __launch_bounds__(256) k_costate_mma(Dev v, const int32_t* __restrict__ tiles,
                                                     int ntiles) {
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, nup = d.nup;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int64_t gw = (int64_t)blockIdx.x * 8 + warp;
  if (gw >= (int64_t)d.B * ntiles) return;
  const int b = (int)(gw / ntiles), t = (int)(gw % ntiles);
  const int* tl = tiles + (int64_t)t * 12;
  const int K = tl[1], nc = tl[2];
  const bool gv = g < nc;
  const int cg = gv ? tl[4 + g] : 0;
  const double st = sqrt(v.tau[b]);
  const double* A = v.A + (int64_t)b * d.T * nx * nx;
  const double* Bm = v.Bm + (int64_t)b * d.T * nx * nu;
  const double* Psi = v.Psi + (int64_t)b * (d.T + 1) * nx * nx;
  double* bh = v.bhat + (int64_t)b * d.E + (gv ? v.off[cg] : 0);
  double* Bd = v.Bd + (int64_t)b * d.EB + (gv ? v.offB[cg] : 0);
  // TMA path: also the tile-interleaved copies ([k][cone][.], tma.cu) -- same tiles
  const bool tl2 = v.fused == 2;
  double* bht = tl2 ? v.bhat_t + (int64_t)b * v.Est + v.ttb[2 * t] + g * nx : nullptr;
  double* bdt = tl2 ? v.Bd_t + (int64_t)b * v.EBst + v.ttb[2 * t + 1] + g * nup : nullptr;
  const double* grad = v.grad + ((int64_t)b * d.ng + cg) * nx;
  double C[NTI][2];
#pragma unroll
  for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int i = 2 * q + r + 8 * nt;
      C[nt][r] = (gv && i < nx) ? grad[i] : 0.0;
    }
  for (int k = K; k >= 0; --k) {
    double a[4];
    if (k < K) {
      c_as_a<NTI>(C, g, q, a);                        // C = c_{k+1} rows
      const double* Bk = Bm + (int64_t)k * nx * nu;
      const double* Ak = A + (int64_t)k * nx * nx;
      double bb[2] = {0.0, 0.0};
      double Cn[NTI][2];
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) { Cn[nt][0] = 0.0; Cn[nt][1] = 0.0; }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int r = 4 * ks + q;
        const double bop = (r < nx && g < nu) ? __ldg(Bk + r * nu + g) : 0.0;
        dmma(bb, a[ks], bop);
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt) {
          const int i = g + 8 * nt;
          const double aop = (r < nx && i < nx) ? __ldg(Ak + r * nx + i) : 0.0;
          dmma(Cn[nt], a[ks], aop);
        }
      }
      if (gv) {                                        // b_k row (padded to nup)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int m = 2 * q + rr;
          if (m < nup) {
            const double val = (m < nu) ? bb[rr] : 0.0;
            Bd[(int64_t)k * nup + m] = val;
            if (tl2) bdt[(int64_t)k * nc * nup + m] = val;
          }
        }
      }
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) { C[nt][0] = Cn[nt][0]; C[nt][1] = Cn[nt][1]; }
    }
    c_as_a<NTI>(C, g, q, a);                          // C = c_k rows
    const double* Pk = Psi + (int64_t)k * nx * nx;
    double h[NTI][2];
#pragma unroll
    for (int nt = 0; nt < NTI; ++nt) { h[nt][0] = 0.0; h[nt][1] = 0.0; }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int r = 4 * ks + q;
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) {
        const int i = g + 8 * nt;
        const double pop = (r < nx && i < nx) ? __ldg(Pk + i * nx + r) : 0.0;   // Psi_k^T
        dmma(h[nt], a[ks], pop);
      }
    }
    if (gv) {
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int i = 2 * q + rr + 8 * nt;
          if (i < nx) {
            bh[(int64_t)k * nx + i] = st * h[nt][rr];
            if (tl2) bht[(int64_t)k * nc * nx + i] = st * h[nt][rr];
          }
        }
    }
  }
}

// Control cones for the MMA setup path: b = h'_j (padded), b_hat row = 0.
__global__ void k_costate_ctrl(Dev v) {
  const Dims d = v.d;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)d.B * d.ng) return;
  const int b = (int)(id / d.ng), j = (int)(id % d.ng);
  if (v.kind[j] == 0) return;
  const double* grad = v.grad + ((int64_t)b * d.ng + j) * d.nx;
  double* Bd = v.Bd + (int64_t)b * d.EB + v.offB[j];
  double* bh = v.bhat + (int64_t)b * d.E + v.off[j];
  for (int m = 0; m < d.nup; ++m) Bd[m] = (m < d.nu) ? grad[m] : 0.0;
  for (int i = 0; i < d.nx; ++i) bh[i] = 0.0;
}

// Lambda_k = sum_j b_{j,k} b_{j,k}^T over the cones with a b-block at k, DMMA
// [8 m x 4 c] x [4 c x 8 m'] per 8 cones (same walk as k_zlist_mma).
__global__ void __launch_bounds__(512) k_lam_mma(Dev v) {
  const Dims d = v.d;
  const int nu = d.nu, nup = d.nup;
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int k = blockIdx.y * 16 + warp;
  if (k >= d.T) return;
  const double* Bd = v.Bd + (int64_t)b * d.EB;
  double z[2] = {0.0, 0.0};
  for (int base = v.kptr[k]; base < v.kptr[k + 1]; base += 8) {
    const int cnt = min(8, v.kptr[k + 1] - base);
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int c = q + 4 * ks;
      double a2 = 0.0, bv = 0.0;
      if (c < cnt) {
        const int j = v.kcone[base + c];
        const int kb = (v.kind[j] == 0) ? k : 0;
        const double* row = Bd + v.offB[j] + (int64_t)kb * nup;
        a2 = (g < nu) ? row[g] : 0.0;
        bv = (g < nu) ? row[g] : 0.0;
      }
      dmma(z, a2, bv);
    }
  }
  if (g < nu) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int m2 = 2 * q + r;
      if (m2 < nu) v.Lam[((int64_t)b * d.T + k) * nu * nu + g * nu + m2] = z[r];
    }
  }
}

cudaError_t launch_setup_mma(nrto_handle_s* h, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  const int nst = v.nstate_tiles;
  if ((int64_t)d.B * d.ng > 0) {
    k_costate_ctrl<<<(unsigned)(((int64_t)d.B * d.ng + 255) / 256), 256, 0, st>>>(v);
    h->launches++;
  }
  if (nst > 0) {
    const int64_t nw = (int64_t)d.B * nst;
    if (d.nx <= 8)
      k_costate_mma<1><<<(unsigned)((nw + 7) / 8), 256, 0, st>>>(v, v.tiles, nst);
    else
      k_costate_mma<2><<<(unsigned)((nw + 7) / 8), 256, 0, st>>>(v, v.tiles, nst);
    h->launches++;
  }
  dim3 grid(d.B, (d.T + 15) / 16);
  k_lam_mma<<<grid, 512, 0, st>>>(v);
  h->launches++;
  if (v.fused != 2) {
    // Zb_k = sum_j b_{j,k} b_hat_{j,k}^T : the list adjoint with y = b_hat
    return launch_zlist(h, v.bhat, nullptr, nullptr, nullptr, nullptr, d.ng, nullptr, v.Zb, st);
  }
  // TMA path: G0 = sum b b^T, H0 = sum b b_hat^T over state cones
  // from it; control rows have b_hat = 0, so Zb = H0.
  return launch_gram_tiles(h, st);   // the tile layout was written by k_costate_mma
}

static int fused_variant(const Dims& d, int* nti, int* nks) {
  *nti = (d.nx + 7) / 8;
  *nks = (d.nu + 3) / 4;
  return (*nti <= 2 && *nks <= 2);
}

size_t fused_smem_bytes(const Dims& d) {
  const int nti = (d.nx + 7) / 8;
  return ((size_t)d.T * 8 * 8 * nti + kRing * 64) * sizeof(double) + 2 * kRing * sizeof(int);
}

bool fused_supported(const Dims& d) {
  int a, c;
  return fused_variant(d, &a, &c) && fused_smem_bytes(d) <= 200 * 1024;
}

template <int NTI, int NKS>
static cudaError_t launch_fused_t(nrto_handle_s* h, cudaStream_t st) {
  const size_t smem = fused_smem_bytes(h->dev.d);
  auto kfn = k_fa_fused<NTI, NKS>;
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kfn<<<h->dev.nwitems, 256, smem, st>>>(h->dev, h->dev.tiles, h->dev.witems);
  h->launches++;
  return cudaGetLastError();
}

template <int NTI, int NKS, int KK>
static cudaError_t launch_fused_r(nrto_handle_s* h, cudaStream_t st) {
  k_fa_fused_r<NTI, NKS, KK><<<h->dev.nwitems, 512, 0, st>>>(h->dev, h->dev.tiles, h->dev.witems);
  h->launches++;
  return cudaGetLastError();
}

template <int KK>
static cudaError_t launch_fused_rk(nrto_handle_s* h, int nti, int nks, cudaStream_t st) {
  if (nti == 1 && nks == 1) return launch_fused_r<1, 1, KK>(h, st);
  if (nti == 1 && nks == 2) return launch_fused_r<1, 2, KK>(h, st);
  if (nti == 2 && nks == 1) return launch_fused_r<2, 1, KK>(h, st);
  return launch_fused_r<2, 2, KK>(h, st);
}

cudaError_t launch_fa_fused(nrto_handle_s* h, cudaStream_t st) {
  int nti, nks;
  fused_variant(h->dev.d, &nti, &nks);
  if (h->dev.nwitems == 0) return cudaSuccess;
  const int T = h->dev.d.T;
  if (T <= 32) return launch_fused_rk<2>(h, nti, nks, st);
  if (T <= 64) return launch_fused_rk<4>(h, nti, nks, st);
  if (T <= 112) return launch_fused_rk<7>(h, nti, nks, st);
  if (nti == 1 && nks == 1) return launch_fused_t<1, 1>(h, st);
  if (nti == 1 && nks == 2) return launch_fused_t<1, 2>(h, st);
  if (nti == 2 && nks == 1) return launch_fused_t<2, 1>(h, st);
  return launch_fused_t<2, 2>(h, st);
}

__global__ void k_zero_active(double* Z, int64_t per, int B, const int32_t* act) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)B * per) return;
  if (act && !act[id / per]) return;
  Z[id] = 0.0;
}

cudaError_t launch_zlist(nrto_handle_s* h, const double* y, const int32_t* clist, const double* cw,
                         const double* scale, const int32_t* ncnt, int nfixed, const int32_t* act,
                         double* Zout, cudaStream_t st, int lazy, int ghmode, double* dG,
                         double* dH, int prezeroed) {
  Dev& v = h->dev;
  if (v.d.nu <= 8 && v.d.nx <= 16) {
    // split the list when the batch alone cannot fill the GPU (dense lists only)
    int nsp = 1;
    if (!ncnt && nfixed > 256 && !ghmode) {
      // fixed (dense) lists, small batches (e.g. one DR instance): split each step's
      // list until the grid has ~32 warps per SM, keeping >= 8 entries per split
      // (measured on c2: 8 -> 32 splits, adjoint 29 -> 16 us per DR iteration)
      const int64_t warps = (int64_t)v.d.B * v.d.T;
      const int64_t navg = std::max<int64_t>(1, nfixed / 2);
      // long lists (one huge instance, c4 T = 800: ~83 k cones per step) keep splitting
      // past the warp target while a split still walks >= 1024 entries (measured
      // at c4 T = 800: 2 -> 64 splits, DR adjoint 11.8 -> 5.6 ms)
      while (nsp < 64 && navg / (nsp * 2) >= 8 &&
             (warps * nsp * 2 <= 32 * v.nsm || navg / (nsp * 2) >= 1024)) nsp *= 2;
      static const int dsp = [] { const char* e = getenv("NRTO_ZLIST_DSPLIT"); return e ? atoi(e) : 0; }();
      if (dsp > 0) nsp = dsp;
    }
    // device-sized lists (TMA path): a fixed split so that long lists (early
    // iterations: most cones in case 3) are walked by nsp warps per step; splits
    // past the list end exit at once, empty splits add nothing
    static const int lsp = [] { const char* e = getenv("NRTO_ZLIST_SPLIT"); return e ? atoi(e) : 0; }();
    if (ncnt && ghmode && lsp > 1) nsp = lsp;
    if (ncnt && ghmode && lsp == 0) {
      // small batches (latency bound, e.g. one c3 instance): split the list until the
      // grid has ~32 warps per SM; the bench batch (B T >= 32 x 148 warps) stays unsplit
      const int64_t warps = (int64_t)v.d.B * v.d.T;
      // a few huge instances (c4 T = 800: 166 k cones, most of them on the list in
      // the first iterations) keep splitting while a split may hold >= 2048 cones
      while (nsp < 32 && (warps * nsp * 2 <= 32 * v.nsm ||
                          (v.d.B <= 4 && (int64_t)v.d.ng / (nsp * 2) >= 2048)))
        nsp *= 2;
    }
    if (nsp > 1 && !prezeroed) {   // zero the slices of the instances that will be accumulated
      const int64_t per = (int64_t)v.d.T * v.d.nu * v.d.nx;
      k_zero_active<<<(unsigned)(((int64_t)v.d.B * per + 255) / 256), 256, 0, st>>>(Zout, per, v.d.B, act);
      h->launches++;
      if (ghmode) {
        const int64_t pg = (int64_t)v.d.T * v.d.nu * v.d.nu;
        k_zero_active<<<(unsigned)(((int64_t)v.d.B * pg + 255) / 256), 256, 0, st>>>(dG, pg, v.d.B, act);
        k_zero_active<<<(unsigned)(((int64_t)v.d.B * per + 255) / 256), 256, 0, st>>>(dH, per, v.d.B, act);
        h->launches += 2;
      }
    }
    // warps (steps) per CTA: small CTAs fit beside the co-resident QP CTAs
    static const int zw0 = [] { const char* e = getenv("NRTO_ZLIST_WARPS"); return e ? atoi(e) : 4; }();
    const int zw = (nsp > 1) ? 2 : zw0;              // split lists: 2-warp CTAs spread wider
    dim3 grid(v.d.B, (v.d.T + zw - 1) / zw, nsp);
    // NRTO_ZLIST_WARPS = 4: 128-thread CTAs; NRTO_ZLIST_MINB = 8 / 6: capped at 64 / 80 registers
    static const int zmb = [] { const char* e = getenv("NRTO_ZLIST_MINB"); return e ? atoi(e) : 8; }();
    if (v.d.nx <= 8)
      k_zlist_mma<1><<<grid, 32 * zw, 0, st>>>(v, y, clist, cw, scale, ncnt, nfixed, act, Zout, lazy, ghmode, dG, dH);
    else if (zw == 2)
      k_zlist_mma<2, 64, 16><<<grid, 64, 0, st>>>(v, y, clist, cw, scale, ncnt, nfixed, act, Zout, lazy, ghmode, dG, dH);
    else if (zw == 4 && zmb == 8)
      k_zlist_mma<2, 128, 8><<<grid, 128, 0, st>>>(v, y, clist, cw, scale, ncnt, nfixed, act, Zout, lazy, ghmode, dG, dH);
    else if (zw == 4 && zmb == 6)
      k_zlist_mma<2, 128, 6><<<grid, 128, 0, st>>>(v, y, clist, cw, scale, ncnt, nfixed, act, Zout, lazy, ghmode, dG, dH);
    else
      k_zlist_mma<2><<<grid, 32 * zw, 0, st>>>(v, y, clist, cw, scale, ncnt, nfixed, act, Zout, lazy, ghmode, dG, dH);
    h->launches++;
    return cudaGetLastError();
  }
  if (ghmode || lazy) return cudaErrorInvalidValue;   // TMA path only (n_x <= 16, n_u <= 8)
  k_zlist<<<v.d.B * v.d.T, 128, 0, st>>>(v, y, clist, cw, scale, ncnt, nfixed, act, Zout);
  h->launches++;
  return cudaGetLastError();
}

}  // namespace nrto
