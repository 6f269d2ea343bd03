// TMA-pipelined fused FullADMM pass for STATE cones (n_x even) and the exact
// single-block pass for CONTROL cones.  Same arithmetic as k_fa_fused_r
// (fused.cu); the difference is how bytes reach the SM:
//
//  * a producer warp streams each chunk (one tile of <= 8 same-knot cones x 16
//    consecutive time blocks) of y_old, b_hat and b from HBM into a 3-stage
//    shared-memory ring with cp.async.bulk (TMA, SASS UBLKCP) completing on an
//    mbarrier with a transaction count;
//  * 16 consumer warps (warp w <-> block k = kc + w, so the adjoint slice Z_k
//    stays in warp w's registers) run the DMMA forward map / predicted adjoint
//    from shared memory and store y_new straight to HBM;
//  * D_k for the whole horizon is copied to shared memory once per work item.
//
// Control cones have a single time block, so their norm, projection and exact
// adjoint contribution s b y^T are completed inside one warp (k_fa_ctrl).
#include "common.cuh"
#include <algorithm>
#include <cstdlib>

namespace nrto {

__device__ __forceinline__ void dmma2(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) { dmma2(c, a, b); }
__device__ __forceinline__ uint32_t saddr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
// Streaming (read-once) TMA load: L2 evict-first policy so the 30 GB/iteration
// cone stream does not flush the concurrently running QP's working set.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_keep(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}

#ifndef TMA_NW
#define TMA_NW 16
#endif
constexpr int kMaxStages = 8;
constexpr int kRingT = 4;
constexpr int kTI = 12;   // ints per tile
constexpr int kHdr = 32;  // header doubles: 2 kMaxStages barriers + cnt/tag

struct TmaGeom {          // shared-memory geometry of one stage (doubles)
  int SY;                 // b_hat region: 16 blocks x 8 cones x n_x, block-major
  int SB;                 // b region: 16 blocks x 8 cones x nup
  int SD;                 // D region (streamed-D variant): 16 blocks x n_x x n_u
  int stage;              // doubles per stage (SY is a multiple of 16 doubles)
};
__host__ __device__ inline TmaGeom tma_geom(int nx, int nup, int nu = 0, bool ds = false) {
  TmaGeom g;
  g.SY = (16 * 8 * nx + 15) & ~15;
  g.SB = 16 * 8 * nup;
  g.SD = ds ? ((16 * nx * nu + 15) & ~15) : 0;
  g.stage = g.SY + g.SB + g.SD;
  return g;
}
// Per-tile metadata staged by the producer in shared memory (kMetaT-slot ring,
// tile t -> slot t % kMetaT), visible to the consumers once they pass the
// tile's first stage barrier (the producer's arrive releases it).
constexpr int kMetaT = 16;
struct TileMeta {
  int K, nc;
  int cone[8];
  int wy[8];
  long long off[8];
  double omsp[8];
  double pad[7];
};
static_assert(sizeof(TileMeta) == 256, "TileMeta is 32 doubles");
// ds: D_k is streamed per chunk through the stages (long horizons) instead of being
// resident in shared memory for the whole horizon
__host__ __device__ inline size_t tma_fixed_doubles(int T, int nx, int nu, bool ds = false) {
  return kHdr + kRingT * 16 * 8 + kMetaT * 32 + (ds ? 0 : (((size_t)T * nx * nu + 1) & ~(size_t)1));
}

// Fused state-cone pass (norm-only form).  Per cone block k:
//   y^l_k = D_k b_k + b_hat_k + (1 - s^{l-1}) y^{l-1}_k,  ||y^l||^2 accumulated,
// y^l stored where a later step reads it (lazy y).  The adjoint is not formed
// here: Z_pred = G D^T + H (k_fa_gain_w) plus the exact list correction.
// b_hat and b reach shared memory by TMA bulk copies (producer warp, nst-stage
// mbarrier ring); y^{l-1} of the few cones with s^{l-1} != 1 is loaded by the
// consumers straight from global memory, issued before the stage wait.
// NXE, NUE > 0: exact n_x, n_u fixed at compile time (benchmark shapes): every
// bounds predicate of the inner block folds away.
template <int NTI, int NKS, int KK, int NXE, int NUE, int NW = 16, bool DS = false>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
k_fa_tma(Dev v, const int32_t* __restrict__ tiles, const int32_t* __restrict__ witems, int nst,
         int margin) {
  extern __shared__ __align__(128) double sm[];
  constexpr int CH = 16;          // blocks per chunk (stage)
  constexpr int BPW = CH / NW;    // blocks per consumer warp per chunk
  const Dims d = v.d;
  const int nx = NXE > 0 ? NXE : d.nx, nu = NUE > 0 ? NUE : d.nu, T = d.T;
  const int nup = NUE > 0 ? (NUE + (NUE & 1)) : d.nup;
  const TmaGeom G = tma_geom(nx, nup, nu, DS);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + kMaxStages;
  int* cnt = reinterpret_cast<int*>(empty + kMaxStages);
  int* tag = cnt + kRingT;
  double* ring = sm + kHdr;                                // [kRingT][NW][8]
  TileMeta* meta = reinterpret_cast<TileMeta*>(ring + kRingT * NW * 8);   // [kMetaT]
  double* Ds = ring + kRingT * NW * 8 + kMetaT * 32;       // [T][nx][nu]
  double* stg = sm + tma_fixed_doubles(T, nx, nu, DS);     // stages
  const double* __restrict__ Dg = (margin ? v.Ccur : v.D) + (int64_t)witems[4 * blockIdx.x] * T * nx * nu;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int b = witems[4 * blockIdx.x], t0 = witems[4 * blockIdx.x + 1];
  const int t1 = witems[4 * blockIdx.x + 2];
  if (!margin && !v.active[b]) return;
  double* __restrict__ Y = v.Y + (int64_t)b * d.E;
  const int64_t bg = (int64_t)b * d.ng;
  if (!DS) {
    // margin mode (finish): ||C^L_k b + b_hat|| of every state cone, no history, no store
    for (int r = threadIdx.x; r < T * nx * nu; r += blockDim.x) Ds[r] = Dg[r];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < kRingT) { cnt[threadIdx.x] = 0; tag[threadIdx.x] = threadIdx.x; }
  __syncthreads();

  if (warp == NW) {
    // ---------------------------------------------------------------- producer
    // lane c < nc owns cone c of the tile: its offsets are loaded once per tile
    // (one tile ahead) and it issues that cone's bulk copies; lane 0 arms the
    // stage barrier and counts the algorithmic bytes of the launch.
    int st = 0;
    uint32_t ph = 0;
    unsigned long long moved = 0;
    const uint64_t pol = policy_evict_first();
    // per-lane prefetch (one tile ahead) of the cone id, offset, s^{l-1}
    int jn = 0, Kn = 0, ncn = 0;
    long long offn = 0;
    double sn = 1.0;
    auto fetch = [&](int t) {
      const int* tl = tiles + (int64_t)t * kTI;
      Kn = tl[1]; ncn = tl[2];
      if (lane < ncn) { jn = tl[4 + lane]; offn = v.off[jn]; sn = v.s[bg + jn]; }
    };
    if (t0 < t1) fetch(t0);
    const double* __restrict__ bht = v.bhat_t + (int64_t)b * v.Est;
    const double* __restrict__ bdt = v.Bd_t + (int64_t)b * v.EBst;
    for (int t = t0; t < t1; ++t) {
      const int K = Kn, nc = ncn, jc = jn;
      const long long offc = offn;
      const double sc = sn;
      const int64_t tb0 = v.ttb[2 * t], tb1 = v.ttb[2 * t + 1];
      if (t + 1 < t1) fetch(t + 1);
      const bool yrd = !margin && lane < nc && v.iter > 1 && sc != 1.0;
      const bool ywr = !margin && lane < nc && (!v.ylazy || shat_of(v, sc) != 1.0);
      TileMeta* M = meta + ((t - t0) & (kMetaT - 1));
      if (lane < 8) {
        M->cone[lane] = jc;
        M->off[lane] = offc;
        M->omsp[lane] = yrd ? 1.0 - sc : 0.0;
        M->wy[lane] = ywr;
      }
      if (lane == 0) { M->K = K; M->nc = nc; }
      __syncwarp();
      const uint32_t nyr = __popc(__ballot_sync(0xffffffffu, yrd));
      const uint32_t nyw = __popc(__ballot_sync(0xffffffffu, ywr));
      for (int kc = 0; kc <= K; kc += 16) {
        const int nb = min(16, K + 1 - kc), nbB = max(0, min(16, K - kc));
        if (lane == 0) {
          mbar_wait(&empty[st], ph ^ 1);
          const uint32_t hb = (uint32_t)nc * nb * nx * 8u, bb = (uint32_t)nc * nbB * nup * 8u;
          const uint32_t db = DS ? (uint32_t)nbB * nx * nu * 8u : 0u;
          mbar_expect_tx(&full[st], hb + bb + db);
          moved += hb + bb + (unsigned long long)(nyr + nyw) * nb * nx * 8u;
          double* sH = stg + (size_t)st * G.stage;
          double* sB = sH + G.SY;
          // one bulk copy per array: the chunk is contiguous in the tile layout
          bulk_g2s(sH, bht + tb0 + (int64_t)kc * nc * nx, hb, &full[st], pol);
          if (bb > 0) bulk_g2s(sB, bdt + tb1 + (int64_t)kc * nc * nup, bb, &full[st], pol);
          // D_k of the chunk's blocks (re-read by every tile of the instance: L2 hits)
          if (DS && db > 0) bulk_g2s_keep(sB + G.SB, Dg + (int64_t)kc * nx * nu, db, &full[st]);
        }
        __syncwarp();
        if (++st == nst) { st = 0; ph ^= 1; }
      }
    }
    if (lane == 0 && v.pass_bytes && !margin) atomicAdd(v.pass_bytes, moved);
    return;
  }
  // ------------------------------------------------------------------ consumers
  int st = 0;
  uint32_t ph = 0;
  for (int t = t0; t < t1; ++t) {
    const int lt = t - t0, slot = lt % kRingT;
    mbar_wait(&full[st], ph);                     // first stage of the tile: meta visible
    const TileMeta* M = meta + (lt & (kMetaT - 1));
    const int K = M->K, nc = M->nc;
    const bool gv = g < nc;
    const int64_t offg = gv ? M->off[g] : 0;
    const double omsp = gv ? M->omsp[g] : 0.0;    // != 0 <=> y_old is read
    const bool wy = gv && M->wy[g];               // store y^l
    const bool hist = __any_sync(0xffffffffu, omsp != 0.0);     // any y_old in this tile
    double nrm = 0.0;
    // y_old of history cones (s^{l-1} != 1) comes from global memory; each
    // chunk's loads are issued one chunk ahead so their latency overlaps the
    // previous chunk's work
    double2 yo[BPW][NTI], yn[BPW][NTI];
    auto load_y = [&](double2 (&dst)[NTI], int kb) {
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) {
        const int i0 = 2 * q + 8 * nt;
        dst[nt] = make_double2(0.0, 0.0);
        if (kb <= K && omsp != 0.0 && i0 < nx)
          dst[nt] = __ldcs(reinterpret_cast<const double2*>(Y + offg + (int64_t)kb * nx + i0));
      }
    };
    if (hist) {
#pragma unroll
      for (int bb = 0; bb < BPW; ++bb) load_y(yo[bb], warp + NW * bb);
    }
    constexpr int KU = KK <= 26 ? KK : 1;
#pragma unroll KU
    for (int kk = 0; kk < KK; ++kk) {
      const int kc = CH * kk;
      if (kc > K) break;
      if (hist && kc + CH <= K) {
#pragma unroll
        for (int bb = 0; bb < BPW; ++bb) load_y(yn[bb], kc + CH + warp + NW * bb);
      }
      if (kk > 0) mbar_wait(&full[st], ph);
      const double* sH = stg + (size_t)st * G.stage;
      const double* sB = sH + G.SY;
#pragma unroll
      for (int bb = 0; bb < BPW; ++bb) {
        const int lb = warp + NW * bb;            // block within the chunk
        const int k = kc + lb;
        if (k > K) continue;
        double c[NTI][2];
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt) {
          const int i0 = 2 * q + 8 * nt;
          c[nt][0] = 0.0; c[nt][1] = 0.0;
          if (gv && i0 < nx) {
            const double2 bh = *reinterpret_cast<const double2*>(sH + (lb * nc + g) * nx + i0);
            if (hist) {
              c[nt][0] = bh.x + omsp * yo[bb][nt].x;
              c[nt][1] = bh.y + omsp * yo[bb][nt].y;
            } else {
              c[nt][0] = bh.x;
              c[nt][1] = bh.y;
            }
          }
        }
        if (k < K) {
#pragma unroll
          for (int ks = 0; ks < NKS; ++ks) {
            const int m = q + 4 * ks;
            const double a = (gv && m < nu) ? sB[(lb * nc + g) * nup + m] : 0.0;
#pragma unroll
            for (int nt = 0; nt < NTI; ++nt) {
              const int i = g + 8 * nt;
              const double bq = (m < nu && i < nx)
                                    ? (DS ? sB[G.SB + ((size_t)lb * nx + i) * nu + m]
                                          : Ds[((size_t)k * nx + i) * nu + m])
                                    : 0.0;
              dmma2(c[nt], a, bq);
            }
          }
        }
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt) {
          const int i0 = 2 * q + 8 * nt;
          if (wy && i0 < nx)
            __stcs(reinterpret_cast<double2*>(Y + offg + (int64_t)k * nx + i0),
                   make_double2(c[nt][0], c[nt][1]));
          nrm += c[nt][0] * c[nt][0] + c[nt][1] * c[nt][1];
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == nst) { st = 0; ph ^= 1; }
      if (hist) {
#pragma unroll
        for (int bb = 0; bb < BPW; ++bb)
#pragma unroll
          for (int nt = 0; nt < NTI; ++nt) yo[bb][nt] = yn[bb][nt];
      }
    }
    // ---- norm partials -> ring slot; last consumer warp publishes the tile's norms
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 1);
    nrm += __shfl_xor_sync(0xffffffffu, nrm, 2);
    if (lane == 0) {
      while (atomicAdd(&tag[slot], 0) != lt) { __nanosleep(32); }
    }
    __syncwarp();
    if (q == 0) ring[(slot * NW + warp) * 8 + g] = nrm;
    __threadfence_block();
    __syncwarp();
    int last = 0;
    if (lane == 0) last = (atomicAdd(&cnt[slot], 1) == NW - 1);
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence_block();
      if (lane < nc) {
        double n2 = 0.0;
        for (int w = 0; w < NW; ++w) n2 += ring[(slot * NW + w) * 8 + lane];
        v.nrm2[bg + M->cone[lane]] = n2;    // projection decided by k_project
      }
      __syncwarp();
      if (lane == 0) {
        cnt[slot] = 0;
        __threadfence_block();
        atomicExch(&tag[slot], lt + kRingT);
      }
    }
  }
}

// Control cones (single block at step k): y = D_k h' + (1 - s) y_old, ||y||^2,
// and the predicted adjoint Zctrl_k = sum_{ctrl j@k} shat_j h'_j y_j^T
// (k_project appends mispredicted cones to the correction list).
// One warp per step; lane i < n_x holds y_i; Z_k[:, i] accumulates in lane i.
__global__ void __launch_bounds__(512)
k_fa_ctrl(Dev v) {
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu;
  const int b = blockIdx.x;
  if (!v.active[b]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.y * (blockDim.x >> 5) + warp;
  if (k >= d.T) return;
  const int64_t bg = (int64_t)b * d.ng;
  const double* Dk = v.D + ((int64_t)b * d.T + k) * nx * nu;
  double* Y = v.Y + (int64_t)b * d.E;
  const double* Bd = v.Bd + (int64_t)b * d.EB;
  double zc[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) zc[m] = 0.0;
  double drow[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) drow[m] = (lane < nx && m < nu) ? Dk[lane * nu + m] : 0.0;
  const int q0 = v.cptr[k], q1 = v.cptr[k + 1];
  for (int qb = q0; qb < q1; qb += 32) {
    // lane c holds the metadata of cone qb + c (all loads issued together)
    int64_t offc = 0, offBc = 0;
    double sc = 1.0;
    int jc = 0;
    if (qb + lane < q1) {
      jc = v.crow[qb + lane];
      offc = v.off[jc]; offBc = v.offB[jc]; sc = v.s[bg + jc];
    }
    const int nq = min(32, q1 - qb);
    for (int c = 0; c < nq; ++c) {
      const int64_t off = __shfl_sync(0xffffffffu, offc, c);
      const int64_t offB = __shfl_sync(0xffffffffu, offBc, c);
      const double sj = __shfl_sync(0xffffffffu, sc, c);
      const int j = __shfl_sync(0xffffffffu, jc, c);
      const double* bj = Bd + offB;
      double bm[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) bm[m] = (m < nu) ? bj[m] : 0.0;
      double y = 0.0;
      if (lane < nx) {
        // history term (1 - s^{l-1}) y^{l-1}; at l = 1 it is lam_nu^0 = 0 by definition
        y = (v.iter > 1 && sj != 1.0) ? (1.0 - sj) * Y[off + lane] : 0.0;
#pragma unroll
        for (int m = 0; m < 8; ++m) y += drow[m] * bm[m];
        Y[off + lane] = y;
      }
      const double n2 = warp_sum(y * y);
      const double sh = shat_of(v, sj);          // predicted scale (k_project corrects)
      if (lane == 0) v.nrm2[bg + j] = n2;
#pragma unroll
      for (int m = 0; m < 8; ++m) zc[m] += sh * bm[m] * y;
    }
  }
  if (lane < nx) {
    double* Zo = v.Zctrl + ((int64_t)b * d.T + k) * nu * nx;
    for (int m = 0; m < nu; ++m) Zo[m * nx + lane] = zc[m];
  }
}

// Projection of every cone of the batch from its ||y^l||^2 (SM Eq.(18)):
// s^l, p~^l; cones whose s^l differs from the prediction shat used by the
// pass (shat_of(s^{l-1})) go to the correction list with weight s^l - shat.
// Runs after QP(l-1) (it needs t = p^{l-1} + lam_p^{l-1}).
__global__ void k_project(Dev v) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)v.d.B * v.d.ng;
  if (id >= n) return;
  const int b = (int)(id / v.d.ng), j = (int)(id % v.d.ng);
  if (!v.active[b]) return;
  const double shat = shat_of(v, v.s[id]);
  double s;
  const double tp = soc_case(v.tin[id], sqrt(v.nrm2[id]), &s);
  v.s[id] = s;
  v.pt[id] = tp;
  count_case(v, s);
  // TMA path: state cones leaving / entering the interior set {s = 1} update
  // the Gram sums G, H of the predicted adjoint.
  // At l = 1 the interior set restarts from empty (the gain kernel replaces G, H by
  // this iteration's updates), so only the cones with s^1 = 1 are listed (enter).
  const bool gh = v.fused == 2 && v.kind[j] == 0;
  const bool first = v.iter == 1;
  const bool leave = gh && !first && shat == 1.0 && s != 1.0;
  const bool enter = gh && s == 1.0 && (first || shat == 0.0);
  if (s != shat || leave) {
    // lazy y: a state cone predicted interior (shat = 1) was not stored by the
    // pass; flag it so the correction rebuilds y^l (blocks k < K there, the
    // b-free last block y_K = b_hat_K here).
    const bool rec = v.ylazy && leave;
    const int pos = atomicAdd(&v.ncorr[b], 1);
    v.clist[(int64_t)b * v.d.ng + pos] = j | (rec ? kRecompute : 0) | (leave ? kLeave : 0) |
                                         (enter ? kEnter : 0);
    v.cw[(int64_t)b * v.d.ng + pos] = s - shat;
    if (rec) {
      const int64_t o = (int64_t)b * v.d.E + v.off[j] + (int64_t)v.knot[j] * v.d.nx;
      for (int i = 0; i < v.d.nx; ++i) v.Y[o + i] = v.bhat[o + i];
    }
  }
}

cudaError_t launch_project(nrto_handle_s* h, cudaStream_t st) {
  const int64_t n = (int64_t)h->dev.d.B * h->dev.d.ng;
  if (n > 0) {
    k_project<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(h->dev);
    h->launches++;
  }
  return cudaGetLastError();
}

// G0_k = sum_{state c, K_c > k} b_{c,k} b_{c,k}^T, H0_k = sum b_{c,k} b_hat_{c,k}^T (= Zb_k,
// control rows have b_hat = 0), one warp per (instance, k), from the tile layout: the
// 8 cones of a tile at block k are one contiguous slab; DMMA over the cone index.
template <int NTI>
__global__ void __launch_bounds__(256) k_gram_tiles(Dev v) {
  const Dims d = v.d;
  const int nx = d.nx, nu = d.nu, nup = d.nup, T = d.T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int64_t gw = (int64_t)blockIdx.x * 8 + warp;
  if (gw >= (int64_t)d.B * T) return;
  const int b = (int)(gw / T), k = (int)(gw % T);
  const double* bht = v.bhat_t + (int64_t)b * v.Est;
  const double* bdt = v.Bd_t + (int64_t)b * v.EBst;
  double gz[2] = {0.0, 0.0}, hz[NTI][2];
#pragma unroll
  for (int nt = 0; nt < NTI; ++nt) hz[nt][0] = hz[nt][1] = 0.0;
  for (int t = v.ktile0[k]; t < v.nstate_tiles; ++t) {
    const int nc = v.tiles[(int64_t)t * kTI + 2];
    const double* sb = bdt + v.ttb[2 * t + 1] + (int64_t)k * nc * nup;
    const double* sh = bht + v.ttb[2 * t] + (int64_t)k * nc * nx;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int c = q + 4 * ks;
      const bool cv = c < nc;
      const double bcg = (cv && g < nu) ? sb[c * nup + g] : 0.0;
      dmma(gz, bcg, bcg);
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) {
        const int i = g + 8 * nt;
        dmma(hz[nt], bcg, (cv && i < nx) ? sh[c * nx + i] : 0.0);
      }
    }
  }
  if (g < nu) {
    const int64_t bk = (int64_t)b * T + k;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int m2 = 2 * q + r;
      if (m2 < nu) v.G0[bk * nu * nu + g * nu + m2] = gz[r];
    }
#pragma unroll
    for (int nt = 0; nt < NTI; ++nt)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int i = 2 * q + r + 8 * nt;
        if (i < nx) {
          v.H0[bk * nu * nx + g * nx + i] = hz[nt][r];
          v.Zb[bk * nu * nx + g * nx + i] = hz[nt][r];
        }
      }
  }
}

cudaError_t launch_gram_tiles(nrto_handle_s* h, cudaStream_t st) {
  const Dev& v = h->dev;
  const int64_t nw = (int64_t)v.d.B * v.d.T;
  if (nw == 0) return cudaSuccess;
  if (v.d.nx <= 8) k_gram_tiles<1><<<(unsigned)((nw + 7) / 8), 256, 0, st>>>(v);
  else k_gram_tiles<2><<<(unsigned)((nw + 7) / 8), 256, 0, st>>>(v);
  h->launches++;
  return cudaGetLastError();
}

static int tma_stages(const Dims& d, bool ds = false) {
  const TmaGeom G = tma_geom(d.nx, d.nup, d.nu, ds);
  const size_t fixed = tma_fixed_doubles(d.T, d.nx, d.nu, ds);
  // leave room for one k_qp_sparse CTA beside the pass CTA (overlapped QP): its
  // recurrence vector, Acl ring, barriers and per-knot flags (qp.cu)
  const size_t qp = ((size_t)(d.T + 1) * d.nx + (size_t)QP_RING * d.nx * d.nx + QP_RING) * sizeof(double) +
                    (size_t)6 * (d.T + 1) * sizeof(int16_t);
  size_t capb = 225 * 1024;
  if (228 * 1024 > qp + 2048 + 3 * G.stage * sizeof(double) + fixed * sizeof(double))
    capb = std::min<size_t>(capb, 228 * 1024 - 2048 - qp);
  const size_t cap = capb / sizeof(double);
  if (fixed >= cap) return 0;
  return (int)std::min<size_t>(kMaxStages, (cap - fixed) / G.stage);
}

// streamed-D variant: when D of the whole horizon does not fit beside >= 3 stages
static bool tma_dstream(const Dims& d) { return tma_stages(d, false) < 3; }

size_t tma_smem_bytes(const Dims& d) {
  const bool ds = tma_dstream(d);
  const TmaGeom G = tma_geom(d.nx, d.nup, d.nu, ds);
  return (tma_fixed_doubles(d.T, d.nx, d.nu, ds) + (size_t)tma_stages(d, ds) * G.stage) * sizeof(double);
}

bool tma_supported(const Dims& d) {
  // n_x even (16-byte DMMA operand rows), n_x <= 16, n_u <= 8; horizons up to
  // 1023 (64 chunks of 16 blocks per tile); D_k resident in shared memory when it
  // fits beside >= 3 stages, otherwise streamed per chunk through the stages
  if (!((d.nx % 2 == 0) && d.nx <= 16 && d.nu <= 8 && d.T <= 1023)) return false;
  return tma_stages(d, false) >= 3 || tma_stages(d, true) >= 3;
}

template <int NTI, int NKS, int KK, int NXE = 0, int NUE = 0, int NW = 16, bool DS = false>
static cudaError_t launch_tma_t(nrto_handle_s* h, cudaStream_t st) {
  const size_t smem = tma_smem_bytes(h->dev.d);
  auto kfn = k_fa_tma<NTI, NKS, KK, NXE, NUE, NW, DS>;
  cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kfn<<<h->dev.nwitems, (NW + 1) * 32, smem, st>>>(h->dev, h->dev.tiles, h->dev.witems,
                                                   tma_stages(h->dev.d, DS), h->tma_margin);
  h->launches++;
  return cudaGetLastError();
}

template <int KK>
static cudaError_t launch_tma_k(nrto_handle_s* h, int nti, int nks, cudaStream_t st) {
  if (nti == 1 && nks == 1) return launch_tma_t<1, 1, KK>(h, st);
  if (nti == 1 && nks == 2) return launch_tma_t<1, 2, KK>(h, st);
  if (nti == 2 && nks == 1) return launch_tma_t<2, 1, KK>(h, st);
  return launch_tma_t<2, 2, KK>(h, st);
}

template <int KK>
static cudaError_t launch_tma_ds(nrto_handle_s* h, int nti, int nks, cudaStream_t st) {
  if (nti == 1 && nks == 1) return launch_tma_t<1, 1, KK, 0, 0, 16, true>(h, st);
  if (nti == 1 && nks == 2) return launch_tma_t<1, 2, KK, 0, 0, 16, true>(h, st);
  if (nti == 2 && nks == 1) return launch_tma_t<2, 1, KK, 0, 0, 16, true>(h, st);
  return launch_tma_t<2, 2, KK, 0, 0, 16, true>(h, st);
}

cudaError_t launch_fa_tma(nrto_handle_s* h, cudaStream_t st) {
  const Dims& d = h->dev.d;
  const int nti = (d.nx + 7) / 8, nks = (d.nu + 3) / 4;
  cudaError_t e = cudaSuccess;
  if (h->dev.nwitems > 0) {
    // KK = chunks of 16 blocks per tile: covers K <= 16 KK - 1
    if (tma_dstream(d)) {
      if (d.T < 208) e = launch_tma_ds<13>(h, nti, nks, st);
      else if (d.T < 416) e = launch_tma_ds<26>(h, nti, nks, st);
      else e = launch_tma_ds<64>(h, nti, nks, st);
    }
    else if (d.nx == 14 && d.nu == 7 && d.T >= 64 && d.T < 112) e = launch_tma_t<2, 2, 7, 14, 7, TMA_NW>(h, st);
    else if (d.nx == 12 && d.nu == 4 && d.T >= 32 && d.T < 64) e = launch_tma_t<2, 1, 4, 12, 4>(h, st);
    else if (d.T < 32) e = launch_tma_k<2>(h, nti, nks, st);
    else if (d.T < 64) e = launch_tma_k<4>(h, nti, nks, st);
    else if (d.T < 112) e = launch_tma_k<7>(h, nti, nks, st);
    else if (d.T < 208) e = launch_tma_k<13>(h, nti, nks, st);
    else e = launch_tma_k<26>(h, nti, nks, st);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_fa_ctrl(nrto_handle_s* h, cudaStream_t st) {
  const Dims& d = h->dev.d;
  if (h->dev.nctrl > 0) {
    // warps (steps) per CTA, NRTO_CTRL_WARPS (default 4): small CTAs fit beside the QP CTAs
    static const int cwp = [] { const char* e = getenv("NRTO_CTRL_WARPS"); return e ? atoi(e) : 4; }();
    dim3 grid(d.B, (d.T + cwp - 1) / cwp);
    k_fa_ctrl<<<grid, 32 * cwp, 0, st>>>(h->dev);
    h->launches++;
  }
  return cudaGetLastError();
}

}  // namespace nrto
