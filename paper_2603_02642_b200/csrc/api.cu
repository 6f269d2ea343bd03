// C ABI of libnrto (include/nrto.h): validation, layout, device allocation,
// host orchestration of the inner loop.  No C++ exception crosses the ABI.
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>
#include "common.cuh"

using namespace nrto;

static thread_local std::string g_err = "ok";

static nrto_err fail(nrto_err code, const std::string& msg) {
  g_err = msg;
  return code;
}
static nrto_err cuda_fail(cudaError_t e, const char* where) {
  return fail(NRTO_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CK(call)                                               \
  do {                                                         \
    cudaError_t e_ = (call);                                   \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);        \
  } while (0)

extern "C" const char* nrto_last_error(void) { return g_err.c_str(); }

extern "C" void nrto_default_params(nrto_params* p) {
  if (!p) return;
  p->rho = 10.0; p->rho_admm = 40.0; p->alpha_dr = 0.9; p->sigma_dr = 1e-6; p->r_s = 1.0;
  p->eps_p = 1e-3; p->eps_d = 1e-3; p->eps_dr = 1e-4;
  p->rho_qp = 1.0; p->sigma_qp = 1e-6; p->alpha_qp = 1.6;
  p->max_iter = 40; p->max_admm_iter = 40; p->max_dr_iter = 100; p->qp_iters = 10;
  p->check_every = 1; p->fixed_iters = 0;
}

static nrto_err check_shape(const nrto_shape* s) {
  if (!s) return fail(NRTO_EINVAL, "shape is NULL");
  if (s->n_x < 1 || s->n_x > 32) return fail(NRTO_EINVAL, "n_x must be in [1,32]");
  if (s->n_u < 1 || s->n_u > s->n_x) return fail(NRTO_EINVAL, "n_u must be in [1,n_x]");
  if (s->T < 1) return fail(NRTO_EINVAL, "T must be >= 1");
  if (s->n_g < 0) return fail(NRTO_EINVAL, "n_g must be >= 0");
  if (s->batch < 1) return fail(NRTO_EINVAL, "batch must be >= 1");
  if (s->n_g > 0 && (!s->cone_knot || !s->cone_kind))
    return fail(NRTO_EINVAL, "cone_knot / cone_kind are NULL");
  for (int j = 0; j < s->n_g; ++j) {
    const int k = s->cone_knot[j], kd = s->cone_kind[j];
    if (kd == 0 && (k < 1 || k > s->T))
      return fail(NRTO_EINVAL, "state cone " + std::to_string(j) + ": knot must be in 1..T");
    if (kd == 1 && (k < 0 || k > s->T - 1))
      return fail(NRTO_EINVAL, "control cone " + std::to_string(j) + ": knot must be in 0..T-1");
    if (kd != 0 && kd != 1) return fail(NRTO_EINVAL, "cone_kind must be 0 or 1");
  }
  return NRTO_OK;
}

extern "C" nrto_err nrto_layout(const nrto_shape* s, int64_t* E_out, int64_t* off) {
  nrto_err e = check_shape(s);
  if (e != NRTO_OK) return e;
  int64_t acc = 0;
  for (int j = 0; j < s->n_g; ++j) {
    if (off) off[j] = acc;
    acc += (s->cone_kind[j] == 0) ? (int64_t)(s->cone_knot[j] + 1) * s->n_x : s->n_x;
  }
  if (off) off[s->n_g] = acc;
  if (E_out) *E_out = acc;
  return NRTO_OK;
}

// process-wide workspace allocator (nrto_set_allocator)
static nrto_alloc_fn g_alloc_fn = nullptr;
static nrto_free_fn g_free_fn = nullptr;
static void* g_alloc_ctx = nullptr;

extern "C" nrto_err nrto_set_allocator(nrto_alloc_fn alloc, nrto_free_fn release, void* ctx) {
  if (alloc && !release) return fail(NRTO_EINVAL, "an allocator needs its release function");
  g_alloc_fn = alloc;
  g_free_fn = alloc ? release : nullptr;
  g_alloc_ctx = alloc ? ctx : nullptr;
  return NRTO_OK;
}

template <class T>
static nrto_err dalloc(nrto_handle_s* h, T** p, int64_t n) {
  if (h->nallocs >= (int)(sizeof(h->allocs) / sizeof(h->allocs[0])))
    return fail(NRTO_ENOMEM, "too many allocations");
  void* q = nullptr;
  const size_t bytes = (size_t)std::max<int64_t>(n, 1) * sizeof(T);
  if (h->alloc_fn) {
    q = h->alloc_fn(h->alloc_ctx, bytes, h->alloc_stream);
    if (!q) return fail(NRTO_ENOMEM, "allocator hook returned NULL for " + std::to_string(bytes) + " bytes");
  } else {
    cudaError_t e = cudaMalloc(&q, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(NRTO_ENOMEM, "cudaMalloc(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    }
  }
  h->allocs[h->nallocs++] = q;
  *p = (T*)q;
  return NRTO_OK;
}

static void free_all(nrto_handle_s* h) {
  for (int i = 0; i < h->nallocs; ++i) {
    if (h->free_fn) h->free_fn(h->alloc_ctx, h->allocs[i], h->alloc_stream);
    else cudaFree(h->allocs[i]);
  }
  h->nallocs = 0;
}

#define AL(ptr, n)                                 \
  do {                                             \
    nrto_err e_ = dalloc(h, &(ptr), (int64_t)(n)); \
    if (e_ != NRTO_OK) { free_all(h); delete h; return e_; } \
  } while (0)

extern "C" nrto_err nrto_setup(const nrto_shape* s, const nrto_data* data,
                               const nrto_params* prm, void* stream, nrto_handle* out) {
  if (!out) return fail(NRTO_EINVAL, "out handle pointer is NULL");
  *out = nullptr;
  nrto_err e = check_shape(s);
  if (e != NRTO_OK) return e;
  if (!data || !prm) return fail(NRTO_EINVAL, "data / params is NULL");
  if (!data->A || !data->B || !data->Psi || !data->tau || !data->W_K || !data->R_u ||
      !data->u_hat || !data->r_trust || (s->n_g > 0 && (!data->grad || !data->g0)))
    return fail(NRTO_EINVAL, "a required data pointer is NULL");
  if (prm->max_iter < 0 || prm->max_admm_iter < 0 || prm->max_dr_iter < 0 || prm->qp_iters < 0 ||
      prm->check_every < 1)
    return fail(NRTO_EINVAL, "iteration counts must be >= 0 and check_every >= 1");
  if (!(prm->rho > 0) || !(prm->rho_admm > 0) || !(prm->rho_qp > 0) || !(prm->r_s > 0) ||
      !(prm->sigma_dr >= 0) || !(prm->sigma_qp >= 0) || !(prm->alpha_dr > 0 && prm->alpha_dr < 2) ||
      !(prm->alpha_qp > 0 && prm->alpha_qp < 2))
    return fail(NRTO_EINVAL, "penalty / relaxation parameters out of range");
  cudaStream_t st = (cudaStream_t)stream;

  auto* h = new nrto_handle_s();
  h->stream = st;
  h->alloc_fn = g_alloc_fn; h->free_fn = g_free_fn; h->alloc_ctx = g_alloc_ctx; h->alloc_stream = stream;
  Dev& v = h->dev;
  Dims& d = v.d;
  d.nx = s->n_x; d.nu = s->n_u; d.T = s->T; d.ng = s->n_g; d.B = s->batch;
  d.NK = d.T * d.nu * d.nx;
  v.prm = *prm;
  // ---- host-side layout and CSR lists
  const int ng = d.ng, T = d.T, nx = d.nx, nu = d.nu;
  std::vector<int64_t> off(ng + 1), offB(ng + 1);
  int64_t eb = 0;
  nrto_layout(s, &d.E, off.data());
  d.nup = nu + (nu & 1);
  for (int j = 0; j < ng; ++j) {
    offB[j] = eb;
    eb += (s->cone_kind[j] == 0) ? (int64_t)s->cone_knot[j] * d.nup : d.nup;
  }
  offB[ng] = eb;
  d.EB = eb;
  std::vector<int32_t> kptr(T + 1, 0), kcone, sptr(T + 2, 0), srow, cptr(T + 1, 0), crow;
  for (int k = 0; k < T; ++k) {
    kptr[k] = (int32_t)kcone.size();
    for (int j = 0; j < ng; ++j) {
      const bool st0 = s->cone_kind[j] == 0;
      if ((st0 && s->cone_knot[j] > k) || (!st0 && s->cone_knot[j] == k)) kcone.push_back(j);
    }
  }
  kptr[T] = (int32_t)kcone.size();
  for (int k = 0; k <= T; ++k) {
    sptr[k] = (int32_t)srow.size();
    for (int j = 0; j < ng; ++j)
      if (s->cone_kind[j] == 0 && s->cone_knot[j] == k) srow.push_back(j);
  }
  sptr[T + 1] = (int32_t)srow.size();
  for (int k = 0; k < T; ++k) {
    cptr[k] = (int32_t)crow.size();
    for (int j = 0; j < ng; ++j)
      if (s->cone_kind[j] == 1 && s->cone_knot[j] == k) crow.push_back(j);
  }
  cptr[T] = (int32_t)crow.size();
  std::vector<int32_t> qrow;   // QP row order (qp.cu, pipelined rows phase)
  for (int p = 1; p <= T; ++p) {
    for (int q = sptr[p]; q < sptr[p + 1]; ++q) qrow.push_back(srow[q]);
    for (int q = cptr[p - 1]; q < cptr[p]; ++q) qrow.push_back(crow[q]);
  }
  std::vector<int32_t> knot(s->cone_knot, s->cone_knot + ng), kind(ng);
  for (int j = 0; j < ng; ++j) kind[j] = s->cone_kind[j];
  // ---- tiles of <= 8 cones with equal (kind, knot) for the fused pass, and
  //      work items = contiguous tile ranges of one instance balanced by elements
  std::vector<int32_t> tiles;
  std::vector<int64_t> tile_work;
  auto add_group = [&](int kd, int kn) {
    std::vector<int32_t> cs;
    for (int j = 0; j < ng; ++j)
      if (s->cone_kind[j] == kd && s->cone_knot[j] == kn) cs.push_back(j);
    for (size_t a = 0; a < cs.size(); a += 8) {
      const int nc = (int)std::min<size_t>(8, cs.size() - a);
      tiles.push_back(kd); tiles.push_back(kn); tiles.push_back(nc);
      tiles.push_back(kd == 0 ? 0 : kn);
      for (int c = 0; c < 8; ++c) tiles.push_back(c < nc ? cs[a + c] : 0);
      tile_work.push_back((int64_t)nc * ((kd == 0 ? kn + 1 : 1) * nx + (kd == 0 ? kn : 1) * nu));
    }
  };
  for (int kn = 1; kn <= T; ++kn) add_group(0, kn);
  const int nstate_tiles = (int)tile_work.size();
  for (int kn = 0; kn < T; ++kn) add_group(1, kn);
  int nctrl = 0;
  for (int j = 0; j < ng; ++j) nctrl += (s->cone_kind[j] == 1);
  // path: TMA-pipelined state pass + exact control kernel when the geometry allows
  const bool use_tma = tma_supported(d);
  const int ntiles = use_tma ? nstate_tiles : (int)tile_work.size();
  int nsm = 148;
  { int dev = 0; if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev); cudaGetLastError(); }
  int64_t work_tot = 0;
  for (int t = 0; t < ntiles; ++t) work_tot += tile_work[t];
  const int64_t zbytes = 16LL * T * nu * nx;
  // work items per instance: the tiled fused pass (fused == 1) writes one adjoint
  // partial per item, so its split is capped by the partials' size; the TMA pass
  // forms no adjoint (Gram form), only tiles cap it (single instances
  // then spread over the SMs)
  const int smax = use_tma ? std::max(1, ntiles)
                           : (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, work_tot / std::max<int64_t>(zbytes, 1)));
  int nsplit = (int)std::min<int64_t>(smax, std::max<int64_t>(1, (6LL * 2 * nsm + d.B - 1) / d.B));
  if (ntiles == 0) nsplit = 1;
  std::vector<int32_t> witems;
  for (int b = 0; b < d.B && ntiles > 0; ++b) {
    int t = 0;
    int64_t acc = 0;
    for (int sp = 0; sp < nsplit; ++sp) {
      const int64_t goal = work_tot * (sp + 1) / nsplit;
      const int t0 = t;
      while (t < ntiles && (acc + tile_work[t] <= goal || t == t0)) acc += tile_work[t++];
      if (sp == nsplit - 1) { while (t < ntiles) acc += tile_work[t++]; }
      witems.push_back(b); witems.push_back(t0); witems.push_back(t); witems.push_back(sp);
    }
  }
  v.fused = use_tma ? 2 : ((fused_supported(d) && ntiles > 0) ? 1 : 0);
  {   // NRTO_FUSED=0: generic warp-per-cone pass instead of the tiled fused pass (non-TMA shapes)
    // default: tiny batches (B n_g <= 1024 cones, e.g. one c1 instance) take the generic
    // kernels -- measured c1 FullADMM 104 -> 81 us per iteration
    static const int fenv = [] { const char* e = getenv("NRTO_FUSED"); return e ? atoi(e) : -1; }();
    if (v.fused == 1 && (fenv == 0 || (fenv < 0 && (int64_t)d.B * ng <= 1024))) v.fused = 0;
  }
  v.nsm = nsm;
  v.nctrl = nctrl;
  v.ntiles = ntiles; v.nsplit = nsplit; v.nwitems = (int)(witems.size() / 4);
  v.nstate_tiles = nstate_tiles;
  std::vector<int32_t> ttb;
  int64_t est = 0, ebst = 0;
  if (use_tma) {
    for (int t = 0; t < nstate_tiles; ++t) {
      const int kn = tiles[t * 12 + 1], nc = tiles[t * 12 + 2];
      ttb.push_back((int32_t)est); ttb.push_back((int32_t)ebst);
      est += (int64_t)(kn + 1) * nc * nx;
      ebst += (int64_t)kn * nc * d.nup;
    }
  }
  v.Est = est; v.EBst = ebst;
  std::vector<int32_t> ktile0(T + 1, nstate_tiles);
  if (use_tma)
    for (int k = T; k >= 0; --k)
      for (int t = 0; t < nstate_tiles; ++t)
        if (tiles[t * 12 + 1] > k) { ktile0[k] = t; break; }

  const int64_t B = d.B;
  int32_t *dknot, *dkind, *dkptr, *dkcone, *dsptr, *dsrow, *dcptr, *dcrow;
  int64_t *doff, *doffB;
  AL(dknot, ng); AL(dkind, ng); AL(doff, ng + 1); AL(doffB, ng + 1);
  AL(dkptr, T + 1); AL(dkcone, kcone.size()); AL(dsptr, T + 2); AL(dsrow, srow.size());
  AL(dcptr, T + 1); AL(dcrow, crow.size());
  int32_t* dqrow;
  AL(dqrow, ng);
  v.qrow = dqrow;
  v.knot = dknot; v.kind = dkind; v.off = doff; v.offB = doffB; v.kptr = dkptr; v.kcone = dkcone;
  v.sptr = dsptr; v.srow = dsrow; v.cptr = dcptr; v.crow = dcrow;
  double *A, *Bm, *grad, *g0, *Psi, *tau, *W, *Ru, *uhat, *rtrust;
  AL(A, B * T * nx * nx); AL(Bm, B * T * nx * nu); AL(grad, B * ng * nx); AL(g0, B * ng);
  AL(Psi, B * (T + 1) * nx * nx); AL(tau, B); AL(W, B * T * nu * nu); AL(Ru, B * T * nu * nu);
  AL(uhat, B * T * nu); AL(rtrust, B);
  v.A = A; v.Bm = Bm; v.grad = grad; v.g0 = g0; v.Psi = Psi; v.tau = tau; v.W = W; v.Ru = Ru;
  v.uhat = uhat; v.rtrust = rtrust;
  AL(v.bhat, B * d.E); AL(v.Bd, B * d.EB); AL(v.Zb, B * T * nu * nx); AL(v.Lam, B * T * nu * nu);
  AL(v.U, B * T * nx * nx); AL(v.Ulam, B * T * nx); AL(v.Urep, B * T); AL(v.psame, B * T);
  v.scanM = 0; v.scanC = 0;
  v.qpgrid = 0; v.qg_s = nullptr; v.qg_a = nullptr; v.qg_part = nullptr; v.qg_bar = nullptr;
  v.cone_lo = 0; v.cone_hi = ng;
  if (B <= kScanMaxBatch && T >= 2 && nx <= 32 && nu <= 32) {
    // one large instance (many rows or a horizon whose QP vectors exceed one CTA's
    // shared memory): the grid-wide QP with its own chunking; else the one-CTA scan QP
    if (qp_grid_plan(d, nsm, v.scanM, v.scanC)) v.qpgrid = 1;
    else scan_plan(T, v.scanM, v.scanC);
  }
  for (EngineFactors* F : {&v.fa, &v.dr}) {
    AL(F->V, B * T * nu * nu); AL(F->den, B * T * nu * nx); AL(F->Kf, B * T * nu * nx);
    AL(F->Acl, B * T * nx * nx); AL(F->AclT, B * T * nx * nx); AL(F->Hinv, B * T * nu * nu); AL(F->HB, B * T * nu * nx);
    F->PhiB = nullptr; F->PhiF = nullptr;
    if (v.scanC > 0) { AL(F->PhiB, B * T * nx * nx); AL(F->PhiF, B * T * nx * nx); }
  }
  AL(v.Y, B * d.E); AL(v.s, B * ng); AL(v.tin, B * ng); AL(v.pt, B * ng); AL(v.ptprev, B * ng);
  AL(v.p, B * ng); AL(v.lamp, B * ng); AL(v.K, B * d.NK); AL(v.Ccur, B * T * nx * nu);
  AL(v.Cprev, B * T * nx * nu); AL(v.D, B * T * nx * nu); AL(v.Z, B * T * nu * nx); AL(v.Zg, B * T * nu * nx);
  AL(v.du, B * T * nu); AL(v.zl, B * ng); AL(v.yl, B * ng); AL(v.zb, B * (T + 1) * nx);
  AL(v.yb, B * (T + 1) * nx); AL(v.rp, B * ng); AL(v.wq, B * ng); AL(v.rx, B * (T + 1) * nx);
  AL(v.ru, B * T * nu); AL(v.kff, B * T * nu); AL(v.dxt, B * (T + 1) * nx); AL(v.dut, B * T * nu);
  AL(v.Kt, B * d.NK); AL(v.pit, B * ng); AL(v.tt, B * ng); AL(v.rdr_part, B * ng); AL(v.rdr, B);
  AL(v.dr_active, B); AL(v.status, B); AL(v.iters, B); AL(v.active, B); AL(v.r_p, B); AL(v.r_d, B);
  int32_t *dtiles, *dwitems;
  AL(dtiles, tiles.size()); AL(dwitems, witems.size());
  v.tiles = dtiles; v.witems = dwitems;
  AL(v.Zpart, (v.fused == 1 ? B * nsplit : 1) * T * nu * nx); AL(v.Zc, B * T * nu * nx);
  if (v.fused == 2) {
    AL(v.ttb, ttb.size()); AL(v.bhat_t, B * est); AL(v.Bd_t, B * ebst); AL(v.ktile0, T + 1);
    AL(v.G, B * T * nu * nu); AL(v.G0, B * T * nu * nu); AL(v.dG, B * T * nu * nu);
    AL(v.H, B * T * nu * nx); AL(v.H0, B * T * nu * nx); AL(v.dH, B * T * nu * nx);
  }
  AL(v.Zctrl, B * T * nu * nx); AL(v.nrm2, B * ng);
  AL(v.rowpk, B * ng); AL(v.gval, B * ng * 8); AL(v.cu2, B * T * nu);
  AL(v.pass_bytes, 1);
  cudaMemset(v.pass_bytes, 0, sizeof(unsigned long long));
  v.ylazy = 0;
  AL(v.clist, B * ng); AL(v.cw, B * ng); AL(v.ncorr, B);
  if (v.qpgrid) {
    AL(v.qg_s, B * (T + 1) * nx); AL(v.qg_a, B * T * nx); AL(v.qg_part, 2 * 1024); AL(v.qg_bar, 1);
  }
  // persistent DR loop (persist.cu): cone chunks of one instance
  std::vector<int32_t> drch, drkr;
  int drEc = 0, drEBc = 0;
  dr_loop_plan(d, s->cone_knot, s->cone_kind, nsm, drch, drkr, drEc, drEBc);
  v.drQ = drch.empty() ? 0 : (int)drch.size() - 1;
  v.drchunk = nullptr; v.drkr = nullptr; v.drZpart = nullptr; v.drrq = nullptr; v.drbar = nullptr;
  v.drEc = drEc; v.drEBc = drEBc;
  if (v.drQ > 0) {
    int32_t *dch, *dkr;
    AL(dch, drch.size()); AL(dkr, drkr.size());
    v.drchunk = dch; v.drkr = dkr;
    AL(v.drZpart, B * v.drQ * T * nu * nx); AL(v.drrq, B * v.drQ); AL(v.drbar, 1);
  }

  // shape arrays (pageable host vectors: synchronous copies)
  cudaError_t ce = cudaSuccess;
  auto hup = [&](void* dst, const void* src, size_t bytes) {
    if (ce == cudaSuccess && bytes) ce = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
  };
  hup(dknot, knot.data(), ng * 4); hup(dkind, kind.data(), ng * 4);
  hup(doff, off.data(), (ng + 1) * 8); hup(doffB, offB.data(), (ng + 1) * 8);
  hup(dkptr, kptr.data(), (T + 1) * 4); hup(dkcone, kcone.data(), kcone.size() * 4);
  hup(dsptr, sptr.data(), (T + 2) * 4); hup(dsrow, srow.data(), srow.size() * 4);
  hup(dcptr, cptr.data(), (T + 1) * 4); hup(dcrow, crow.data(), crow.size() * 4);
  hup(dqrow, qrow.data(), qrow.size() * 4);
  hup(dtiles, tiles.data(), tiles.size() * 4); hup(dwitems, witems.data(), witems.size() * 4);
  if (v.qpgrid && ce == cudaSuccess) {
    h->qp_grid = qp_grid_size(h);
    if (h->qp_grid == 0) { v.qpgrid = 0; v.scanM = 0; v.scanC = 0; }   // not co-resident: older QP kernels
  }
  if (v.drQ > 0) {
    hup((void*)v.drchunk, drch.data(), drch.size() * 4);
    hup((void*)v.drkr, drkr.data(), drkr.size() * 4);
    if (ce == cudaSuccess) ce = cudaMemset(v.drbar, 0, sizeof(unsigned long long));
    if (ce == cudaSuccess) h->dr_loop_grid = dr_loop_grid(v);
  }
  if (v.fused == 2) {
    hup(v.ttb, ttb.data(), ttb.size() * 4);
    hup(v.ktile0, ktile0.data(), (T + 1) * 4);
  }
  if (ce != cudaSuccess) { free_all(h); delete h; return cuda_fail(ce, "nrto_setup shape upload"); }
  nrto_err re = nrto_refresh(h, data, stream);
  if (re != NRTO_OK) { free_all(h); delete h; return re; }
  h->dr_fresh = 1;
  *out = h;
  return NRTO_OK;
}


extern "C" nrto_err nrto_refresh(nrto_handle h, const nrto_data* data, void* stream) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (!data) return fail(NRTO_EINVAL, "data is NULL");
  if (h->general && !h->gen_refresh_ok)
    return fail(NRTO_EINVAL, "nrto_refresh of a general-set handle: call nrto_setup_general again");
  if (h->sharded) return fail(NRTO_EINVAL, "nrto_refresh of a cone-sharded handle: set it up again");
  Dev& v = h->dev;
  const Dims& d = v.d;
  const int ng = d.ng, T = d.T, nx = d.nx, nu = d.nu;
  const int64_t B = d.B;
  if (!data->A || !data->B || !data->Psi || !data->tau || !data->W_K || !data->R_u ||
      !data->u_hat || !data->r_trust || (ng > 0 && (!data->grad || !data->g0)))
    return fail(NRTO_EINVAL, "a required data pointer is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  const bool hostin = data->memory == NRTO_MEM_HOST;
  const size_t D8 = sizeof(double);
  cudaError_t ce = cudaSuccess;
  auto up = [&](const double* dst, const double* src, int64_t n) {
    if (ce == cudaSuccess && n > 0)
      ce = cudaMemcpyAsync((void*)dst, src, (size_t)n * D8,
                           hostin ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st);
  };
  up(v.A, data->A, B * T * nx * nx); up(v.Bm, data->B, B * T * nx * nu);
  up(v.grad, data->grad, B * ng * nx); up(v.g0, data->g0, B * ng);
  up(v.Psi, data->Psi, B * (T + 1) * nx * nx); up(v.tau, data->tau, B);
  up(v.W, data->W_K, B * T * nu * nu); up(v.Ru, data->R_u, B * T * nu * nu);
  up(v.uhat, data->u_hat, B * T * nu); up(v.rtrust, data->r_trust, B);
  if (ce != cudaSuccess) return cuda_fail(ce, "nrto_refresh upload");
  ce = launch_setup(h, st);
  if (ce != cudaSuccess) return cuda_fail(ce, "nrto_refresh kernels");
  const int se = read_setup_error(st);   // synchronises the stream
  ce = cudaGetLastError();
  if (ce != cudaSuccess) return cuda_fail(ce, "nrto_refresh sync");
  if (se) return fail(NRTO_ENOTSPD, se == 1 ? "W_K (+ sigma_dr/2) is not SPD" : "Riccati H_uu is not SPD");
  h->dr_fresh = 1;
  return NRTO_OK;
}

static cudaEvent_t prof_event(nrto_handle_s* h) {
  cudaEvent_t e = nullptr;
  if (!h->pool.empty()) { e = h->pool.back(); h->pool.pop_back(); return e; }
  cudaEventCreate(&e);
  return e;
}

static cudaError_t copy_out(void* dst, const void* src, size_t bytes, bool host, cudaStream_t st) {
  if (!dst || bytes == 0) return cudaSuccess;
  return cudaMemcpyAsync(dst, src, bytes, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                         st);
}

static int poll_active(nrto_handle_s* h, int32_t* dcount, int dr, cudaStream_t st, cudaError_t* ce) {
  int32_t c = 0;
  *ce = launch_count_active(h, dcount, dr, st);
  if (*ce == cudaSuccess) *ce = cudaMemcpyAsync(&c, dcount, 4, cudaMemcpyDeviceToHost, st);
  if (*ce == cudaSuccess) *ce = cudaStreamSynchronize(st);
  return c;
}


// finish kernels (nu, lam_nu, margins, objective) and the copies of every output
static nrto_err write_outputs(nrto_handle_s* h, int engine, const nrto_out* o, cudaStream_t st,
                              double* nu_d, double* lam_d, double* obj_d, double* mc_d, double* ml_d) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  const bool host = o->memory == NRTO_MEM_HOST;
  const int64_t B = d.B;
  const size_t D8 = sizeof(double);
  nrto_out od = *o;
  od.nu = nu_d; od.lam_nu = lam_d; od.objective = obj_d; od.margin_cone = mc_d; od.margin_lin = ml_d;
  CK(launch_finish(h, engine, &od, st));
  CK(copy_out(o->kv, v.K, B * d.NK * D8, host, st));
  CK(copy_out(o->du, v.du, B * d.T * d.nu * D8, host, st));
  CK(copy_out(o->p, v.p, B * d.ng * D8, host, st));
  CK(copy_out(o->p_tilde, v.pt, B * d.ng * D8, host, st));
  CK(copy_out(o->lam_p, v.lamp, B * d.ng * D8, host, st));
  CK(copy_out(o->iters, v.iters, B * 4, host, st));
  CK(copy_out(o->status, v.status, B * 4, host, st));
  CK(copy_out(o->r_p, v.r_p, B * D8, host, st));
  CK(copy_out(o->r_d, v.r_d, B * D8, host, st));
  if (v.hist) CK(copy_out(o->hist, v.hist, (size_t)B * v.hist_L * 3 * D8, host, st));
  v.hist = nullptr;
  if (host) {
    CK(copy_out(o->nu, nu_d, B * d.E * D8, true, st));
    CK(copy_out(o->lam_nu, lam_d, B * d.E * D8, true, st));
    CK(copy_out(o->objective, obj_d, B * D8, true, st));
    CK(copy_out(o->margin_cone, mc_d, B * d.ng * D8, true, st));
    CK(copy_out(o->margin_lin, ml_d, B * d.ng * D8, true, st));
  }
  if (host) CK(cudaStreamSynchronize(st));
  return NRTO_OK;
}

// handle-owned staging of the kernel-written optional outputs in host mode
static nrto_err out_staging(nrto_handle_s* h, const nrto_out* o, double** nu_d, double** lam_d,
                            double** obj_d, double** mc_d, double** ml_d) {
  const Dims& d = h->dev.d;
  const int64_t B = d.B;
  const size_t D8 = sizeof(double);
  *nu_d = o->nu; *lam_d = o->lam_nu; *obj_d = o->objective; *mc_d = o->margin_cone; *ml_d = o->margin_lin;
  if (!h->dcount) {
    CK(cudaMalloc((void**)&h->dcount, 4));
    CK(cudaMalloc((void**)&h->stage_ng2, (size_t)std::max<int64_t>(2 * B * d.ng, 1) * D8));
    CK(cudaMalloc((void**)&h->stage_b, (size_t)B * D8));
  }
  if (o->memory == NRTO_MEM_HOST) {
    if ((o->nu || o->lam_nu) && !h->stage_e2)
      CK(cudaMalloc((void**)&h->stage_e2, (size_t)std::max<int64_t>(2 * B * d.E, 1) * D8));
    if (o->nu) *nu_d = h->stage_e2;
    if (o->lam_nu) *lam_d = h->stage_e2 + B * d.E;
    if (o->objective) *obj_d = h->stage_b;
    if (o->margin_cone) *mc_d = h->stage_ng2;
    if (o->margin_lin) *ml_d = h->stage_ng2 + B * d.ng;
  }
  return NRTO_OK;
}

constexpr int kQpSparseRows = 512;   // rows from which the sparse-row QP is used for any batch

extern "C" nrto_err nrto_inner_solve(nrto_handle h, int32_t engine, const nrto_out* o,
                                     void* stream) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (!o) return fail(NRTO_EINVAL, "out is NULL");
  if (engine != NRTO_FULLADMM && engine != NRTO_DR) return fail(NRTO_EINVAL, "unknown engine");
  if (h->sharded) return fail(NRTO_EINVAL, "cone-sharded handle: drive it with nrto_solve_begin / nrto_dr_step / nrto_solve_end");
  cudaStream_t st = (cudaStream_t)stream;
  Dev& v = h->dev;
  const Dims& d = v.d;
  const nrto_params& prm = v.prm;
  const int64_t B = d.B;
  double *nu_d, *lam_d, *obj_d, *mc_d, *ml_d;
  {
    const nrto_err se = out_staging(h, o, &nu_d, &lam_d, &obj_d, &mc_d, &ml_d);
    if (se != NRTO_OK) return se;
  }
  int32_t* dcount = h->dcount;
  // optional residual trace: handle-owned device buffer, zeroed per solve
  const int histL = engine == NRTO_FULLADMM ? prm.max_iter : prm.max_admm_iter;
  v.hist = nullptr;
  v.hist_L = histL;
  if (o->hist && histL > 0) {
    const size_t need = (size_t)B * histL * 3;
    if (h->hist_cap < need) {
      if (h->hist_buf) cudaFree(h->hist_buf);
      h->hist_buf = nullptr; h->hist_cap = 0;
      CK(cudaMalloc((void**)&h->hist_buf, need * sizeof(double)));
      h->hist_cap = need;
    }
    CK(cudaMemsetAsync(h->hist_buf, 0, need * sizeof(double), st));
    v.hist = h->hist_buf;
  }

  // optional projection-case statistics (FullADMM): handle-owned counters, zeroed per solve
  v.case_cnt = nullptr;
  if (h->case_stats && engine == NRTO_FULLADMM && prm.max_iter > 0) {
    const int64_t need = 3LL * prm.max_iter;
    if (h->case_cap < need) {
      if (h->case_buf) cudaFree(h->case_buf);
      h->case_buf = nullptr; h->case_cap = 0;
      CK(cudaMalloc((void**)&h->case_buf, need * sizeof(unsigned long long)));
      h->case_cap = need;
    }
    CK(cudaMemsetAsync(h->case_buf, 0, need * sizeof(unsigned long long), st));
    v.case_cnt = h->case_buf;
    h->case_L = prm.max_iter;
  }

  cudaError_t ce = cudaSuccess;
  auto timed = [&](int cls, auto&& fn) -> cudaError_t {
    cudaEvent_t a = nullptr, b = nullptr;
    if (h->prof) { a = prof_event(h); b = prof_event(h); cudaEventRecord(a, st); }
    cudaError_t e = fn(h, st);
    if (h->prof) { cudaEventRecord(b, st); h->recs.push_back({cls, a, b}); }
    return e;
  };
  auto timed_qp = [&](int eng, int l) -> cudaError_t {
    cudaEvent_t a = nullptr, b = nullptr;
    if (h->prof) { a = prof_event(h); b = prof_event(h); cudaEventRecord(a, st); }
    cudaError_t e = (d.ng >= kQpSparseRows) ? launch_qp_sparse(h, eng, l, st) : launch_qp(h, eng, l, st);
    if (h->prof) { cudaEventRecord(b, st); h->recs.push_back({NRTO_K_QP, a, b}); }
    return e;
  };
  if (h->general) {                     // general (Gamma, S) set, FullADMM in order
    if (engine != NRTO_FULLADMM) return fail(NRTO_EINVAL, "general-set handles support NRTO_FULLADMM only");
    CK(launch_fa_reset(h, st));
    CK(gen_reset(h, st));
    for (int l = 1; l <= prm.max_iter; ++l) {
      CK(gen_iteration(h, l, st));
      if (!prm.fixed_iters && l % prm.check_every == 0 && l < prm.max_iter) {
        const int c = poll_active(h, dcount, 0, st, &ce);
        if (ce != cudaSuccess) return cuda_fail(ce, "poll");
        if (c == 0) break;
      }
    }
    v.case_cnt = nullptr;
    CK(gen_finish(h, mc_d, st));
    CK(launch_finish_inst(h, ml_d, obj_d, st));
    const bool host = o->memory == NRTO_MEM_HOST;
    const size_t D8 = sizeof(double);
    const int64_t nzr = B * d.ng * h->gen.nz;
    CK(copy_out(o->kv, v.K, B * d.NK * D8, host, st));
    CK(copy_out(o->du, v.du, B * d.T * d.nu * D8, host, st));
    CK(copy_out(o->p, v.p, B * d.ng * D8, host, st));
    CK(copy_out(o->p_tilde, v.pt, B * d.ng * D8, host, st));
    CK(copy_out(o->lam_p, v.lamp, B * d.ng * D8, host, st));
    CK(copy_out(o->iters, v.iters, B * 4, host, st));
    CK(copy_out(o->status, v.status, B * 4, host, st));
    CK(copy_out(o->r_p, v.r_p, B * D8, host, st));
    CK(copy_out(o->r_d, v.r_d, B * D8, host, st));
    CK(copy_out(o->nu, h->gen.nu, nzr * D8, host, st));
    CK(copy_out(o->lam_nu, h->gen.lam, nzr * D8, host, st));
    if (v.hist) CK(copy_out(o->hist, v.hist, (size_t)B * v.hist_L * 3 * D8, host, st));
    v.hist = nullptr;
    if (host) {
      CK(copy_out(o->objective, obj_d, B * D8, true, st));
      CK(copy_out(o->margin_cone, mc_d, B * d.ng * D8, true, st));
      CK(copy_out(o->margin_lin, ml_d, B * d.ng * D8, true, st));
      CK(cudaStreamSynchronize(st));
    }
    return NRTO_OK;
  }
  if (engine == NRTO_FULLADMM) {
    CK(launch_fa_reset(h, st));
    // QP(l) only gates project(l+1): in fixed-iteration mode it runs on the aux
    // stream concurrently with gain(l) and pass(l+1).
    // overlap needs enough instances to keep the SMs busy with the pass while the
    // QP runs; for small batches the QP is on the critical path and the wide
    // staged variant (Acl in shared memory, 1024 threads) is used in order.
    const int nsm = v.nsm;
#ifndef QP_OVERLAP_CTAS_PER_SM
#define QP_OVERLAP_CTAS_PER_SM 2
#endif
#ifdef NRTO_NOOVERLAP
    const bool overlap = false;
#else
    const bool overlap = v.fused >= 1 && prm.fixed_iters && d.B >= nsm;
#endif
    // the sparse-row QP (k_qp_sparse, one 256-thread CTA per instance) also for small
    // batches with many rows: its row phase scatters into the knot accumulators
    // instead of gathering per knot (c3: 1.72 -> 1.32 ms per iteration); the staged
    // 1024-thread kernel stays for tiny instances (c1: 207 vs 240 us)
    const bool wide = v.fused >= 1 && (d.B >= nsm || d.ng >= kQpSparseRows);
    if (overlap && !h->aux) {
      // the cone-pass chain gets the highest stream priority so that SM slots freed
      // by finishing pass CTAs go to pass CTAs; QP CTAs fill the leftover room
      int lo = 0, hp = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hp));
      CK(cudaStreamCreateWithPriority(&h->aux, cudaStreamNonBlocking, lo));
      CK(cudaStreamCreateWithPriority(&h->hi, cudaStreamNonBlocking, hp));
      CK(cudaEventCreateWithFlags(&h->ev_proj, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_qp, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming));
      CK(cudaStreamCreateWithPriority(&h->hi2, cudaStreamNonBlocking, hp));
      CK(cudaEventCreateWithFlags(&h->ev_g, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_c, cudaEventDisableTiming));
    }
    cudaStream_t st2 = h->aux;
    const cudaStream_t user_st = st;
    if (overlap) {                 // run the loop on the internal streams, joined to `st`
      CK(cudaEventRecord(h->ev_in, user_st));
      CK(cudaStreamWaitEvent(h->hi, h->ev_in, 0));
      st = h->hi;
    }
    auto timed2 = [&](cudaStream_t s2, int cls, auto&& fn) -> cudaError_t {
      cudaEvent_t a = nullptr, b = nullptr;
      if (h->prof) { a = prof_event(h); b = prof_event(h); cudaEventRecord(a, s2); }
      cudaError_t e = fn(s2);
      if (h->prof) { cudaEventRecord(b, s2); h->recs.push_back({cls, a, b}); }
      return e;
    };
    // in-order (small batch) fixed-iteration solves: the loop is device-only, so it is
    // captured once into a CUDA graph (keyed by the device-state descriptor before
    // the loop) and replayed -- the per-iteration kernels are short, launch gaps matter
    static const int use_graph_fa = [] { const char* e = getenv("NRTO_GRAPH"); return e ? atoi(e) : 1; }();
    if (!overlap && fa_small_ok(h)) {
      // small instances: the whole loop (all outer iterations, per-instance termination)
      // in one launch, one CTA per instance (qp.cu k_fa_small)
      v.iter = 0;
      CK(timed(NRTO_K_QP, [&](nrto_handle_s* hh, cudaStream_t s2) { return launch_fa_small(hh, prm.max_iter, s2); }));
      v.iter = prm.max_iter;
    } else if (!overlap && prm.fixed_iters && !h->prof && use_graph_fa) {
      if (!h->gst) CK(cudaStreamCreateWithFlags(&h->gst, cudaStreamNonBlocking));
      if (!h->ev_in) CK(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
      if (!h->ev_out) CK(cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming));
      v.iter = 0; v.ylazy = 0;             // loop-set fields: normalised for the key
      if (!h->fa_exec || std::memcmp(&h->fa_key, &v, sizeof(Dev)) != 0) {
        if (h->fa_exec) { cudaGraphExecDestroy(h->fa_exec); h->fa_exec = nullptr; }
        Dev key;
        std::memcpy(&key, &v, sizeof(Dev));
        const int64_t l0 = h->launches;
        cudaStream_t gs = h->gst;
        CK(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
        cudaError_t e = cudaSuccess;
        for (int l = 1; l <= prm.max_iter && e == cudaSuccess; ++l) {
          v.iter = l;
          v.ylazy = (v.fused == 2 && l < prm.max_iter) ? 1 : 0;
          if (v.fused == 0) {
            e = launch_fa_pass(h, gs);
            if (e == cudaSuccess) e = launch_adjoint(h, v.Y, v.s, v.active, gs);
            if (e == cudaSuccess) e = launch_fa_gain(h, gs);
            if (e == cudaSuccess) e = launch_qp(h, NRTO_FULLADMM, l, gs);
          } else {
            e = v.fused == 2 ? launch_fa_tma(h, gs) : launch_fa_fused(h, gs);
            if (e == cudaSuccess && v.fused == 2) e = launch_fa_ctrl(h, gs);
            if (e == cudaSuccess) e = launch_project(h, gs);
            if (e == cudaSuccess)
              e = launch_zlist(h, v.Y, v.clist, v.cw, nullptr, v.ncorr, 0, v.active, v.Zc, gs, v.ylazy,
                               v.fused == 2 ? 1 : 0, v.dG, v.dH);
            if (e == cudaSuccess) e = launch_fa_gain(h, gs);
            if (e == cudaSuccess) e = wide ? launch_qp_sparse(h, NRTO_FULLADMM, l, gs) : launch_qp(h, NRTO_FULLADMM, l, gs);
          }
        }
        cudaGraph_t g = nullptr;
        const cudaError_t ee = cudaStreamEndCapture(gs, &g);
        if (e == cudaSuccess) e = ee;
        if (e == cudaSuccess) e = cudaGraphInstantiate(&h->fa_exec, g, 0);
        if (g) cudaGraphDestroy(g);
        v.ylazy = 0;
        if (e != cudaSuccess) { h->fa_exec = nullptr; return cuda_fail(e, "FullADMM loop graph capture"); }
        h->fa_graph_launches = h->launches - l0;
        h->launches = l0;
        std::memcpy(&h->fa_key, &key, sizeof(Dev));
      }
      v.iter = prm.max_iter;
      CK(cudaEventRecord(h->ev_in, st));
      CK(cudaStreamWaitEvent(h->gst, h->ev_in, 0));
      CK(cudaGraphLaunch(h->fa_exec, h->gst));
      CK(cudaEventRecord(h->ev_out, h->gst));
      CK(cudaStreamWaitEvent(st, h->ev_out, 0));
      h->launches += h->fa_graph_launches;
    } else
    for (int l = 1; l <= prm.max_iter; ++l) {
      v.iter = l;
      // lazy y storage needs a known last iteration (it stores every y^L)
      v.ylazy = (v.fused == 2 && prm.fixed_iters && l < prm.max_iter) ? 1 : 0;
      if (v.fused == 0) {
        CK(timed(NRTO_K_PASS, launch_fa_pass));
        CK(timed(NRTO_K_ADJOINT, [](nrto_handle_s* hh, cudaStream_t s2) {
          return launch_adjoint(hh, hh->dev.Y, hh->dev.s, hh->dev.active, s2); }));
        CK(timed(NRTO_K_GAIN, launch_fa_gain));
        CK(timed_qp(NRTO_FULLADMM, l));
      } else {
        // overlapped mode: the control-cone kernel (needs D from gain(l-1) only) runs on
        // a second high-priority stream beside the state-cone pass
        const bool ctrl_side = overlap && v.fused == 2;
        if (ctrl_side) {
          CK(cudaEventRecord(h->ev_g, st));
          CK(cudaStreamWaitEvent(h->hi2, h->ev_g, 0));
          CK(timed2(h->hi2, NRTO_K_CTRL, [&](cudaStream_t s2) { return launch_fa_ctrl(h, s2); }));
          CK(cudaEventRecord(h->ev_c, h->hi2));
        }
        CK(timed(NRTO_K_PASS, v.fused == 2 ? launch_fa_tma : launch_fa_fused));
        if (v.fused == 2 && !ctrl_side) CK(timed(NRTO_K_CTRL, launch_fa_ctrl));
        if (ctrl_side) CK(cudaStreamWaitEvent(st, h->ev_c, 0));
        if (overlap && l > 1) CK(cudaStreamWaitEvent(st, h->ev_qp, 0));
        CK(timed(NRTO_K_OTHER, launch_project));
        if (overlap) {
          CK(cudaEventRecord(h->ev_proj, st));
          CK(cudaStreamWaitEvent(st2, h->ev_proj, 0));
          CK(timed2(st2, NRTO_K_QP, [&](cudaStream_t s2) { return launch_qp_sparse(h, NRTO_FULLADMM, l, s2, QP_OVERLAP_CTAS_PER_SM * nsm); }));
          CK(cudaEventRecord(h->ev_qp, st2));
        }
        CK(timed(NRTO_K_ADJOINT, [](nrto_handle_s* hh, cudaStream_t s2) {
          Dev& w = hh->dev;
          return launch_zlist(hh, w.Y, w.clist, w.cw, nullptr, w.ncorr, 0, w.active, w.Zc, s2, w.ylazy,
                              w.fused == 2 ? 1 : 0, w.dG, w.dH); }));
        CK(timed(NRTO_K_GAIN, launch_fa_gain));
        if (!overlap) {
          if (wide) CK(timed2(st, NRTO_K_QP, [&](cudaStream_t s2) { return launch_qp_sparse(h, NRTO_FULLADMM, l, s2); }));
          else CK(timed_qp(NRTO_FULLADMM, l));
        }
      }
      if (!prm.fixed_iters && l % prm.check_every == 0 && l < prm.max_iter) {
        const int c = poll_active(h, dcount, 0, st, &ce);
        if (ce != cudaSuccess) return cuda_fail(ce, "poll");
        if (c == 0) break;
      }
    }
    v.ylazy = 0;
    if (overlap) {
      CK(cudaStreamWaitEvent(st, h->ev_qp, 0));
      CK(cudaEventRecord(h->ev_out, st));
      CK(cudaStreamWaitEvent(user_st, h->ev_out, 0));
      st = user_st;
    }
  } else {
    if (!h->dr_ready) {                  // DR factors on first use after setup/refresh
      CK(launch_engine_factors(h, NRTO_DR, st));
      const int se = read_setup_error(st);
      if (se) return fail(NRTO_ENOTSPD, se == 1 ? "W_K + sigma_dr/2 is not SPD" : "Riccati H_uu is not SPD");
      h->dr_ready = 1;
    }
    CK(launch_dr_reset(h, h->dr_fresh, st));
    h->dr_fresh = 0;
    // fixed iteration count, no profiling: the whole loop is device-only, so it is
    // captured once into a CUDA graph (per device-state descriptor) and replayed --
    // ~20 k small launches per c2 solve become one graph launch (NRTO_GRAPH=0: off)
    static const int use_graph = [] { const char* e = getenv("NRTO_GRAPH"); return e ? atoi(e) : 1; }();
    if (prm.fixed_iters && !h->prof && use_graph) {
      if (!h->gst) CK(cudaStreamCreateWithFlags(&h->gst, cudaStreamNonBlocking));
      if (!h->ev_in) CK(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
      if (!h->ev_out) CK(cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming));
      if (!h->dr_exec || std::memcmp(&h->dr_key, &v, sizeof(Dev)) != 0) {
        if (h->dr_exec) { cudaGraphExecDestroy(h->dr_exec); h->dr_exec = nullptr; }
        const int64_t l0 = h->launches;
        CK(cudaStreamBeginCapture(h->gst, cudaStreamCaptureModeThreadLocal));
        cudaError_t e = cudaSuccess;
        for (int l = 1; l <= prm.max_admm_iter && e == cudaSuccess; ++l) {
          e = launch_dr_arm(h, h->gst);
          if (e == cudaSuccess && dr_loop_supported(h)) e = launch_dr_loop(h, prm.max_dr_iter, h->gst);
          else
          for (int m = 1; m <= prm.max_dr_iter && e == cudaSuccess; ++m) {
            if (e == cudaSuccess) e = launch_dr_gain(h, h->gst);
            if (e == cudaSuccess) e = launch_dr_pass(h, h->gst);
            if (e == cudaSuccess) e = launch_dr_adjoint(h, h->gst);
            if (e == cudaSuccess) e = launch_dr_reduce(h, h->gst);
          }
          if (e == cudaSuccess)
            e = (d.ng >= kQpSparseRows) ? launch_qp_sparse(h, NRTO_DR, l, h->gst) : launch_qp(h, NRTO_DR, l, h->gst);
        }
        cudaGraph_t g = nullptr;
        const cudaError_t ee = cudaStreamEndCapture(h->gst, &g);
        if (e == cudaSuccess) e = ee;
        if (e == cudaSuccess) e = cudaGraphInstantiate(&h->dr_exec, g, 0);
        if (g) cudaGraphDestroy(g);
        if (e != cudaSuccess) { h->dr_exec = nullptr; return cuda_fail(e, "DR loop graph capture"); }
        h->dr_graph_launches = h->launches - l0;
        h->launches = l0;
        std::memcpy(&h->dr_key, &v, sizeof(Dev));
      }
      CK(cudaEventRecord(h->ev_in, st));
      CK(cudaStreamWaitEvent(h->gst, h->ev_in, 0));
      CK(cudaGraphLaunch(h->dr_exec, h->gst));
      CK(cudaEventRecord(h->ev_out, h->gst));
      CK(cudaStreamWaitEvent(st, h->ev_out, 0));
      h->launches += h->dr_graph_launches;
    } else
    for (int l = 1; l <= prm.max_admm_iter; ++l) {
      CK(launch_dr_arm(h, st));
      if (dr_loop_supported(h)) {
        // one cooperative launch runs the whole DR loop (and its own stop test)
        CK(timed(NRTO_K_PASS, [&](nrto_handle_s* hh, cudaStream_t s2) {
          return launch_dr_loop(hh, prm.max_dr_iter, s2); }));
      } else
      for (int m = 1; m <= prm.max_dr_iter; ++m) {
        CK(timed(NRTO_K_GAIN, launch_dr_gain));
        CK(timed(NRTO_K_PASS, launch_dr_pass));
        CK(timed(NRTO_K_ADJOINT, launch_dr_adjoint));
        CK(timed(NRTO_K_OTHER, launch_dr_reduce));
        if (!prm.fixed_iters && (m % 4) == 0 && m < prm.max_dr_iter) {
          const int c = poll_active(h, dcount, 1, st, &ce);
          if (ce != cudaSuccess) return cuda_fail(ce, "poll");
          if (c == 0) break;
        }
      }
      CK(timed_qp(NRTO_DR, l));
      if (!prm.fixed_iters && l % prm.check_every == 0 && l < prm.max_admm_iter) {
        const int c = poll_active(h, dcount, 0, st, &ce);
        if (ce != cudaSuccess) return cuda_fail(ce, "poll");
        if (c == 0) break;
      }
    }
  }
  v.case_cnt = nullptr;
  return write_outputs(h, engine, o, st, nu_d, lam_d, obj_d, mc_d, ml_d);
}

extern "C" nrto_err nrto_gain_update(nrto_handle h, const double* nu, const double* kv_prev,
                                     double* kv_next, void* stream) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (!nu || !kv_prev || !kv_next) return fail(NRTO_EINVAL, "NULL argument");
  if (h->general) return fail(NRTO_EINVAL, "nrto_gain_update is not available for a general-set handle");
  CK(launch_gain_update(h, nu, kv_prev, kv_next, (cudaStream_t)stream));
  return NRTO_OK;
}

extern "C" nrto_err nrto_soc_project(const double* t, const double* y, const int64_t* off,
                                     int64_t n, double* to, double* yo, void* stream) {
  if (n < 0) return fail(NRTO_EINVAL, "n_cones < 0");
  if (n > 0 && (!t || !y || !off || !to || !yo)) return fail(NRTO_EINVAL, "NULL argument");
  CK(launch_soc_project(t, y, off, n, to, yo, (cudaStream_t)stream));
  return NRTO_OK;
}

extern "C" int64_t nrto_launch_count(nrto_handle h) { return h ? h->launches : 0; }

extern "C" nrto_err nrto_destroy(nrto_handle h) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  cudaDeviceSynchronize();
  for (auto& r : h->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : h->pool) cudaEventDestroy(e);
  if (h->ev_proj) cudaEventDestroy(h->ev_proj);
  if (h->ev_qp) cudaEventDestroy(h->ev_qp);
  if (h->aux) cudaStreamDestroy(h->aux);
  if (h->hi) cudaStreamDestroy(h->hi);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_out) cudaEventDestroy(h->ev_out);
  if (h->dr_exec) cudaGraphExecDestroy(h->dr_exec);
  if (h->hi2) cudaStreamDestroy(h->hi2);
  if (h->ev_g) cudaEventDestroy(h->ev_g);
  if (h->ev_c) cudaEventDestroy(h->ev_c);
  if (h->fa_exec) cudaGraphExecDestroy(h->fa_exec);
  if (h->gst) cudaStreamDestroy(h->gst);
  if (h->dcount) cudaFree(h->dcount);
  if (h->hist_buf) cudaFree(h->hist_buf);
  if (h->stage_ng2) cudaFree(h->stage_ng2);
  if (h->stage_b) cudaFree(h->stage_b);
  if (h->stage_e2) cudaFree(h->stage_e2);
  if (h->case_buf) cudaFree(h->case_buf);
  gen_free(h);
  free_all(h);
  delete h;
  return NRTO_OK;
}

extern "C" nrto_err nrto_profile_enable(nrto_handle h, int32_t enable) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  h->prof = enable != 0;
  return NRTO_OK;
}

extern "C" nrto_err nrto_profile_read(nrto_handle h, int32_t cls, double* total_ms,
                                      int64_t* launches) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (cls < 0 || cls >= NRTO_K_COUNT) return fail(NRTO_EINVAL, "bad kernel class");
  double tot = 0.0;
  int64_t n = 0;
  std::vector<nrto_prof_rec> keep;
  for (auto& r : h->recs) {
    if (r.cls != cls) { keep.push_back(r); continue; }
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    tot += ms;
    ++n;
    h->pool.push_back(r.a);
    h->pool.push_back(r.b);
  }
  h->recs.swap(keep);
  if (total_ms) *total_ms = tot;
  if (launches) *launches = n;
  return NRTO_OK;
}

extern "C" nrto_err nrto_pass_bytes(nrto_handle h, int64_t* bytes) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (!bytes) return fail(NRTO_EINVAL, "bytes is NULL");
  unsigned long long v = 0;
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(&v, h->dev.pass_bytes, sizeof(v), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(h->dev.pass_bytes, 0, sizeof(v));
  if (e != cudaSuccess) return cuda_fail(e, "nrto_pass_bytes");
  *bytes = (int64_t)v;
  return NRTO_OK;
}

extern "C" nrto_err nrto_case_stats_enable(nrto_handle h, int32_t enable) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  h->case_stats = enable != 0;
  return NRTO_OK;
}

extern "C" nrto_err nrto_case_stats_read(nrto_handle h, int64_t* counts, int32_t L) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (!counts || L < 0) return fail(NRTO_EINVAL, "counts is NULL or L < 0");
  std::memset(counts, 0, sizeof(int64_t) * 3 * (size_t)L);
  const int n = std::min<int>(L, h->case_L);
  if (n <= 0 || !h->case_buf) return NRTO_OK;
  std::vector<unsigned long long> tmp((size_t)3 * n);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(tmp.data(), h->case_buf, tmp.size() * sizeof(unsigned long long),
                                       cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "nrto_case_stats_read");
  for (size_t i = 0; i < tmp.size(); ++i) counts[i] = (int64_t)tmp[i];
  return NRTO_OK;
}

// ---------------------------------------------------------------------------
// Incremental driving (nrto_solve_begin / _iterate / _flags / _end): the same
// kernels as the in-order schedule of nrto_inner_solve, in chunks of outer
// iterations, so that a multi-rank caller can interleave a batch-wide collective
// of the residual flags between chunks.
static cudaError_t fa_iteration_inorder(nrto_handle_s* h, int l, cudaStream_t st) {
  Dev& v = h->dev;
  const Dims& d = v.d;
  v.iter = l;
  v.ylazy = 0;
  cudaError_t e;
  if (v.fused == 0) {
    e = launch_fa_pass(h, st);
    if (e == cudaSuccess) e = launch_adjoint(h, v.Y, v.s, v.active, st);
    if (e == cudaSuccess) e = launch_fa_gain(h, st);
    if (e == cudaSuccess) e = launch_qp(h, NRTO_FULLADMM, l, st);
    return e;
  }
  e = v.fused == 2 ? launch_fa_tma(h, st) : launch_fa_fused(h, st);
  if (e == cudaSuccess && v.fused == 2) e = launch_fa_ctrl(h, st);
  if (e == cudaSuccess) e = launch_project(h, st);
  if (e == cudaSuccess)
    e = launch_zlist(h, v.Y, v.clist, v.cw, nullptr, v.ncorr, 0, v.active, v.Zc, st, 0,
                     v.fused == 2 ? 1 : 0, v.dG, v.dH);
  if (e == cudaSuccess) e = launch_fa_gain(h, st);
  const bool wide = d.B >= v.nsm || d.ng >= kQpSparseRows;
  if (e == cudaSuccess) e = wide ? launch_qp_sparse(h, NRTO_FULLADMM, l, st) : launch_qp(h, NRTO_FULLADMM, l, st);
  return e;
}

static cudaError_t dr_iteration(nrto_handle_s* h, int l, cudaStream_t st) {
  Dev& v = h->dev;
  cudaError_t e = launch_dr_arm(h, st);
  for (int m = 1; m <= v.prm.max_dr_iter && e == cudaSuccess; ++m) {
    e = launch_dr_gain(h, st);
    if (e == cudaSuccess) e = launch_dr_pass(h, st);
    if (e == cudaSuccess) e = launch_dr_adjoint(h, st);
    if (e == cudaSuccess) e = launch_dr_reduce(h, st);
  }
  if (e == cudaSuccess)
    e = (v.d.ng >= kQpSparseRows) ? launch_qp_sparse(h, NRTO_DR, l, st) : launch_qp(h, NRTO_DR, l, st);
  return e;
}

extern "C" nrto_err nrto_solve_begin(nrto_handle h, int32_t engine, void* stream) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (engine != NRTO_FULLADMM && engine != NRTO_DR) return fail(NRTO_EINVAL, "unknown engine");
  cudaStream_t st = (cudaStream_t)stream;
  Dev& v = h->dev;
  v.hist = nullptr;
  v.hist_L = engine == NRTO_FULLADMM ? v.prm.max_iter : v.prm.max_admm_iter;
  v.case_cnt = nullptr;
  if (h->general) return fail(NRTO_EINVAL, "general-set handles: use nrto_inner_solve");
  if (engine == NRTO_FULLADMM) {
    CK(launch_fa_reset(h, st));
  } else {
    if (!h->dr_ready) {
      CK(launch_engine_factors(h, NRTO_DR, st));
      const int se = read_setup_error(st);
      if (se) return fail(NRTO_ENOTSPD, se == 1 ? "W_K + sigma_dr/2 is not SPD" : "Riccati H_uu is not SPD");
      h->dr_ready = 1;
    }
    CK(launch_dr_reset(h, h->dr_fresh, st));
    h->dr_fresh = 0;
  }
  h->inc_engine = engine;
  h->inc_l = 0;
  return NRTO_OK;
}

extern "C" nrto_err nrto_solve_iterate(nrto_handle h, int32_t n_iters, int32_t* done, void* stream) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (h->inc_engine < 0) return fail(NRTO_ESTATE, "nrto_solve_iterate before nrto_solve_begin");
  if (n_iters < 0) return fail(NRTO_EINVAL, "n_iters < 0");
  cudaStream_t st = (cudaStream_t)stream;
  const int Lmax = h->inc_engine == NRTO_FULLADMM ? h->dev.prm.max_iter : h->dev.prm.max_admm_iter;
  const int l1 = std::min(Lmax, h->inc_l + n_iters);
  for (int l = h->inc_l + 1; l <= l1; ++l) {
    CK(h->inc_engine == NRTO_FULLADMM ? fa_iteration_inorder(h, l, st) : dr_iteration(h, l, st));
    h->inc_l = l;
  }
  if (done) *done = h->inc_l;
  return NRTO_OK;
}

extern "C" nrto_err nrto_solve_flags(nrto_handle h, double* flags, void* stream) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (!flags) return fail(NRTO_EINVAL, "flags is NULL");
  CK(launch_solve_flags(h, flags, (cudaStream_t)stream));
  return NRTO_OK;
}

// ---------------------------------------------------------------------------
// Cone sharding of one instance over ranks: the handle
// keeps the whole problem (setup, gain factors and QP over all rows, replicated on
// every rank) but its DR pass and adjoint cover cones [cone_lo, cone_hi) only; the
// caller sums the adjoint partials Z over ranks after every pass and gathers pi
// before every QP (nrto_buffer), stepping the DR loop with nrto_dr_step.
extern "C" nrto_err nrto_shard_cones(nrto_handle h, int32_t cone_lo, int32_t cone_hi) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  Dev& v = h->dev;
  const Dims& d = v.d;
  if (h->general) return fail(NRTO_EINVAL, "cone sharding needs a block-diagonal (nrto_setup) handle");
  if (cone_lo < 0 || cone_hi < cone_lo || cone_hi > d.ng) return fail(NRTO_EINVAL, "cone range out of [0, n_g]");
  cudaError_t ce = cudaDeviceSynchronize();
  std::vector<int32_t> knot(d.ng), kind(d.ng);
  if (ce == cudaSuccess && d.ng > 0) ce = cudaMemcpy(knot.data(), v.knot, d.ng * 4, cudaMemcpyDeviceToHost);
  if (ce == cudaSuccess && d.ng > 0) ce = cudaMemcpy(kind.data(), v.kind, d.ng * 4, cudaMemcpyDeviceToHost);
  // static per-step lists of the DR adjoint: owned cones with a b-block at step k
  std::vector<int32_t> kptr(d.T + 1, 0), kcone;
  for (int k = 0; k < d.T; ++k) {
    kptr[k] = (int32_t)kcone.size();
    for (int j = cone_lo; j < cone_hi; ++j)
      if ((kind[j] == 0 && knot[j] > k) || (kind[j] != 0 && knot[j] == k)) kcone.push_back(j);
  }
  kptr[d.T] = (int32_t)kcone.size();
  if (ce == cudaSuccess) ce = cudaMemcpy((void*)v.kptr, kptr.data(), (d.T + 1) * 4, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess && !kcone.empty())
    ce = cudaMemcpy((void*)v.kcone, kcone.data(), kcone.size() * 4, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMemset(v.rdr_part, 0, (size_t)std::max<int64_t>((int64_t)d.B * d.ng, 1) * 8);
  if (ce != cudaSuccess) return cuda_fail(ce, "nrto_shard_cones");
  v.cone_lo = cone_lo; v.cone_hi = cone_hi;
  h->sharded = 1;
  if (h->dr_exec) { cudaGraphExecDestroy(h->dr_exec); h->dr_exec = nullptr; }
  return NRTO_OK;
}

extern "C" nrto_err nrto_dr_step(nrto_handle h, int32_t phase, int32_t l, void* stream) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (h->inc_engine != NRTO_DR) return fail(NRTO_ESTATE, "nrto_dr_step outside nrto_solve_begin(NRTO_DR) .. _end");
  cudaStream_t st = (cudaStream_t)stream;
  Dev& v = h->dev;
  switch (phase) {
    case 0: CK(launch_dr_arm(h, st)); break;
    case 1: CK(launch_dr_gain(h, st)); break;
    case 2:
      CK(launch_dr_pass(h, st));
      CK(launch_dr_adjoint(h, st));
      CK(launch_dr_reduce(h, st));
      break;
    case 3:
      if (l < 1) return fail(NRTO_EINVAL, "outer iteration l >= 1");
      CK((v.d.ng >= kQpSparseRows) ? launch_qp_sparse(h, NRTO_DR, l, st) : launch_qp(h, NRTO_DR, l, st));
      h->inc_l = l;
      break;
    default: return fail(NRTO_EINVAL, "phase must be 0..3");
  }
  return NRTO_OK;
}

extern "C" nrto_err nrto_buffer(nrto_handle h, int32_t which, double** ptr, int64_t* count) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (!ptr || !count) return fail(NRTO_EINVAL, "NULL argument");
  const Dev& v = h->dev;
  const Dims& d = v.d;
  switch (which) {
    case 0: *ptr = v.Z; *count = (int64_t)d.B * d.T * d.nu * d.nx; break;
    case 1: *ptr = v.pt; *count = (int64_t)d.B * d.ng; break;
    case 2: *ptr = v.rdr_part; *count = (int64_t)d.B * d.ng; break;
    default: return fail(NRTO_EINVAL, "which must be 0..2");
  }
  return NRTO_OK;
}

extern "C" nrto_err nrto_solve_end(nrto_handle h, const nrto_out* o, void* stream) {
  if (!h) return fail(NRTO_ESTATE, "handle is NULL");
  if (!o) return fail(NRTO_EINVAL, "out is NULL");
  if (h->inc_engine < 0) return fail(NRTO_ESTATE, "nrto_solve_end before nrto_solve_begin");
  const int engine = h->inc_engine;
  h->inc_engine = -1;
  double *nu_d, *lam_d, *obj_d, *mc_d, *ml_d;
  const nrto_err se = out_staging(h, o, &nu_d, &lam_d, &obj_d, &mc_d, &ml_d);
  if (se != NRTO_OK) return se;
  return write_outputs(h, engine, o, (cudaStream_t)stream, nu_d, lam_d, obj_d, mc_d, ml_d);
}

// ---------------------------------------------------------------------------
// General uncertainty set (general.cu)
__global__ void k_fill_eye_blocks(double* Psi, int nblk, int nx, double* tau, int B) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)nblk * nx * nx;
  if (id < n) { const int64_t r = id % ((int64_t)nx * nx); Psi[id] = (r / nx == r % nx) ? 1.0 : 0.0; }
  if (id < B) tau[id] = 1.0;
}

extern "C" nrto_err nrto_setup_general(const nrto_shape* s, const nrto_data* data,
                                       const nrto_uncertainty* unc, const nrto_params* prm,
                                       void* stream, nrto_handle* out) {
  if (!out) return fail(NRTO_EINVAL, "out handle pointer is NULL");
  *out = nullptr;
  nrto_err e = check_shape(s);
  if (e != NRTO_OK) return e;
  if (!data || !unc || !prm) return fail(NRTO_EINVAL, "data / uncertainty / params is NULL");
  if (unc->n_z < 1 || !unc->Gamma || !unc->Psi) return fail(NRTO_EINVAL, "n_z >= 1, Gamma and Psi required");
  const int64_t NK = (int64_t)s->T * s->n_u * s->n_x;
  if (NK > 4096) return fail(NRTO_EINVAL, "general sets: T n_u n_x must be <= 4096 (dense M^-1)");
  cudaStream_t st = (cudaStream_t)stream;
  const bool host = data->memory == NRTO_MEM_HOST;
  const int64_t B = s->batch;
  // shadow primitives: Psi_k = I, tau = 1 -> the regular setup yields the raw costates
  double *psi = nullptr, *tau1 = nullptr, *taud = nullptr;
  const int64_t npsi = B * (s->T + 1) * s->n_x * s->n_x;
  CK(cudaMalloc((void**)&psi, (size_t)npsi * 8));
  CK(cudaMalloc((void**)&tau1, (size_t)B * 8));
  k_fill_eye_blocks<<<(unsigned)((std::max<int64_t>(npsi, B) + 255) / 256), 256, 0, st>>>(
      psi, (int)(B * (s->T + 1)), s->n_x, tau1, (int)B);
  nrto_data sd = *data;
  sd.memory = NRTO_MEM_DEVICE;
  std::vector<double*> tmp;
  auto dev_copy = [&](const double* src, int64_t n) -> const double* {
    if (!host || !src) return src;
    double* p = nullptr;
    if (cudaMalloc((void**)&p, (size_t)std::max<int64_t>(n, 1) * 8) != cudaSuccess) return nullptr;
    cudaMemcpyAsync(p, src, (size_t)n * 8, cudaMemcpyHostToDevice, st);
    tmp.push_back(p);
    return p;
  };
  const int T = s->T, nx = s->n_x, nu = s->n_u, ng = s->n_g;
  sd.A = dev_copy(data->A, B * T * nx * nx); sd.B = dev_copy(data->B, B * T * nx * nu);
  sd.grad = dev_copy(data->grad, B * ng * nx); sd.g0 = dev_copy(data->g0, B * ng);
  sd.W_K = dev_copy(data->W_K, B * T * nu * nu); sd.R_u = dev_copy(data->R_u, B * T * nu * nu);
  sd.u_hat = dev_copy(data->u_hat, B * T * nu); sd.r_trust = dev_copy(data->r_trust, B);
  sd.Psi = psi; sd.tau = tau1;
  nrto_handle h = nullptr;
  e = nrto_setup(s, &sd, prm, stream, &h);
  if (e == NRTO_OK) {
    cudaError_t ce = cudaMalloc((void**)&taud, (size_t)B * 8);
    if (ce == cudaSuccess) {
      h->gen.allocs[h->gen.nallocs++] = taud;
      ce = cudaMemcpyAsync(taud, data->tau, (size_t)B * 8, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st);
    }
    h->gen.tau = taud;
    int spd = 0;
    if (ce == cudaSuccess) ce = gen_setup(h, unc->Gamma, unc->Psi, unc->n_z, unc->memory == NRTO_MEM_HOST, st, &spd);
    if (ce != cudaSuccess) { e = cuda_fail(ce, "nrto_setup_general"); nrto_destroy(h); h = nullptr; }
    else if (spd) { e = fail(NRTO_ENOTSPD, "M^-1 = Q_v + rho sum A_hat^T A_hat is not SPD"); nrto_destroy(h); h = nullptr; }
    else h->general = 1;
  }
  cudaStreamSynchronize(st);
  for (double* p : tmp) cudaFree(p);
  cudaFree(psi); cudaFree(tau1);
  *out = h;
  return e;
}
