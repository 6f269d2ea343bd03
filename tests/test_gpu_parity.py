"""GPU parity: libnrto (through the C ABI) vs the CPU oracle on seeded inputs.

Tolerances (north_star): iterates 1e-9 normwise relative, final
objective and margins 1e-7.  Accumulators built from cancelling differences
(lam_p, lam_nu, margins) are measured against the norm of their operands
(tests.helpers.close).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen import make_instance, make_batch, stack_instances
from gen.problems import make_franka, make_quad, make_unicycle
from oracle import structured as st
from oracle.params import make_params
from oracle.soc import proj_soc
from tests.helpers import close

from paper_2603_02642_b200 import nrto


def _require_gpu():
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests must run on a B200")


def gpu_solve(shape, batch, engine, memory=nrto.NRTO_MEM_DEVICE, **pkw):
    _require_gpu()
    data = nrto.to_tensors(batch, device="cpu" if memory == nrto.NRTO_MEM_HOST else "cuda",
                           pinned=memory == nrto.NRTO_MEM_HOST)
    s = nrto.InnerSolver(shape, data, memory=memory, **pkw)
    out = s.solve(engine, memory=memory)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    s.close()
    return res


def single(shape, data):
    return stack_instances([(shape, data)])[1]


def oracle_run(shape, data, engine, **pkw):
    sp = st.StructuredProblem(shape, data)
    prm = make_params(**pkw)
    return st.fulladmm(sp, prm) if engine == nrto.NRTO_FULLADMM else st.nrto_admm_dr(sp, prm)


def assert_parity(g, o, i=0, tol=1e-9, tol_final=1e-7, engine=0):
    sc_p = np.linalg.norm(o["p"]) + np.linalg.norm(o["p_tilde"])
    assert close(g["kv"][i], o["kv"], tol=tol), "kv"
    assert close(g["du"][i], o["du"], tol=tol), "du"
    assert close(g["p"][i], o["p"], sc_p, tol=tol), "p"
    assert close(g["p_tilde"][i], o["p_tilde"], sc_p, tol=tol), "p_tilde"
    assert close(g["lam_p"][i], o["lam_p"], (40.0 if engine else 1.0) * sc_p, tol=tol), "lam_p"
    if engine == 0:
        assert close(g["nu"][i], o["nu"], tol=tol), "nu"
        assert close(g["lam_nu"][i], o["lam_nu"], np.linalg.norm(o["nu"]), tol=tol), "lam_nu"
    assert g["objective"][i] == pytest.approx(o["objective"], rel=tol_final, abs=1e-12)
    assert close(g["margin_cone"][i], o["margin_cone"], sc_p, tol=tol_final), "margin_cone"
    assert close(g["margin_lin"][i], o["margin_lin"], sc_p + np.linalg.norm(o["margin_lin"]),
                 tol=tol_final), "margin_lin"
    assert g["r_p"][i] == pytest.approx(o["r_p"], rel=1e-6, abs=1e-9 * (1 + sc_p))
    assert g["r_d"][i] == pytest.approx(o["r_d"], rel=1e-6, abs=1e-9 * (1 + sc_p))


# ------------------------------------------------------------------- SOC
def test_soc_project_parity():
    _require_gpu()
    rng = np.random.default_rng(0)
    lens = rng.integers(1, 200, 3000)
    lens[:5] = [1, 2, 31, 32, 33]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    y = rng.standard_normal(off[-1])
    t = rng.standard_normal(len(lens)) * rng.uniform(0.1, 20, len(lens))
    y[off[10]:off[11]] = 0.0; t[10] = 0.0          # a = 0, t = 0 -> keep
    y[off[11]:off[12]] = 0.0; t[11] = -1.0         # a = 0, t < 0 -> origin
    a12 = np.linalg.norm(y[off[12]:off[13]]); t[12] = a12     # boundary a = t
    a13 = np.linalg.norm(y[off[13]:off[14]]); t[13] = -a13    # boundary a = -t
    dt = torch.tensor(t, device="cuda"); dy = torch.tensor(y, device="cuda")
    doff = torch.tensor(off, device="cuda")
    to = torch.empty_like(dt); yo = torch.empty_like(dy)
    nrto.nrto_soc_project(dt, dy, doff, to, yo)
    to, yo = to.cpu().numpy(), yo.cpu().numpy()
    for j in range(len(lens)):
        tr, yr = proj_soc(t[j], y[off[j]:off[j + 1]])
        # the map is continuous: at a = +-t the reduction order of ||y|| may pick
        # the neighbouring case, which differs by O(ulp * (|t| + a))
        sc = 1e-14 * (abs(t[j]) + np.linalg.norm(y[off[j]:off[j + 1]]))
        assert abs(to[j] - tr) <= sc + 1e-14 * abs(tr)
        np.testing.assert_allclose(yo[off[j]:off[j + 1]], yr, rtol=1e-14, atol=sc)


# ----------------------------------------------------------- gain update
@pytest.mark.parametrize("maker", [lambda: make_unicycle(1, 0), lambda: make_franka(3, 0, T=10)])
def test_gain_update_parity(maker):
    _require_gpu()
    shape, data = maker()
    batch = single(shape, data)
    dt = nrto.to_tensors(batch)
    s = nrto.InnerSolver(shape, dt)
    sp = st.StructuredProblem(shape, data)
    rng = np.random.default_rng(1)
    nu = rng.standard_normal(sp.E)
    kp = rng.standard_normal(sp.NK)
    out = torch.empty(1, sp.NK, dtype=torch.float64, device="cuda")
    s.gain_update(torch.tensor(nu[None], device="cuda"), torch.tensor(kp[None], device="cuda"), out)
    torch.cuda.synchronize()
    # oracle: (14b) literally, M(Q_v k + rho sum A^T (nu - b_hat)) with M^-1 summed explicitly
    import scipy.linalg as sla
    rho = 10.0
    H = sp.gram_blocks(rho, 0.0)
    T, nu_, nx = shape.T, shape.n_u, shape.n_x
    K = st.unvec_cm(kp.reshape(T, -1), nu_, nx)
    Qk = st.vec_cm(2.0 * np.einsum("kab,kbc->kac", sp.W, K)).reshape(-1)
    rhs = Qk + rho * sp.adj(nu - sp.bhat_flat())
    n = nu_ * nx
    ref = np.concatenate([sla.solve(H[k], rhs[k * n:(k + 1) * n], assume_a="pos") for k in range(T)])
    assert close(out.cpu().numpy()[0], ref, tol=1e-11)
    s.close()


# ------------------------------------------------------------- FullADMM
CASES = {
    "c1": lambda: make_instance("c1"),
    "c2": lambda: make_instance("c2"),
    "c3s": lambda: make_franka(3, 0, T=12),
    "c4s": lambda: make_quad(4, 0, T=24, n_obs=30),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("L", [1, 2, 5, 40])
def test_fulladmm_parity(case, L):
    shape, data = CASES[case]()
    g = gpu_solve(shape, single(shape, data), nrto.NRTO_FULLADMM, max_iter=L, fixed_iters=1)
    o = oracle_run(shape, data, nrto.NRTO_FULLADMM, max_iter=L, fixed_iters=1)
    assert_parity(g, o)
    assert g["iters"][0] == L and g["status"][0] == nrto.NRTO_MAX_ITERS


def test_fulladmm_full_c3():
    shape, data = make_instance("c3")
    g = gpu_solve(shape, single(shape, data), nrto.NRTO_FULLADMM, max_iter=50, fixed_iters=1)
    o = oracle_run(shape, data, nrto.NRTO_FULLADMM, max_iter=50, fixed_iters=1)
    assert_parity(g, o)


@pytest.mark.parametrize("case", ["c1", "c3s"])
def test_fulladmm_termination(case):
    shape, data = CASES[case]()
    kw = dict(max_iter=400, eps_p=1e-4, eps_d=1e-4, check_every=2)
    g = gpu_solve(shape, single(shape, data), nrto.NRTO_FULLADMM, **kw)
    o = oracle_run(shape, data, nrto.NRTO_FULLADMM, **kw)
    assert g["status"][0] == o["status"]
    assert g["iters"][0] == o["iters"]
    assert_parity(g, o)


# ------------------------------------------------------------------- DR
@pytest.mark.parametrize("case,La,Ld", [("c1", 3, 12), ("c1", 6, 30), ("c2", 2, 6), ("c3s", 2, 8)])
def test_dr_parity(case, La, Ld):
    shape, data = CASES[case]()
    kw = dict(max_admm_iter=La, max_dr_iter=Ld, fixed_iters=1)
    g = gpu_solve(shape, single(shape, data), nrto.NRTO_DR, **kw)
    o = oracle_run(shape, data, nrto.NRTO_DR, **kw)
    assert_parity(g, o, engine=1)


def _solve_hist(shape, batch, engine, L, **pkw):
    _require_gpu()
    data = nrto.to_tensors(batch, device="cuda")
    s = nrto.InnerSolver(shape, data, **pkw)
    out = nrto.alloc_out(shape, 1, s.E, device="cuda")
    out["hist"] = torch.full((1, L, 3), -1.0, dtype=torch.float64, device="cuda")
    s.solve(engine, out=out)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    s.close()
    return res


@pytest.mark.parametrize("case", ["c1", "c3s"])
def test_residual_trace_fulladmm(case):
    """hist[l-1] = (r_p, r_d, 0) after iteration l vs the oracle's trace;
    rows after the instance stops are 0."""
    shape, data = CASES[case]()
    L = 60
    kw = dict(max_iter=L, eps_p=1e-4, eps_d=1e-4)
    g = _solve_hist(shape, single(shape, data), nrto.NRTO_FULLADMM, L, **kw)
    o = oracle_run(shape, data, nrto.NRTO_FULLADMM, **kw)
    n = int(o["iters"])
    assert int(g["iters"][0]) == n
    H = g["hist"][0]
    np.testing.assert_allclose(H[:n, 0], o["hist"][:, 0], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(H[:n, 1], o["hist"][:, 1], rtol=1e-6, atol=1e-9)
    assert np.all(H[:n, 2] == 0.0) and np.all(H[n:] == 0.0)


def test_residual_trace_dr():
    shape, data = CASES["c1"]()
    La, Ld = 5, 20
    kw = dict(max_admm_iter=La, max_dr_iter=Ld, fixed_iters=1)
    g = _solve_hist(shape, single(shape, data), nrto.NRTO_DR, La, **kw)
    tr = []
    sp = st.StructuredProblem(shape, data)
    st.nrto_admm_dr(sp, make_params(**kw), trace=tr)
    H = g["hist"][0]
    for l, t in enumerate(tr):
        assert H[l, 0] == pytest.approx(t["r_p"], rel=1e-6, abs=1e-9)
        assert H[l, 1] == pytest.approx(t["r_d"], rel=1e-6, abs=1e-9)
        assert H[l, 2] == pytest.approx(t["r_dr"], rel=1e-6, abs=1e-9)


def test_dr_early_stop_parity():
    shape, data = CASES["c1"]()
    kw = dict(max_admm_iter=8, max_dr_iter=100, eps_dr=1e-6, eps_p=1e-6, eps_d=1e-6)
    g = gpu_solve(shape, single(shape, data), nrto.NRTO_DR, **kw)
    o = oracle_run(shape, data, nrto.NRTO_DR, **kw)
    assert g["iters"][0] == o["iters"] and g["status"][0] == o["status"]
    assert_parity(g, o, engine=1)


# ---------------------------------------------------------------- batches
def test_batch_parity_c5_shape():
    items = [make_franka(5, i, T=12, jitter=True) for i in range(6)]
    shape, batch = stack_instances(items)
    g = gpu_solve(shape, batch, nrto.NRTO_FULLADMM, max_iter=20, fixed_iters=1)
    for i, (_, d) in enumerate(items):
        o = oracle_run(shape, d, nrto.NRTO_FULLADMM, max_iter=20, fixed_iters=1)
        assert_parity(g, o, i=i)


def test_dr_batch_parity_graph():
    """A small batch through the DR engine (fixed iterations: CUDA-graph replay,
    split fixed-list adjoint, CTA-per-cone pass) matches the oracle per instance."""
    items = [make_quad(2, i, T=12, n_obs=3) for i in range(3)]
    shape, batch = stack_instances(items)
    kw = dict(max_admm_iter=2, max_dr_iter=8, fixed_iters=1)
    g = gpu_solve(shape, batch, nrto.NRTO_DR, **kw)
    for i, (_, d) in enumerate(items):
        o = oracle_run(shape, d, nrto.NRTO_DR, **kw)
        assert_parity(g, o, i=i, engine=1)


def test_batch_per_instance_freeze():
    """Instances converge at different iterations and are frozen (R12)."""
    items = [make_unicycle(1, i) for i in range(5)]
    shape, batch = stack_instances(items)
    kw = dict(max_iter=300, eps_p=1e-5, eps_d=1e-5)
    g = gpu_solve(shape, batch, nrto.NRTO_FULLADMM, **kw)
    its = []
    for i, (_, d) in enumerate(items):
        o = oracle_run(shape, d, nrto.NRTO_FULLADMM, **kw)
        assert g["iters"][i] == o["iters"] and g["status"][i] == o["status"]
        assert_parity(g, o, i=i)
        its.append(o["iters"])
    assert len(set(its)) > 1


def test_bench_config_sampled():
    """The bench workload (c5 batch of Franka c3 instances, L=50 fixed) at full
    size: every instance finite; two sampled instances against the oracle."""
    B = 64
    shape, batch = make_batch("c5", B)
    g = gpu_solve(shape, batch, nrto.NRTO_FULLADMM, max_iter=50, fixed_iters=1)
    for k in ("kv", "du", "p", "p_tilde", "nu", "lam_nu", "objective"):
        assert np.all(np.isfinite(g[k])), k
    for i in (0, B - 1):
        d = {k: v[i] for k, v in batch.items()}
        d["tau"] = float(d["tau"]); d["r_trust"] = float(d["r_trust"])
        o = oracle_run(shape, d, nrto.NRTO_FULLADMM, max_iter=50, fixed_iters=1)
        assert_parity(g, o, i=i)


def test_overlapped_lazy_batch():
    """B >= #SMs and fixed iterations: QP overlapped with the next pass and lazy
    y storage.  Sampled instances against the oracle; the whole batch
    against the eager in-order schedule (termination mode, eps = 0); the pass
    byte counter between its bounds."""
    _require_gpu()
    B, L = 160, 20
    items = [make_franka(5, i, T=12, jitter=True) for i in range(B)]
    shape, batch = stack_instances(items)
    data = nrto.to_tensors(batch, device="cuda")
    s = nrto.InnerSolver(shape, data, max_iter=L, fixed_iters=1)
    s.pass_bytes()
    g = {k: v.cpu().numpy() for k, v in s.solve(nrto.NRTO_FULLADMM).items()}
    moved = s.pass_bytes()
    s.close()
    for i in (0, 77, B - 1):
        o = oracle_run(shape, items[i][1], nrto.NRTO_FULLADMM, max_iter=L, fixed_iters=1)
        assert_parity(g, o, i=i)
    e = gpu_solve(shape, batch, nrto.NRTO_FULLADMM, max_iter=L, eps_p=0.0, eps_d=0.0)
    assert np.all(e["iters"] == L)
    for k in ("kv", "du", "p", "p_tilde", "lam_p", "nu", "lam_nu", "objective"):
        assert close(g[k], e[k], tol=1e-11), k
    kind = np.asarray(shape.cone_kind); knot = np.asarray(shape.cone_knot)
    st_ = kind == 0
    Es = int(((knot[st_] + 1) * shape.n_x).sum())
    EBs = int((knot[st_] * (shape.n_u + shape.n_u % 2)).sum())
    lo = 8 * B * L * (Es + EBs)                    # b_hat and b every iteration
    hi = 8 * B * L * (3 * Es + EBs)                # + y read and written every iteration
    assert lo < moved < hi


def test_host_memory_path_matches_device():
    shape, data = CASES["c3s"]()
    b = single(shape, data)
    gd = gpu_solve(shape, b, nrto.NRTO_FULLADMM, max_iter=7, fixed_iters=1)
    gh = gpu_solve(shape, b, nrto.NRTO_FULLADMM, memory=nrto.NRTO_MEM_HOST, max_iter=7, fixed_iters=1)
    for k in gd:   # same kernels; only the (atomic) order of the adjoint correction differs
        assert close(gh[k], gd[k], tol=1e-12), k


def test_setup_rejects_non_spd_weights():
    _require_gpu()
    shape, data = CASES["c1"]()
    data = dict(data)
    data["W_K"] = -np.asarray(data["W_K"])
    with pytest.raises(nrto.NrtoError) as ei:
        nrto.InnerSolver(shape, nrto.to_tensors(single(shape, data)))
    assert ei.value.code == nrto.NRTO_ENOTSPD


def test_empty_cone_set():
    """n_g = 0: M = Q_v^-1, k_v stays 0, the QP has only the trust region."""
    _require_gpu()
    from gen.problems import Shape
    shape, data = make_unicycle(1, 0, T=5)
    sh0 = Shape(shape.n_x, shape.n_u, shape.T, np.zeros(0, np.int32), np.zeros(0, np.int8))
    d0 = dict(data); d0["grad"] = np.zeros((0, shape.n_x)); d0["g0"] = np.zeros(0)
    g = gpu_solve(sh0, single(sh0, d0), nrto.NRTO_FULLADMM, max_iter=5, fixed_iters=1)
    o = oracle_run(sh0, d0, nrto.NRTO_FULLADMM, max_iter=5, fixed_iters=1)
    assert np.all(g["kv"] == 0)
    assert close(g["du"][0], o["du"], tol=1e-9)


# ------------------------------------------------ c4: long horizons (other kernel paths)
@pytest.mark.parametrize("T,n_obs,L", [(150, 6, 3), (200, 4, 2), (400, 2, 1)])
def test_fulladmm_long_horizon(T, n_obs, L):
    """T=150: shared-memory-Z fused pass; T>=200: generic pass + dense adjoint."""
    shape, data = make_quad(4, 7, T=T, n_obs=n_obs)
    g = gpu_solve(shape, single(shape, data), nrto.NRTO_FULLADMM, max_iter=L, fixed_iters=1)
    o = oracle_run(shape, data, nrto.NRTO_FULLADMM, max_iter=L, fixed_iters=1)
    assert_parity(g, o)


def test_dr_long_horizon():
    shape, data = make_quad(4, 8, T=150, n_obs=4)
    kw = dict(max_admm_iter=2, max_dr_iter=3, fixed_iters=1)
    g = gpu_solve(shape, single(shape, data), nrto.NRTO_DR, **kw)
    o = oracle_run(shape, data, nrto.NRTO_DR, **kw)
    assert_parity(g, o, engine=1)


@pytest.mark.gpu
def test_dr_graph_replay_matches_stream_path():
    """The fixed-iteration DR loop runs as a captured CUDA graph (replayed on the
    second solve of a handle); with the profiler on it runs launch by launch.
    Both orders of the same kernels must give the same warm-started result."""
    _require_gpu()
    shape, data = CASES["c2"]()
    kw = dict(max_admm_iter=3, max_dr_iter=10, fixed_iters=1)
    outs = []
    for prof in (False, True):
        s = nrto.InnerSolver(shape, nrto.to_tensors(single(shape, data), device="cuda"), **kw)
        o = nrto.alloc_out(shape, 1, s.E, device="cuda")
        s.solve(nrto.NRTO_DR, out=o)
        s.solve(nrto.NRTO_DR, out=o)            # graph replay (prof off)
        if prof:
            s.profile(True)
        s.solve(nrto.NRTO_DR, out=o)
        torch.cuda.synchronize()
        outs.append({k: v.cpu().numpy() for k, v in o.items()})
        s.close()
    g, e = outs
    for k in ("kv", "du", "p", "p_tilde", "lam_p"):
        assert close(g[k], e[k], tol=1e-12), k


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c1", "c3s"])
def test_fulladmm_graph_replay_matches_stream_path(case):
    """Small-batch fixed-iteration FullADMM solves run as a captured CUDA graph
    (replayed from the second solve on); with the profiler on they run launch by
    launch.  The same solve must give the same result either way, and match the
    oracle."""
    _require_gpu()
    shape, data = CASES[case]()
    kw = dict(max_iter=6, fixed_iters=1)
    outs = []
    for prof in (False, True):
        s = nrto.InnerSolver(shape, nrto.to_tensors(single(shape, data), device="cuda"), **kw)
        o = nrto.alloc_out(shape, 1, s.E, device="cuda")
        s.solve(nrto.NRTO_FULLADMM, out=o)
        s.solve(nrto.NRTO_FULLADMM, out=o)        # graph replay (prof off)
        if prof:
            s.profile(True)
        s.solve(nrto.NRTO_FULLADMM, out=o)
        torch.cuda.synchronize()
        outs.append({k: v.cpu().numpy() for k, v in o.items()})
        s.close()
    g, e = outs
    for k in ("kv", "du", "p", "p_tilde", "lam_p"):
        assert close(g[k], e[k], tol=1e-12), k
    assert_parity({k: v for k, v in g.items()}, oracle_run(shape, data, nrto.NRTO_FULLADMM, **kw))
