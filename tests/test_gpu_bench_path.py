"""GPU parity of the exact bench path and of the configurations round 1 left untested.

* the bench workload itself: c5, B = 512, T = 100, L = 50 fixed iterations, in
  the overlapped schedule bench.py times (B >= #SMs: QP(l) on the low-priority
  stream beside pass(l+1), persistent QP grid looping over > 1 instance per CTA,
  control cones on the second high-priority stream, lazy y) -- instances
  {0, 137, 300, 511} against the oracle normwise AND element-wise, and the
  stationarity invariant sum_j rho A_hat_j^T lam_nu,j + Q_v k_v = 0
  on EVERY instance, evaluated by an independent torch checker (test-side code,
  plain batched matmuls, no libnrto kernel);
* the same workload with termination on (eps_p = eps_d = 1e-3): the iteration at
  which each sampled instance stops equals the oracle's, recorded by
  scripts/workload_check.py (oracle only) in tests/golden/workload_c3_c5.json;
* c2 NRTO-DR at the bench's 40 x 100 warm-started configuration;
* c4 at T = 800 (generic pass, dense list adjoint, 128-thread QP, DR long-cone pass);
* random SPD W_K, non-diagonal R_u and a distinct Psi_k per step;
* a NaN input gives status NRTO_DIVERGED for that instance only;
* nrto_gain_update between two DR solves leaves the DR warm start intact.

Element-wise parity (tests.helpers.elementwise): max_i |x_i - ref_i| /
(|ref_i| + f ||ref||_inf) <= tol, f = 1e-3 -- an error confined to a small subset
of entries (e.g. the control-cone entries of nu) cannot hide in a norm.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen import make_instance, make_batch, stack_instances
from gen.problems import make_franka, make_quad, make_unicycle
from oracle import structured as st
from oracle.params import make_params
from tests.helpers import close, elementwise, golden

from paper_2603_02642_b200 import nrto

from tests.test_gpu_parity import assert_parity, gpu_solve, oracle_run, single, _require_gpu


def _inst(batch, i):
    d = {k: np.array(v[i]) for k, v in batch.items()}
    d["tau"] = float(d["tau"]); d["r_trust"] = float(d["r_trust"])
    return d


def assert_elementwise(g, o, i=0, tol=1e-9, engine=0):
    keys = ["kv", "du", "p", "p_tilde"] + (["nu"] if engine == 0 else [])
    for k in keys:
        err = elementwise(g[k][i], o[k])
        assert err <= tol, f"{k}: element-wise {err:.3e} > {tol:.1e}"


# ------------------------------------------------ independent stationarity checker
def stationarity_torch(shape, batch, kv, lam_nu, rho, dev):
    """|| sum_j rho A_hat_j^T lam_nu,j + Q_v k_v || per instance, relative to
    1 + ||Q_v k_v||, from the definitions of P:846-869 (costate sweeps
    c_{j,k} = A_k^T c_{j,k+1}, b_{j,k} = B_k^T c_{j,k+1}; block k of A_hat_j^T e_j =
    sqrt(tau) vec(b_{j,k} (Psi_k^T e_{j,k})^T); Q_v = 2 blkdiag(I (x) W_k)).
    Plain batched torch matmuls on the GPU (test-side; shares no code with libnrto)."""
    B = kv.shape[0]
    nx, nu, T = shape.n_x, shape.n_u, shape.T
    knot = np.asarray(shape.cone_knot); kind = np.asarray(shape.cone_kind)
    off = st.ragged_layout(shape)
    t = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.float64, device=dev)
    A, Bm, grad, Psi = t(batch["A"]), t(batch["B"]), t(batch["grad"]), t(batch["Psi"])
    W = t(batch["W_K"]); sq = torch.sqrt(t(batch["tau"])).view(B, 1, 1)
    lam = torch.as_tensor(lam_nu, device=dev)
    G = torch.zeros(B, T, nu, nx, dtype=torch.float64, device=dev)
    for kj in range(1, T + 1):                        # state cones, grouped by knot
        rows = np.nonzero((kind == 0) & (knot == kj))[0]
        if len(rows) == 0:
            continue
        c = grad[:, rows, :]                           # c_{j,k_j} = grad g_j
        for k in range(kj - 1, -1, -1):
            b = torch.einsum("brx,bxu->bru", c, Bm[:, k])          # B_k^T c_{j,k+1}
            idx = torch.as_tensor((off[rows][:, None] + k * nx + np.arange(nx)[None, :]), device=dev)
            e = lam[:, idx]                                         # [B, r, nx]
            pe = torch.einsum("brx,bxy->bry", e, Psi[:, k])        # (Psi_k^T e)^T
            G[:, k] += torch.einsum("bru,bry->buy", b, pe)
            c = torch.einsum("brx,bxy->bry", c, A[:, k])           # A_k^T c_{j,k+1}
    for k in range(T):                                 # control cones: b = h'_j at block k
        rows = np.nonzero((kind == 1) & (knot == k))[0]
        if len(rows) == 0:
            continue
        b = grad[:, rows, :nu]
        idx = torch.as_tensor(off[rows][:, None] + np.arange(nx)[None, :], device=dev)
        pe = torch.einsum("brx,bxy->bry", lam[:, idx], Psi[:, k])
        G[:, k] += torch.einsum("bru,bry->buy", b, pe)
    K = torch.as_tensor(kv, device=dev).view(B, T, nx, nu).transpose(-1, -2)   # column-major vec
    QK = 2.0 * torch.einsum("bkuv,bkvx->bkux", W, K)
    R = QK + rho * sq.view(B, 1, 1, 1) * G
    res = torch.linalg.vector_norm(R.reshape(B, -1), dim=1)
    ref = 1.0 + torch.linalg.vector_norm(QK.reshape(B, -1), dim=1)
    return (res / ref).cpu().numpy()


# --------------------------------------------------------------- the bench path
@pytest.fixture(scope="module")
def bench_batch():
    return make_batch("c5", 512)


def test_bench_path_overlapped_b512(bench_batch):
    """The exact bench configuration (bench.py: c5, 512 instances, L = 50,
    fixed_iters, overlapped schedule) against the oracle, element-wise."""
    _require_gpu()
    shape, batch = bench_batch
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    assert 512 >= 2 * nsm, "the persistent QP grid must loop over > 1 instance per CTA"
    L = 50
    data = nrto.to_tensors(batch, device="cuda")
    s = nrto.InnerSolver(shape, data, max_iter=L, fixed_iters=1)
    out = nrto.alloc_out(shape, 512, s.E, device="cuda", full=True)
    s.solve(nrto.NRTO_FULLADMM, out=out)          # first solve (state of a fresh handle)
    s.solve(nrto.NRTO_FULLADMM, out=out)          # second solve: the bench's steady state
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    for k in ("kv", "du", "p", "p_tilde", "lam_p", "nu", "lam_nu", "objective", "margin_cone",
              "margin_lin", "r_p", "r_d"):
        assert np.all(np.isfinite(g[k])), k
    assert np.all(g["iters"] == L) and np.all(g["status"] == nrto.NRTO_MAX_ITERS)
    for i in (0, 137, 300, 511):
        o = oracle_run(shape, _inst(batch, i), nrto.NRTO_FULLADMM, max_iter=L, fixed_iters=1)
        assert_parity(g, o, i=i)
        assert_elementwise(g, o, i=i)
    inv = stationarity_torch(shape, batch, out["kv"], out["lam_nu"], 10.0, "cuda")
    assert np.all(inv <= 1e-10), f"stationarity invariant max {inv.max():.3e}"
    s.close()


def test_bench_workload_converges_like_the_oracle(bench_batch):
    """Termination on (eps_p = eps_d = 1e-3, checked every iteration, L_max = 600):
    the sampled instances stop at the oracle's iteration (golden record written
    by scripts/workload_check.py, oracle only) and every instance converges."""
    _require_gpu()
    shape, batch = bench_batch
    ref = {(c["cfg"], c["instance"]): c for c in golden("workload_c3_c5.json")["cases"]}
    g = gpu_solve(shape, batch, nrto.NRTO_FULLADMM, max_iter=600, eps_p=1e-3, eps_d=1e-3)
    assert np.all(g["status"] == nrto.NRTO_CONVERGED), \
        f"{int(np.sum(g['status'] != 0))} instances did not converge in 600 iterations"
    for i in (0, 137, 300, 511):
        assert int(g["iters"][i]) == ref[("c5", i)]["iters"], i
    # c3 (the single-instance Franka config) converges at the oracle's iteration too
    sh3, d3 = make_instance("c3")
    g3 = gpu_solve(sh3, single(sh3, d3), nrto.NRTO_FULLADMM, max_iter=600, eps_p=1e-3, eps_d=1e-3)
    assert int(g3["status"][0]) == 0 and int(g3["iters"][0]) == ref[("c3", 0)]["iters"]


# --------------------------------------------------------------- other configs
def test_c2_dr_bench_configuration():
    """c2 quadcopter NRTO-DR at the bench's 40 x 100 (fixed, warm-started DR)."""
    shape, data = make_instance("c2")
    kw = dict(max_admm_iter=40, max_dr_iter=100, fixed_iters=1)
    g = gpu_solve(shape, single(shape, data), nrto.NRTO_DR, **kw)
    o = oracle_run(shape, data, nrto.NRTO_DR, **kw)
    assert_parity(g, o, engine=1)
    assert_elementwise(g, o, engine=1, tol=1e-8)


def test_c4_t800_fulladmm_and_dr():
    """T = 800 (beyond the TMA pass's shared-memory horizon): the generic pass,
    dense list adjoint, 128-thread QP and the DR long-cone pass."""
    shape, data = make_quad(4, 11, T=800, n_obs=2)
    g = gpu_solve(shape, single(shape, data), nrto.NRTO_FULLADMM, max_iter=2, fixed_iters=1)
    o = oracle_run(shape, data, nrto.NRTO_FULLADMM, max_iter=2, fixed_iters=1)
    assert_parity(g, o)
    kw = dict(max_admm_iter=2, max_dr_iter=2, fixed_iters=1)
    g = gpu_solve(shape, single(shape, data), nrto.NRTO_DR, **kw)
    o = oracle_run(shape, data, nrto.NRTO_DR, **kw)
    assert_parity(g, o, engine=1)


def _random_weights(shape, data, seed):
    """Random SPD W_K and R_u per step (non-diagonal) and a distinct upper-triangular
    Psi_k (positive diagonal) per step -- exercises the generalised eigen chain with
    W != I, non-diagonal R_u in the Riccati / QP, and per-step Psi / U."""
    rng = np.random.default_rng(seed)
    T, nu, nx = shape.T, shape.n_u, shape.n_x
    d = dict(data)

    def spd(n, lo, hi):
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        return (Q * rng.uniform(lo, hi, n)) @ Q.T

    d["W_K"] = np.stack([spd(nu, 0.3, 3.0) for _ in range(T)])
    d["R_u"] = np.stack([spd(nu, 0.02, 0.5) for _ in range(T)])
    P = np.array(data["Psi"], float)
    for k in range(T + 1):
        U = np.triu(rng.standard_normal((nx, nx))) * 0.3 * np.abs(np.diag(P[k])).mean()
        U[np.diag_indices(nx)] = np.abs(np.diag(P[k])) * rng.uniform(0.5, 2.0, nx)
        P[k] = U
    d["Psi"] = P
    return d


@pytest.mark.parametrize("case", ["c1", "c3s"])
def test_random_weights_and_psi(case):
    shape, data = make_instance("c1") if case == "c1" else make_franka(3, 0, T=12)
    d = _random_weights(shape, data, 7)
    for L in (2, 20):
        g = gpu_solve(shape, single(shape, d), nrto.NRTO_FULLADMM, max_iter=L, fixed_iters=1)
        o = oracle_run(shape, d, nrto.NRTO_FULLADMM, max_iter=L, fixed_iters=1)
        assert_parity(g, o)
        assert_elementwise(g, o, tol=1e-8)
    kw = dict(max_admm_iter=3, max_dr_iter=10, fixed_iters=1)
    g = gpu_solve(shape, single(shape, d), nrto.NRTO_DR, **kw)
    o = oracle_run(shape, d, nrto.NRTO_DR, **kw)
    assert_parity(g, o, engine=1)


def test_random_weights_batch_tma_path():
    """Random W_K / R_u / Psi_k through the batched TMA pass and sparse QP."""
    items = []
    for i in range(4):
        sh, d = make_franka(5, i, T=12, jitter=True)
        items.append((sh, _random_weights(sh, d, 100 + i)))
    shape, batch = stack_instances(items)
    g = gpu_solve(shape, batch, nrto.NRTO_FULLADMM, max_iter=10, fixed_iters=1)
    for i, (_, d) in enumerate(items):
        o = oracle_run(shape, d, nrto.NRTO_FULLADMM, max_iter=10, fixed_iters=1)
        assert_parity(g, o, i=i)


def test_nan_input_diverges_that_instance_only():
    """Non-finite iterates are reported as NRTO_DIVERGED per instance, not
    as an error; the other instances of the batch are unaffected."""
    items = [make_unicycle(1, i) for i in range(3)]
    bad = dict(items[1][1]); g0 = np.array(bad["g0"], float); g0[5] = np.nan; bad["g0"] = g0
    items[1] = (items[1][0], bad)
    shape, batch = stack_instances(items)
    g = gpu_solve(shape, batch, nrto.NRTO_FULLADMM, max_iter=40)
    assert g["status"][1] == nrto.NRTO_DIVERGED
    for i in (0, 2):
        o = oracle_run(shape, items[i][1], nrto.NRTO_FULLADMM, max_iter=40)
        assert g["status"][i] == o["status"] and g["iters"][i] == o["iters"]
        assert_parity(g, o, i=i)


def test_gain_update_keeps_dr_warm_start():
    """DR solve -> nrto_gain_update -> DR solve equals DR solve -> DR solve (the DR
    warm state persists across calls)."""
    _require_gpu()
    shape, data = make_instance("c1")
    kw = dict(max_admm_iter=3, max_dr_iter=10, fixed_iters=1)
    res = []
    for between in (False, True):
        s = nrto.InnerSolver(shape, nrto.to_tensors(single(shape, data), device="cuda"), **kw)
        o = nrto.alloc_out(shape, 1, s.E, device="cuda")
        s.solve(nrto.NRTO_DR, out=o)
        if between:
            nu = torch.randn(1, s.E, dtype=torch.float64, device="cuda")
            kp = torch.randn(1, shape.T * shape.n_u * shape.n_x, dtype=torch.float64, device="cuda")
            s.gain_update(nu, kp, torch.empty_like(kp))
        s.solve(nrto.NRTO_DR, out=o)
        torch.cuda.synchronize()
        res.append({k: v.cpu().numpy() for k, v in o.items()})
        s.close()
    for k in ("kv", "du", "p", "p_tilde", "lam_p"):
        assert close(res[1][k], res[0][k], tol=1e-13), k


# ------------------------------------------------ incremental ABI, case stats, collective
@pytest.mark.parametrize("case", ["c1", "c3s", "batch"])
def test_incremental_solve_matches_inner_solve(case):
    """nrto_solve_begin/_iterate/_flags/_end (chunks of check_every, the host-side
    termination test of the multi-rank loop) give the same per-instance
    iterations, status and iterates as nrto_inner_solve in termination mode."""
    _require_gpu()
    from paper_2603_02642_b200.dist import solve_collective
    if case == "batch":
        items = [make_franka(5, i, T=12, jitter=True) for i in range(6)]
        shape, batch = stack_instances(items)
    else:
        shape, data = make_instance("c1") if case == "c1" else make_franka(3, 0, T=12)
        batch = single(shape, data)
    kw = dict(max_iter=300, eps_p=1e-4, eps_d=1e-4, check_every=3)
    ref = gpu_solve(shape, batch, nrto.NRTO_FULLADMM, **kw)
    s = nrto.InnerSolver(shape, nrto.to_tensors(batch, device="cuda"), **kw)
    out, done, ncoll = solve_collective(s, nrto.NRTO_FULLADMM, allreduce=None)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    s.close()
    assert ncoll == 0 and done == int(ref["iters"].max()) and done % 3 == 0
    np.testing.assert_array_equal(g["iters"], ref["iters"])
    np.testing.assert_array_equal(g["status"], ref["status"])
    for k in ("kv", "du", "p", "p_tilde", "lam_p", "nu", "lam_nu"):
        assert close(g[k], ref[k], tol=1e-12), k


def test_case_stats_match_oracle():
    """Per-iteration projection-case histogram (nrto_case_stats_*) equals the
    oracle's case counts of SM Eq.(18), iteration by iteration."""
    _require_gpu()
    for shape, data in (make_instance("c1"), make_franka(3, 0, T=12)):
        L = 30
        s = nrto.InnerSolver(shape, nrto.to_tensors(single(shape, data), device="cuda"),
                             max_iter=L, fixed_iters=1)
        s.case_stats(True)
        s.solve(nrto.NRTO_FULLADMM)
        cnt = s.case_stats_read()
        s.close()
        o = oracle_run(shape, data, nrto.NRTO_FULLADMM, max_iter=L, fixed_iters=1)
        assert np.all(cnt.sum(1) == shape.n_g)
        np.testing.assert_array_equal(cnt, np.asarray(o["cases"]))


_MP_CHILD = r"""
import json, os, sys
sys.path.insert(0, %r)
import torch.multiprocessing as mp


def worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_02642_b200 import nrto
    from paper_2603_02642_b200.dist import solve_collective, instance_range
    from gen.problems import make_unicycle
    from gen import stack_instances
    first, count = instance_range(rank, world, 2)
    shape, batch = stack_instances([make_unicycle(1, i) for i in range(first, first + count)])
    s = nrto.InnerSolver(shape, nrto.to_tensors(batch, device="cuda"), max_iter=300, eps_p=1e-5,
                         eps_d=1e-5, check_every=2)

    def allreduce(f):                 # gloo on one GPU: reduce a host copy of the device flags
        c = f.cpu()
        dist.all_reduce(c, op=dist.ReduceOp.MAX)
        f.copy_(c)

    o, done, ncoll = solve_collective(s, nrto.NRTO_FULLADMM, allreduce=allreduce)
    torch.cuda.synchronize()
    q.put((rank, first, o["iters"].cpu().numpy().tolist(), o["kv"].cpu().numpy().tolist(), done, ncoll))
    s.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    port = int(sys.argv[1])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps: p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in ps: p.join()
    print(json.dumps({str(r[0]): r[1:] for r in res}))
"""


def test_two_process_collective_loop_on_one_gpu():
    """Two ranks (processes) on one GPU, instances sharded, the termination test
    allreduced every check_every iterations: both ranks run until the slowest
    instance of EITHER shard has converged, and every instance's result equals
    its single-process solve.  The ranks run under a child interpreter, so this
    pytest process never forks (an OpenBLAS call of the oracle deadlocked in it
    after an in-process torch.multiprocessing Manager)."""
    _require_gpu()
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s_ = socket.socket(); s_.bind(("127.0.0.1", 0)); port = s_.getsockname()[1]; s_.close()
    import tempfile
    with tempfile.TemporaryDirectory() as td:         # spawn re-imports the main module: a file
        script = os.path.join(td, "two_ranks.py")
        with open(script, "w") as f:
            f.write(_MP_CHILD % root)
        r = subprocess.run([sys.executable, script, str(port)], capture_output=True, text=True,
                           timeout=280)
    assert r.returncode == 0, r.stderr[-3000:]
    out = {int(k): v for k, v in json.loads(r.stdout.strip().splitlines()[-1]).items()}
    items = [make_unicycle(1, i) for i in range(4)]
    shape, batch = stack_instances(items)
    ref = gpu_solve(shape, batch, nrto.NRTO_FULLADMM, max_iter=300, eps_p=1e-5, eps_d=1e-5, check_every=2)
    last = int(ref["iters"].max())
    for rk in range(2):
        first, iters, kv, done, ncoll = out[rk]
        assert done == last and ncoll == last // 2          # global stop, one collective per chunk
        np.testing.assert_array_equal(iters, ref["iters"][first:first + 2])
        assert close(np.array(kv), ref["kv"][first:first + 2], tol=1e-12)


def _oracle_c5(i):
    """Oracle FullADMM of c5 instance i, L = 50 (worker of a spawn-context pool)."""
    import os, sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from threadpoolctl import threadpool_limits
    from gen import make_instance
    from oracle import structured as st_
    from oracle.params import make_params as mp_
    with threadpool_limits(limits=1):
        shape, data = make_instance("c5", i)
        o = st_.fulladmm(st_.StructuredProblem(shape, data), mp_(max_iter=50, fixed_iters=1))
    return i, {k: o[k] for k in ("kv", "du", "p", "p_tilde", "lam_p", "nu", "lam_nu", "objective",
                                 "margin_cone", "margin_lin", "r_p", "r_d")}


def test_bench_path_64_instances_vs_oracle(bench_batch):
    """SURVEY §8(c) c5 protocol: the exact bench configuration (512 instances,
    overlapped schedule, L = 50) against the oracle on 64 instances (every 8th),
    element-wise; the oracle runs in a spawn-context process pool (this pytest
    process never forks)."""
    _require_gpu()
    import multiprocessing as mp
    import os
    shape, batch = bench_batch
    s = nrto.InnerSolver(shape, nrto.to_tensors(batch, device="cuda"), max_iter=50, fixed_iters=1)
    out = nrto.alloc_out(shape, 512, s.E, device="cuda", full=True)
    s.solve(nrto.NRTO_FULLADMM, out=out)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    s.close()
    ids = list(range(0, 512, 8))
    with mp.get_context("spawn").Pool(max(1, min(32, os.cpu_count() or 1))) as pool:
        res = dict(pool.map(_oracle_c5, ids))
    for i in ids:
        assert_parity(g, res[i], i=i)
        assert_elementwise(g, res[i], i=i)
