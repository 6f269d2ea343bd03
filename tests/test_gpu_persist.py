"""GPU: the single-instance paths of SURVEY §8f NEXT-3 against the oracle and
against the kernels they replace (switched off by environment in a child
process): the persistent single-launch DR loop (csrc/persist.cu, NEXT-3(ii),
NRTO_DR_PERSIST=0) and the chunked-scan (parallel-in-time) Riccati QP
(csrc/qp.cu k_qp_scan, NEXT-3(iii), NRTO_QP_SCAN=0)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen import stack_instances
from gen.problems import make_quad, make_unicycle
from tests.helpers import close
from tests.test_gpu_parity import CASES, assert_parity, gpu_solve, oracle_run, single

from paper_2603_02642_b200 import nrto

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np, torch
from tests.test_gpu_parity import CASES, single
from paper_2603_02642_b200 import nrto
case, eng = sys.argv[1], int(sys.argv[2])
shape, data = CASES[case]()
kw = dict(max_admm_iter=3, max_dr_iter=12, fixed_iters=1) if eng else dict(max_iter=12, fixed_iters=1)
s = nrto.InnerSolver(shape, nrto.to_tensors(single(shape, data), device="cuda"), **kw)
o = nrto.alloc_out(shape, 1, s.E, device="cuda")
res = []
for _ in range(2):                      # second solve: warm DR state (P:1340)
    s.solve(eng, out=o)
    torch.cuda.synchronize()
    res.append({k: o[k].cpu().numpy().ravel().tolist() for k in ("kv", "du", "p", "p_tilde", "lam_p")})
print(json.dumps(res))
"""


def _run_child(case, eng, **env_kw):
    env = dict(os.environ, **{k: str(v) for k, v in env_kw.items()})
    r = subprocess.run([sys.executable, "-c", CHILD % ROOT, case, str(eng)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_persistent_dr_matches_launch_per_phase_path():
    """Same warm-started c2 solves (two calls) through both DR implementations."""
    a = _run_child("c2", 1, NRTO_DR_PERSIST=1)
    b = _run_child("c2", 1, NRTO_DR_PERSIST=0, NRTO_QP_SCAN=1)
    for sa, sb in zip(a, b):
        for k in sa:
            assert close(np.array(sa[k]), np.array(sb[k]), tol=1e-11), k


def test_persistent_dr_batch_ragged_instances():
    """A batch of 5 quadcopters (persistent path, several instances share the grid:
    item and task loops wrap) matches the oracle instance by instance."""
    items = [make_quad(2, i, T=16, n_obs=4) for i in range(5)]
    shape, batch = stack_instances(items)
    kw = dict(max_admm_iter=3, max_dr_iter=9, fixed_iters=1)
    g = gpu_solve(shape, batch, nrto.NRTO_DR, **kw)
    for i, (_, d) in enumerate(items):
        o = oracle_run(shape, d, nrto.NRTO_DR, **kw)
        assert_parity(g, o, i=i, engine=1)


def test_persistent_dr_early_stop_per_instance():
    """DR stop test inside the persistent loop (every CTA derives r_dr itself):
    instances stop their DR loops at different iterations, as in the oracle."""
    items = [make_unicycle(1, i) for i in range(4)]
    shape, batch = stack_instances(items)
    kw = dict(max_admm_iter=6, max_dr_iter=60, eps_dr=1e-5, eps_p=1e-7, eps_d=1e-7)
    g = gpu_solve(shape, batch, nrto.NRTO_DR, **kw)
    for i, (_, d) in enumerate(items):
        o = oracle_run(shape, d, nrto.NRTO_DR, **kw)
        assert_parity(g, o, i=i, engine=1)


def test_persistent_dr_zero_dr_iterations():
    """max_dr_iter = 0: the loop runs no pass; the solve still matches the oracle."""
    shape, data = CASES["c1"]()
    kw = dict(max_admm_iter=2, max_dr_iter=0, fixed_iters=1)
    g = gpu_solve(shape, single(shape, data), nrto.NRTO_DR, **kw)
    o = oracle_run(shape, data, nrto.NRTO_DR, **kw)
    assert_parity(g, o, engine=1)


@pytest.mark.parametrize("case,eng", [("c1", 0), ("c3s", 0), ("c2", 0), ("c2", 1)])
def test_scan_qp_matches_sequential_recurrences(case, eng):
    """The chunked-scan QP against the sequential-recurrence QP kernels (staged /
    pipelined sparse) on the same solves: reassociated sums only."""
    a = _run_child(case, eng, NRTO_QP_SCAN=1)
    b = _run_child(case, eng, NRTO_QP_SCAN=0)
    for sa, sb in zip(a, b):
        for k in sa:
            assert close(np.array(sa[k]), np.array(sb[k]), tol=1e-10), (case, eng, k)


def test_scan_qp_long_horizon_chunks():
    """T = 200 (chunks of 15 steps, 14 chunks) and T = 7 (chunks of 3): the scan
    QP inside FullADMM matches the oracle."""
    from gen.problems import make_quad
    for T in (7, 200):
        shape, data = make_quad(4, 1, T=T, n_obs=3)
        g = gpu_solve(shape, single(shape, data), nrto.NRTO_FULLADMM, max_iter=6, fixed_iters=1)
        o = oracle_run(shape, data, nrto.NRTO_FULLADMM, max_iter=6, fixed_iters=1)
        assert_parity(g, o)


@pytest.mark.parametrize("case", ["c1"])
def test_small_instance_megakernel_matches_launch_per_phase(case):
    """The whole-loop FullADMM kernel for small instances (k_fa_small, one CTA per
    instance) against the four-launches-per-iteration path on the same solves."""
    a = _run_child(case, 0, NRTO_FA_SMALL=1)
    b = _run_child(case, 0, NRTO_FA_SMALL=0)
    for sa, sb in zip(a, b):
        for k in sa:
            assert close(np.array(sa[k]), np.array(sb[k]), tol=1e-11), (case, k)


def test_small_instance_megakernel_termination_and_trace():
    """Per-instance termination inside the whole-loop kernel: a batch of unicycles
    stops each instance at the oracle's iteration, with the residual trace."""
    items = [make_unicycle(1, i) for i in range(5)]
    shape, batch = stack_instances(items)
    kw = dict(max_iter=200, eps_p=1e-4, eps_d=1e-4, check_every=3)
    g = gpu_solve(shape, batch, nrto.NRTO_FULLADMM, **kw)
    for i, (_, d) in enumerate(items):
        o = oracle_run(shape, d, nrto.NRTO_FULLADMM, **kw)
        assert int(g["iters"][i]) == int(o["iters"]), i
        assert_parity(g, o, i=i)


@pytest.mark.parametrize("case,eng", [("c1", 0), ("c3s", 0), ("c2", 1)])
def test_grid_qp_matches_one_cta_qp(case, eng):
    """The grid-wide QP (k_qp_grid, forced with NRTO_QP_GRID=1 on small single
    instances) against the one-CTA chunked-scan QP on the same solves."""
    a = _run_child(case, eng, NRTO_QP_GRID=1, NRTO_FA_SMALL=0)
    b = _run_child(case, eng, NRTO_QP_GRID=0)
    for sa, sb in zip(a, b):
        for k in sa:
            assert close(np.array(sa[k]), np.array(sb[k]), tol=1e-10), (case, eng, k)


def test_grid_qp_large_instance_matches_oracle():
    """A single quadcopter with 18.5 k rows (T = 60, 300 obstacles) takes the
    grid-wide QP by default; FullADMM and NRTO-DR match the oracle."""
    from gen.problems import make_quad
    shape, data = make_quad(4, 2, T=60, n_obs=300)
    assert shape.n_g >= 16384
    for eng, kw in ((nrto.NRTO_FULLADMM, dict(max_iter=3, fixed_iters=1)),
                    (nrto.NRTO_DR, dict(max_admm_iter=2, max_dr_iter=2, fixed_iters=1))):
        g = gpu_solve(shape, single(shape, data), eng, **kw)
        o = oracle_run(shape, data, eng, **kw)
        assert_parity(g, o, engine=eng)


def test_torch_caching_allocator_backs_the_workspace():
    """nrto_set_allocator with torch's caching allocator: the handle's workspace is
    torch memory while the handle lives, results equal the cudaMalloc handle's."""
    shape, data = CASES["c3s"]()
    kw = dict(max_iter=6, fixed_iters=1)
    ref = gpu_solve(shape, single(shape, data), nrto.NRTO_FULLADMM, **kw)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    nrto.use_torch_allocator(True)
    try:
        s = nrto.InnerSolver(shape, nrto.to_tensors(single(shape, data), device="cuda"), **kw)
        held = torch.cuda.memory_allocated() - before
        out = s.solve(nrto.NRTO_FULLADMM)
        torch.cuda.synchronize()
        g = {k: v.cpu().numpy() for k, v in out.items()}
        del out
        s.close()
    finally:
        nrto.use_torch_allocator(False)
    assert held > 1_000_000, held                       # workspace came from torch
    for k in ("kv", "du", "p", "p_tilde", "lam_p", "objective"):   # atomics: last-bit order only
        assert close(g[k], ref[k], tol=1e-12), k


def test_cone_sharded_dr_two_ranks_in_lockstep():
    """Cone sharding of one instance (NEXT-3(i), nrto_shard_cones / nrto_dr_step):
    two handles on this GPU own the two halves of the cones and exchange the
    adjoint (sum) after every pass and pi before every QP, exactly the ranks'
    protocol; their replicated outputs equal the unsharded solve and the oracle."""
    from paper_2603_02642_b200 import dist as nd
    shape, data = CASES["c2"]()
    kw = dict(max_admm_iter=3, max_dr_iter=6, fixed_iters=1)
    ref = gpu_solve(shape, single(shape, data), nrto.NRTO_DR, **kw)
    t = nrto.to_tensors(single(shape, data), device="cuda")
    ranks = [nd.cone_range(r, 2, shape) for r in range(2)]
    sol = [nrto.InnerSolver(shape, t, **kw) for _ in range(2)]
    for s, (lo, hi) in zip(sol, ranks):
        nrto.nrto_shard_cones(s.handle, lo, hi)
    Z = [nrto.nrto_buffer(s.handle, 0) for s in sol]
    pi = [nrto.nrto_buffer(s.handle, 1) for s in sol]
    for s in sol:
        nrto.nrto_solve_begin(s.handle, nrto.NRTO_DR)

    def allreduce(bufs):
        tot = bufs[0] + bufs[1]
        for b in bufs:
            b.copy_(tot)

    for l in range(1, kw["max_admm_iter"] + 1):
        for s in sol:
            nrto.nrto_dr_step(s.handle, 0, l)
        for _ in range(kw["max_dr_iter"]):
            for s in sol:
                nrto.nrto_dr_step(s.handle, 1, l)
                nrto.nrto_dr_step(s.handle, 2, l)
            allreduce(Z)
        for p, (lo, hi) in zip(pi, ranks):
            p[:lo] = 0.0
            p[hi:] = 0.0
        allreduce(pi)
        for s in sol:
            nrto.nrto_dr_step(s.handle, 3, l)
    outs = []
    for s in sol:
        o = nrto.alloc_out(shape, 1, s.E, device="cuda")
        nrto.nrto_solve_end(s.handle, o)
        torch.cuda.synchronize()
        outs.append({k: v.cpu().numpy() for k, v in o.items()})
    o_ref = oracle_run(shape, data, nrto.NRTO_DR, **kw)
    for g in outs:
        for k in ("kv", "du", "p", "p_tilde", "lam_p"):
            assert close(g[k], ref[k], tol=1e-10), k
        assert close(g["kv"][0], o_ref["kv"], tol=1e-9)
    with pytest.raises(nrto.NrtoError):
        sol[0].solve(nrto.NRTO_DR)               # inner_solve refuses a sharded handle
    for s in sol:
        s.close()


def test_cone_sharded_dr_one_rank_equals_unsharded():
    """world = 1 through the sharded driver (no collectives) equals the plain solve."""
    from paper_2603_02642_b200 import dist as nd
    shape, data = CASES["c2"]()
    kw = dict(max_admm_iter=2, max_dr_iter=5, fixed_iters=1)
    ref = gpu_solve(shape, single(shape, data), nrto.NRTO_DR, **kw)
    s = nrto.InnerSolver(shape, nrto.to_tensors(single(shape, data), device="cuda"), **kw)
    o = nd.sharded_dr_solve(s, 0, shape.n_g, None)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in o.items()}
    for k in ("kv", "du", "p", "p_tilde", "lam_p", "objective"):
        assert close(g[k], ref[k], tol=1e-10), k
    s.close()
