"""Pins of the oracle with a GENERAL uncertainty set:
zeta = Gamma z, z^T S z <= tau with Gamma in R^{(T+1) n_x x n_z} (n_z < (T+1) n_x)
and a dense S, so A_hat_j = sqrt(tau) Psi Gamma^T [A_bar_j; 0] and
b_hat_j = sqrt(tau) Psi Gamma^T F_zeta^T grad g_j couple every time
block (no F1/F2 structure).

* support function: simulating the linearised closed loop with
  zeta = Gamma z gives the uncertain part c_j^T Gamma z; its worst case over the
  ellipsoid is sqrt(tau (Gamma^T c_j)^T S^-1 (Gamma^T c_j)) = ||A_hat_j k_v + b_hat_j||;
* FullADMM: the stationarity invariant at every iteration and the
  brute-force interior-point optimum of Problem 2 at convergence;
* NRTO-ADMM + DR reaches the same optimum (cross-engine).
"""
import numpy as np
import pytest

from oracle import dense, ip
from oracle.params import make_params
from tests.helpers import tiny, make_feasible, relerr
from tests.test_oracle_construction import _closed_loop_c


def general_set(shape, nz, seed):
    """A random full-rank Gamma ((T+1) n_x x n_z) and a dense SPD S (n_z x n_z)."""
    rng = np.random.default_rng(seed)
    NX = (shape.T + 1) * shape.n_x
    Gamma = rng.standard_normal((NX, nz)) / np.sqrt(nz)
    Q, _ = np.linalg.qr(rng.standard_normal((nz, nz)))
    S = (Q * rng.uniform(0.5, 4.0, nz)) @ Q.T * 1e2      # scale: ||zeta|| ~ sqrt(tau) / 10
    return Gamma, S


def general_instance(kind="uni", T=3, nz=7, seed=0, r_trust=0.15):
    shape, data = tiny(kind, T=T, seed=seed, r_trust=r_trust)
    Gamma, S = general_set(shape, nz, seed)
    pb = dense.DenseProblem(shape, data, S=S, Gamma=Gamma)
    data = make_feasible(pb, data, np.random.default_rng(seed), lo=0.002, hi=0.05)
    return shape, data, Gamma, S, dense.DenseProblem(shape, data, S=S, Gamma=Gamma)


@pytest.mark.parametrize("kind,T,nz", [("uni", 3, 7), ("uni", 4, 15), ("quad", 2, 20)])
def test_general_support_function_identity(kind, T, nz):
    shape, data = tiny(kind, T=T)
    Gamma, S = general_set(shape, nz, 3)
    pb = dense.DenseProblem(shape, data, S=S, Gamma=Gamma)
    assert pb.Ahat.shape[1] == nz and pb.bhat.shape[1] == nz
    Sinv = np.linalg.inv(S)
    rng = np.random.default_rng(4)
    for trial in range(3):
        kv = rng.standard_normal(pb.NK) * (0 if trial == 0 else 0.7)
        C = _closed_loop_c(shape, data, kv)
        for j in range(pb.ng):
            g = Gamma.T @ C[j]
            worst = np.sqrt(pb.tau * g @ Sinv @ g)
            soc = np.linalg.norm(pb.Ahat[j] @ kv + pb.bhat[j])
            assert soc == pytest.approx(worst, rel=1e-10, abs=1e-14)


def test_general_stationarity_invariant():
    shape, data, Gamma, S, pb = general_instance()
    tr = []
    dense.fulladmm(pb, make_params(max_iter=25, fixed_iters=1), trace=tr)
    for rec in tr:
        kv, lam = rec["kv"], rec["lam_nu"]
        stat = 10.0 * sum(pb.Ahat[j].T @ lam[j] for j in range(pb.ng)) + pb.Qv @ kv
        assert np.linalg.norm(stat) <= 1e-10 * (1 + np.linalg.norm(pb.Qv @ kv))


@pytest.mark.parametrize("seed", [0, 1])
def test_general_fulladmm_and_dr_vs_ip(seed):
    shape, data, Gamma, S, pb = general_instance(seed=seed)
    sol = ip.solve_problem2(pb)
    r = dense.fulladmm(pb, make_params(max_iter=2500, fixed_iters=1, qp_iters=20))
    assert r["objective"] == pytest.approx(sol["objective"], rel=1e-7)
    assert relerr(r["kv"], sol["kv"]) < 1e-5 and relerr(r["du"], sol["du"]) < 1e-5
    rd = dense.nrto_admm_dr(pb, make_params(max_admm_iter=400, max_dr_iter=40, fixed_iters=1,
                                            qp_iters=20))
    assert rd["objective"] == pytest.approx(sol["objective"], rel=1e-7)
