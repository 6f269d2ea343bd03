"""Pins for the inner-loop algorithms of oracle.dense / oracle.structured.

* gain operators: hand instances S:426-427
* stationarity invariant sum_j rho A_hat_j^T lam_nu_j + Q_v k_v = 0 at every
  iteration, and (14b) == argmin definition while it holds
* dual telescoping
* DR affine prox == KKT of P:936-943; s = b - A chi; fixed point
* (14a) QP: unconstrained closed form, r_trust = 0, generic NLP solution
* whole loop: brute-force barrier IP optimum of Problem 2 for
  FullADMM and for NRTO-ADMM+DR, cross-engine agreement
* linearised robust check: sampled disturbances never violate the
  linearised constraints beyond the residuals
"""
import numpy as np
import pytest

from oracle import dense, ip
from oracle import structured as st
from oracle.params import make_params
from tests.helpers import golden, tiny, make_feasible, relerr


def test_gain_operators_hand_instance():
    g = golden("spec_examples.json")["gain_update_hand"]
    n = 3
    Qv = g["Qv_scale"] * np.eye(n)
    bhat = np.array([3.0, -1.0, 2.0])
    M, q, calM, calMbar = dense.gain_operators(Qv, [np.eye(n)], [bhat], g["rho"])
    np.testing.assert_allclose(M, g["M_scale"] * np.eye(n), atol=1e-15)
    np.testing.assert_allclose(calM, g["calM_scale"] * np.eye(n), atol=1e-15)
    np.testing.assert_allclose(calMbar[0], g["calMbar_scale"] * np.eye(n), atol=1e-15)
    np.testing.assert_allclose(q, g["q_over_bhat"] * bhat, atol=1e-15)
    # b_hat = 0, nu = (1,0,..): k1 = k0/2 + nu/2
    k0 = np.array([0.4, -2.0, 1.0]); nu = np.array([1.0, 0.0, 0.0])
    M, q, calM, calMbar = dense.gain_operators(Qv, [np.eye(n)], [np.zeros(n)], g["rho"])
    np.testing.assert_allclose(q + calM @ k0 + calMbar[0] @ nu, 0.5 * k0 + 0.5 * nu, atol=1e-15)
    # no cones
    M, q, calM, calMbar = dense.gain_operators(Qv, [], [], 10.0)
    np.testing.assert_allclose(M, np.linalg.inv(Qv)); np.testing.assert_allclose(calM, np.eye(n))
    np.testing.assert_allclose(q, 0)


def _active_instance(kind="uni", T=3, seed=0, r_trust=0.15):
    shape, data = tiny(kind, T=T, seed=seed, r_trust=r_trust)
    pb = dense.DenseProblem(shape, data)
    data = make_feasible(pb, data, np.random.default_rng(seed), lo=0.002, hi=0.05)
    return shape, data, dense.DenseProblem(shape, data)


def test_stationarity_invariant_and_argmin():
    shape, data, pb = _active_instance()
    prm = make_params(max_iter=25, fixed_iters=1)
    tr = []
    dense.fulladmm(pb, prm, trace=tr)
    rho = prm["rho"]
    lam_prev = np.zeros((pb.ng, pb.NX))
    for rec in tr:
        kv, lam = rec["kv"], rec["lam_nu"]
        stat = rho * sum(pb.Ahat[j].T @ lam[j] for j in range(pb.ng)) + pb.Qv @ kv
        assert np.linalg.norm(stat) <= 1e-10 * (1 + np.linalg.norm(pb.Qv @ kv))
        # (14b) result == argmin_k sum rho/2||A_j k + b_j - nu_j + lam_j^{l-1}||^2 + 1/2 k^T Q_v k
        Hm = pb.Qv + rho * sum(pb.Ahat[j].T @ pb.Ahat[j] for j in range(pb.ng))
        rhs = -rho * sum(pb.Ahat[j].T @ (pb.bhat[j] - rec["nu"][j] + lam_prev[j]) for j in range(pb.ng))
        assert relerr(kv, np.linalg.solve(Hm, rhs)) < 1e-9
        lam_prev = lam


def test_dual_telescoping():
    shape, data, pb = _active_instance(seed=1)
    tr = []
    dense.fulladmm(pb, make_params(max_iter=8, fixed_iters=1), trace=tr)
    acc = np.zeros((pb.ng, pb.NX))
    for rec in tr:
        for j in range(pb.ng):
            acc[j] += pb.Ahat[j] @ rec["kv"] + pb.bhat[j] - rec["nu"][j]
        np.testing.assert_allclose(rec["lam_nu"], acc, atol=1e-12)


def test_dr_prox_is_kkt_minimiser():
    shape, data, pb = _active_instance(seed=2)
    dr = dense.DenseDR(pb, 40.0, 0.9, 1e-6, 1.0)
    rng = np.random.default_rng(0)
    dr.chit = rng.standard_normal(dr.chit.shape)
    dr.st = rng.standard_normal(dr.st.shape)
    qvec = np.concatenate([np.zeros(pb.NK), rng.standard_normal(pb.ng)])
    n = dr.P.shape[0]
    rhs = np.concatenate([dr.Rchi @ dr.chit - qvec, dr.bvec - dr.st])
    sol = np.linalg.solve(dr.Kkkt, rhs)
    chi, y = sol[:n], sol[n:]
    s = dr.st - np.linalg.solve(dr.Rs, y)
    np.testing.assert_allclose(s, dr.bvec - dr.A @ chi, atol=1e-10)       # s = b - A chi
    # independent: minimise 1/2 chi^T P chi + q^T chi + 1/2||chi-chi~||_Rchi^2 + 1/2||b-A chi-s~||_Rs^2
    Hm = dr.P + dr.Rchi + dr.A.T @ dr.Rs @ dr.A
    g = qvec - dr.Rchi @ dr.chit - dr.A.T @ dr.Rs @ (dr.bvec - dr.st)
    assert relerr(chi, np.linalg.solve(Hm, -g)) < 1e-9
    # S:343 2x2 instance
    K = golden("spec_examples.json")["dr_kkt_2x2"]["K_KKT"]
    np.testing.assert_array_equal(np.block([[np.zeros((1, 1)) + np.eye(1), np.eye(1)],
                                            [np.eye(1), -np.eye(1)]]), K)


def test_dr_fixed_point():
    shape, data, pb = _active_instance(seed=3)
    dr = dense.DenseDR(pb, 40.0, 0.9, 1e-6, 1.0)
    qvec = np.concatenate([np.zeros(pb.NK), -40.0 * np.full(pb.ng, 0.3)])
    dr.run(qvec, 4000, 0.0, True)
    st0 = dr.st.copy()
    _, _, r_dr, _ = dr.run(qvec, 1, 0.0, True)
    assert r_dr <= 1e-9 * (1 + np.linalg.norm(st0))


def test_qp_closed_forms():
    shape, data = tiny("uni", T=3, seed=4, r_trust=1e3)
    data = dict(data); data["g0"] = np.full(shape.n_g, -1e3)        # rows inactive
    pb = dense.DenseProblem(shape, data)
    qp = dense.DenseQP(pb, 10.0, 1.0, 1e-6, 1.6)
    v = np.random.default_rng(0).standard_normal(pb.ng)
    du, p = qp.solve(v, 3000)
    np.testing.assert_allclose(du, -pb.u_hat, atol=1e-8)            # argmin of Q_u alone
    np.testing.assert_allclose(p, v, atol=1e-8)
    data["r_trust"] = 0.0
    pb0 = dense.DenseProblem(shape, data)
    du, p = dense.DenseQP(pb0, 10.0, 1.0, 1e-6, 1.6).solve(v, 3000)
    assert np.linalg.norm(du) < 1e-7


def test_qp_against_nlp():
    from scipy.optimize import minimize
    shape, data, pb = _active_instance(seed=5, r_trust=0.1)
    rho = 10.0
    v = np.random.default_rng(2).uniform(0, 0.2, pb.ng)
    du, p = dense.DenseQP(pb, rho, 1.0, 1e-6, 1.6).solve(v, 6000)
    NU = pb.NU
    f = lambda x: (pb.u_hat + x[:NU]) @ pb.Ru @ (pb.u_hat + x[:NU]) + 0.5 * rho * np.sum((x[NU:] - v) ** 2)
    cons = [dict(type="ineq", fun=lambda x: -(pb.g0 + pb.b @ x[:NU] + x[NU:])),
            dict(type="ineq", fun=lambda x: pb.r_trust ** 2 - np.sum((pb.F_u @ x[:NU]) ** 2))]
    r = minimize(f, np.zeros(NU + pb.ng), constraints=cons, method="SLSQP",
                 options=dict(ftol=1e-15, maxiter=1000))
    assert f(np.concatenate([du, p])) == pytest.approx(r.fun, rel=1e-6, abs=1e-10)
    np.testing.assert_allclose(du, r.x[:NU], atol=1e-5)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_whole_loop_fulladmm_vs_ip(seed):
    shape, data, pb = _active_instance(seed=seed)
    sol = ip.solve_problem2(pb)
    sp = st.StructuredProblem(shape, data)
    r = st.fulladmm(sp, make_params(max_iter=2500, fixed_iters=1, qp_iters=20))
    assert r["objective"] == pytest.approx(sol["objective"], rel=1e-7)
    assert relerr(r["kv"], sol["kv"]) < 1e-5 and relerr(r["du"], sol["du"]) < 1e-5
    assert np.all(r["margin_cone"] >= -1e-7) and np.all(r["margin_lin"] >= -1e-7)


def test_whole_loop_dr_vs_ip_and_cross_engine():
    shape, data, pb = _active_instance(seed=1)
    sol = ip.solve_problem2(pb)
    sp = st.StructuredProblem(shape, data)
    rd = st.nrto_admm_dr(sp, make_params(max_admm_iter=400, max_dr_iter=40, fixed_iters=1,
                                         qp_iters=20))
    rf = st.fulladmm(sp, make_params(max_iter=2500, fixed_iters=1, qp_iters=20))
    assert rd["objective"] == pytest.approx(sol["objective"], rel=1e-7)
    assert relerr(rd["kv"], sol["kv"]) < 1e-5
    assert rd["objective"] == pytest.approx(rf["objective"], rel=1e-6)   # cross-engine


def test_linearised_robust_check():
    """Sampled zeta (1000 interior + 1000 edge) on the linearised model."""
    from tests.test_oracle_construction import _closed_loop_c
    shape, data, pb = _active_instance(seed=0)
    sp = st.StructuredProblem(shape, data)
    r = st.fulladmm(sp, make_params(max_iter=2500, fixed_iters=1, qp_iters=20))
    C = _closed_loop_c(shape, data, r["kv"])
    rng = np.random.default_rng(732)
    L = np.linalg.cholesky(np.linalg.inv(pb.S))
    W = rng.standard_normal((1000, pb.NX)); W /= np.linalg.norm(W, axis=1, keepdims=True)
    rad = rng.uniform(0, 1, (1000, 1)) ** (1.0 / pb.NX)
    Zi = np.sqrt(pb.tau) * (rad * W) @ L.T                      # interior, volumetric
    Sinv = np.linalg.inv(pb.S)
    Zs = np.stack([np.sqrt(pb.tau) * Sinv @ C[j] / np.sqrt(C[j] @ Sinv @ C[j])
                   for j in range(pb.ng) if np.linalg.norm(C[j]) > 0])
    cw = rng.dirichlet(np.ones(len(Zs)), 1000)                  # convex combos of worst cases
    Ze = cw @ Zs
    Ze *= np.sqrt(pb.tau / np.einsum("ni,ij,nj->n", Ze, pb.S, Ze))[:, None]
    lin = pb.g0 + pb.b @ r["du"]
    for Z in (Zi, Ze):
        viol = lin[None, :] + Z @ C.T
        assert viol.max() <= r["r_p"] + 1e-9
