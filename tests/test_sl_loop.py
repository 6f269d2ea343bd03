"""Host SL outer loop + Monte-Carlo / edge validation (
P:182-239 Fig. 2, §V-A).

CPU tests inject the oracle as the inner solver (test infrastructure); the GPU
test runs the loop through libnrto.  Pins:
* interior samples lie in the ellipsoid, edge samples on its boundary, both
  deterministic under the seed; 1-D volumetric uniformity (KS test);
* robust_terms (the support function ||A_hat_j k_v + b_hat_j||) equals the
  first-order response of the NONLINEAR closed-loop rollout along the
  worst-case direction (finite difference) -- ties the host linearisation to the
  model, not to its own formula;
* accept_step: ratio 1 accepts and grows the radius, no reduction rejects and
  shrinks it, r_min floor;
* the loop: merit never increases over accepted steps, it converges, and the
  converged policy passes validation.
"""
import math

import numpy as np
import pytest

from paper_2603_02642_b200 import sl


def _scenario(T=12, obstacles=((1.2, 0.35, 0.25),)):
    return sl.UnicycleScenario(T=T, dt=0.15, goal=(2.0, 0.8), r_goal=0.3, obstacles=obstacles)


class OracleInner:
    """Inner solve by the CPU oracle (tests only)."""

    def __call__(self, sc, data, params):
        from gen.problems import Shape
        from oracle import structured as st
        from oracle.params import make_params
        knot, kind = sc.rows()
        shape = Shape(sc.n_x, sc.n_u, sc.T, knot, kind)
        r = st.fulladmm(st.StructuredProblem(shape, data), make_params(**params))
        return r


def test_interior_samples_inside_and_deterministic():
    sc = _scenario()
    Z = sl.sample_interior(sc, 500, seed=3)
    v = sl.ellipsoid_value(sc, Z)
    assert np.all(v <= sc.tau * (1 + 1e-12)) and v.max() > 0.5 * sc.tau
    np.testing.assert_array_equal(Z, sl.sample_interior(sc, 500, seed=3))


def test_interior_uniform_1d():
    from scipy.stats import kstest
    sc = sl.UnicycleScenario(T=0, sigma0=1.0, tau=1.0)
    sc.n_x = 1
    Z = sl.sample_interior(sc, 20000, seed=1)[:, 0]
    assert kstest(Z, "uniform", args=(-1.0, 2.0)).pvalue > 0.01


def test_edge_samples_on_boundary():
    sc = _scenario()
    u = np.tile([1.0, 0.2], (sc.T, 1))
    K = np.random.default_rng(0).standard_normal((sc.T, 2, 3)) * 0.3
    _, data = sl.linearize(sc, u, 1.0)
    Z = sl.sample_edge(sc, data, K, 300, seed=5)
    v = sl.ellipsoid_value(sc, Z)
    np.testing.assert_allclose(v, sc.tau, rtol=1e-9)


def test_support_function_matches_nonlinear_rollout():
    """d/d eps g_j(closed-loop x(eps zeta_j*)) at 0 = ||A_hat_j k_v + b_hat_j|| for
    every row j (P:841-869 with the closed-loop sensitivity; finite differences
    of the nonlinear model)."""
    sc = _scenario(obstacles=((1.0, 0.6, 0.3), (1.6, -0.2, 0.2)))
    rng = np.random.default_rng(2)
    u = np.column_stack([1.0 + 0.2 * rng.standard_normal(sc.T), 0.4 * rng.standard_normal(sc.T)])
    K = rng.standard_normal((sc.T, 2, 3)) * 0.5
    _, data = sl.linearize(sc, u, 1.0)
    rob, vecs = sl.robust_terms(sc, data, K)
    x0, ua0 = sl.closed_loop(sc, u, K, np.zeros((sc.T + 1) * 3))
    g_0, _ = sc.constraint_values(x0, ua0)
    eps = 1e-6
    for j in range(len(rob)):
        if rob[j] == 0.0:
            continue
        w = vecs[j].reshape(-1) / rob[j] * math.sqrt(sc.tau)
        z = sl._psiT(sc, w[None])[0]
        xp, up = sl.closed_loop(sc, u, K, eps * z)
        xm, um = sl.closed_loop(sc, u, K, -eps * z)
        gp, _ = sc.constraint_values(xp, up)
        gm, _ = sc.constraint_values(xm, um)
        fd = (gp[j] - gm[j]) / (2 * eps)
        assert fd == pytest.approx(rob[j], rel=1e-5, abs=1e-9), j


def test_accept_step_rules():
    s = sl.OuterSettings()
    ok, r, rho = sl.accept_step(1.0, 1.0, 1.0, 10.0, 0.0, s)
    assert ok and r == pytest.approx(1.15) and rho == 10.0
    ok, r, _ = sl.accept_step(-0.1, 1.0, 1.0, 10.0, 0.0, s)
    assert not ok and r == pytest.approx(0.8)
    ok, r, _ = sl.accept_step(-0.1, 1.0, s.r_min, 10.0, 0.0, s)
    assert not ok and r == s.r_min
    _, _, rho = sl.accept_step(1.0, 1.0, 1.0, 100.0, 1.0, s)
    assert rho == s.rho_max
    ok, r, _ = sl.accept_step(10.0, 10.0, 5.9, 10.0, 0.0, s)
    assert ok and r == pytest.approx(s.eta2 * s.r0)      # growth cap


def test_sl_loop_with_oracle_inner():
    sc = _scenario()
    res = sl.run_sl(sc, sl.OuterSettings(max_outer=60), inner=OracleInner())
    acc = [h["merit"] for h in res.history if h["accepted"]]
    assert all(b <= a + 1e-9 for a, b in zip(acc, acc[1:]))       # merit never increases
    assert res.status == "converged", res.history[-3:]
    x = sc.rollout(res.u)
    assert abs(x[-1, 0] - sc.goal[0]) <= sc.r_goal + 1e-6 and abs(x[-1, 1] - sc.goal[1]) <= sc.r_goal + 1e-6
    rep = sl.validate(sc, res.u, res.K, n_interior=200, n_edge=200, seed=0)
    assert rep["rate"] >= 0.9, rep


@pytest.mark.gpu
def test_sl_loop_gpu_inner_matches_oracle_inner():
    """The SL loop through libnrto takes the same accept/reject decisions and
    reaches the same policy as with the oracle inner solve; the policy passes
    the paper's validation (1000 interior + 1000 edge rollouts)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device")
    sc = sl.UnicycleScenario(T=30, obstacles=((1.2, 0.9, 0.3),))
    gi = sl.GpuInner()
    res_g = sl.run_sl(sc, inner=gi)
    gi.close()
    res_o = sl.run_sl(sc, inner=OracleInner())
    assert res_g.status == "converged" == res_o.status
    assert [h["accepted"] for h in res_g.history] == [h["accepted"] for h in res_o.history]
    np.testing.assert_allclose(res_g.u, res_o.u, rtol=0, atol=1e-7)
    np.testing.assert_allclose(res_g.K, res_o.K, rtol=0, atol=1e-7)
    rep = sl.validate(sc, res_g.u, res_g.K, seed=0)
    assert rep["rate"] >= 0.9, rep
