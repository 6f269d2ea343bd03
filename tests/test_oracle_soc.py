"""Pins for oracle.soc: SM Eq.(18) against the worked examples,
brute force and the algebraic invariants of a Euclidean cone projection."""
import numpy as np
import pytest

from oracle.soc import proj_soc, proj_soc_scale
from tests.helpers import golden


def test_worked_examples():
    g = golden("spec_examples.json")["soc_projection"]
    for c in g["cases"]:
        t, y = proj_soc(c["t"], np.array(c["y"]))
        assert t == pytest.approx(c["t_out"], abs=1e-15)
        np.testing.assert_allclose(y, c["y_out"], atol=1e-15)
        _, _, case = proj_soc_scale(np.array([c["t"]]), np.array([np.linalg.norm(c["y"])]))
        assert case[0] == c["case"]


def _brute(t0, y0):
    """argmin ||(t,y)-(t0,y0)||^2 s.t. t - ||y|| >= 0 by a generic NLP solver.

    scipy SLSQP on the convex program (concave constraint t - ||y|| >= 0),
    started inside the cone -- independent of the closed form (no case logic)."""
    from scipy.optimize import minimize
    x0 = np.concatenate([[abs(t0) + np.linalg.norm(y0) + 1.0], y0])
    v = np.concatenate([[t0], y0])
    def jac(x):
        ny = np.linalg.norm(x[1:])
        return np.concatenate([[1.0], -x[1:] / max(ny, 1e-300)])
    cons = [dict(type="ineq", fun=lambda x: x[0] - np.linalg.norm(x[1:]), jac=jac)]
    r = minimize(lambda x: 0.5 * (x - v) @ (x - v), x0, jac=lambda x: x - v,
                 constraints=cons, method="SLSQP", options=dict(ftol=1e-15, maxiter=500))
    return r.x[0], r.x[1:]


def test_against_brute_force():
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = rng.integers(1, 9)
        y0 = rng.standard_normal(n) * rng.uniform(0.1, 10)
        t0 = rng.standard_normal() * rng.uniform(0.1, 10)
        t, y = proj_soc(t0, y0)
        tb, yb = _brute(t0, y0)
        d = np.hypot(t - t0, np.linalg.norm(y - y0))
        db = np.hypot(tb - t0, np.linalg.norm(yb - y0))
        assert d <= db + 1e-6 * (1 + db)          # closed form is at least as close (SLSQP tol)
        assert abs(t - tb) <= 1e-5 * (1 + abs(tb))
        np.testing.assert_allclose(y, yb, atol=1e-5 * (1 + np.linalg.norm(yb)))


def test_invariants():
    rng = np.random.default_rng(11)
    for _ in range(3000):
        n = rng.integers(1, 16)
        v = (rng.standard_normal(), rng.standard_normal(n))
        w = (rng.standard_normal(), rng.standard_normal(n))
        pt, py = proj_soc(*v)
        assert np.linalg.norm(py) <= pt + 1e-12                       # membership
        qt, qy = proj_soc(pt, py)
        assert qt == pytest.approx(pt, abs=1e-12) and np.allclose(qy, py, atol=1e-12)  # idempotence
        nt, ny = proj_soc(-v[0], -v[1])                               # Moreau (self-dual K)
        assert pt - nt == pytest.approx(v[0], abs=1e-12)
        np.testing.assert_allclose(py - ny, v[1], atol=1e-12)
        rt, ry = v[0] - pt, v[1] - py                                 # polar orthogonality
        assert abs(rt * pt + ry @ py) <= 1e-10 * (1 + v[0] ** 2 + v[1] @ v[1])
        assert np.linalg.norm(ry) <= -rt + 1e-12                      # v - Pi(v) in the polar cone
        wt, wy = proj_soc(*w)                                         # non-expansive
        d1 = np.hypot(pt - wt, np.linalg.norm(py - wy))
        d0 = np.hypot(v[0] - w[0], np.linalg.norm(v[1] - w[1]))
        assert d1 <= d0 + 1e-12


def test_vectorised_matches_scalar():
    rng = np.random.default_rng(3)
    t = rng.standard_normal(500) * 3
    Y = rng.standard_normal((500, 5))
    Y[:20] = 0.0
    tp, s, case = proj_soc_scale(t, np.linalg.norm(Y, axis=1))
    for i in range(500):
        a, b = proj_soc(t[i], Y[i])
        assert tp[i] == pytest.approx(a, rel=1e-14, abs=1e-300)
        np.testing.assert_allclose(s[i] * Y[i], b, rtol=1e-14, atol=1e-300)
