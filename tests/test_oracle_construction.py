"""Pins for the SOC data construction of SM §I in oracle.dense.

The strongest pin is the support-function identity: simulating the
linearised closed-loop system of P:115-144 (x_{k+1} = A x + B u + d,
u_k = K_k d_{k-1}) gives the uncertain part of constraint j as c_j^T zeta;
its worst case over {zeta : zeta^T S zeta <= tau} is sqrt(tau c^T S^-1 c),
which must equal ||A_hat_j k_v + b_hat_j|| (the SOC of Problem 2).  The
simulation uses none of the paper's formulas for A_hat, b_hat, Psi or vec.
"""
import numpy as np
import pytest

from oracle.dense import DenseProblem
from oracle.structured import vec_cm, unvec_cm
from tests.helpers import golden, tiny


def test_vec_and_kron_examples():
    g = golden("spec_examples.json")
    K = np.array(g["vec_column_major"]["K"], float)
    np.testing.assert_array_equal(vec_cm(K), g["vec_column_major"]["vec"])
    np.testing.assert_array_equal(unvec_cm(vec_cm(K), 2, 2), K)
    kb = g["kron_abar"]
    Abar = np.kron(np.eye(kb["n_x"]), np.array(kb["b"], float)[None, :])
    np.testing.assert_array_equal(Abar, kb["Abar"])
    rng = np.random.default_rng(0)
    for _ in range(20):          # K^T b = (I (x) b^T) vec(K)
        nu, nx = rng.integers(1, 6, 2)
        K = rng.standard_normal((nu, nx)); b = rng.standard_normal(nu)
        np.testing.assert_allclose(np.kron(np.eye(nx), b[None, :]) @ vec_cm(K), K.T @ b, atol=1e-13)


def test_sensitivities_T1():
    g = golden("spec_examples.json")["sensitivities_T1"]
    A0, B0 = np.array(g["A0"]), np.array(g["B0"])
    from gen.problems import Shape
    shape = Shape(2, 1, 1, np.array([1], np.int32), np.array([0], np.int8))
    data = dict(A=A0[None], B=B0[None], grad=np.array([[1.0, 0.0]]), g0=np.array([-1.0]),
                Psi=np.tile(np.eye(2), (2, 1, 1)), tau=1.0, W_K=np.ones((1, 1, 1)),
                R_u=np.ones((1, 1, 1)), u_hat=np.zeros((1, 1)), r_trust=1.0)
    pb = DenseProblem(shape, data)
    np.testing.assert_array_equal(pb.F_u, np.vstack([np.zeros((2, 1)), B0]))
    np.testing.assert_array_equal(pb.F_z, np.block([[np.eye(2), np.zeros((2, 2))], [A0, np.eye(2)]]))


def test_sqrt_tau_homogeneity():
    shape, data = tiny("uni", T=3)
    pb1 = DenseProblem(shape, data)
    d2 = dict(data); d2["tau"] = 4 * data["tau"]
    pb2 = DenseProblem(shape, d2)
    np.testing.assert_allclose(pb2.Ahat, 2 * pb1.Ahat, rtol=1e-14, atol=1e-300)
    np.testing.assert_allclose(pb2.bhat, 2 * pb1.bhat, rtol=1e-14, atol=1e-300)


def _closed_loop_c(shape, data, kv):
    """c_j with (uncertain part of row j) = c_j^T zeta, by linear simulation."""
    nx, nu, T = shape.n_x, shape.n_u, shape.T
    A, B = data["A"], data["B"]
    K = unvec_cm(kv.reshape(T, -1), nu, nx)
    NX = (T + 1) * nx
    C = np.zeros((shape.n_g, NX))
    for col in range(NX):
        zeta = np.zeros(NX); zeta[col] = 1.0
        d = zeta.reshape(T + 1, nx)            # d[0] = d_bar_0 = d_{-1}, d[k+1] = d_k
        x = np.zeros((T + 1, nx)); u = np.zeros((T, nu))
        x[0] = d[0]                            # x_0 = x_bar_0 + d_bar_0
        for k in range(T):
            u[k] = K[k] @ d[k]                 # u_k = K_k d_{k-1}
            x[k + 1] = A[k] @ x[k] + B[k] @ u[k] + d[k + 1]
        for j in range(shape.n_g):
            kj = shape.cone_knot[j]
            if shape.cone_kind[j] == 0:
                C[j, col] = data["grad"][j] @ x[kj]
            else:
                C[j, col] = data["grad"][j, :nu] @ u[kj]
    return C


@pytest.mark.parametrize("kind,T", [("uni", 3), ("quad", 2), ("franka", 2)])
def test_support_function_identity(kind, T):
    shape, data = tiny(kind, T=T)
    pb = DenseProblem(shape, data)
    rng = np.random.default_rng(5)
    S = pb.S
    Sinv = np.linalg.inv(S)
    for trial in range(3):
        kv = rng.standard_normal(pb.NK) * (0 if trial == 0 else 0.7)
        C = _closed_loop_c(shape, data, kv)
        for j in range(pb.ng):
            worst = np.sqrt(pb.tau * C[j] @ Sinv @ C[j])
            soc = np.linalg.norm(pb.Ahat[j] @ kv + pb.bhat[j])
            assert soc == pytest.approx(worst, rel=1e-10, abs=1e-14)


def test_support_function_sampling():
    """Boundary samples of the ellipsoid never exceed the SOC and approach it."""
    shape, data = tiny("uni", T=2)
    pb = DenseProblem(shape, data)
    rng = np.random.default_rng(9)
    kv = rng.standard_normal(pb.NK)
    C = _closed_loop_c(shape, data, kv)
    L = np.linalg.cholesky(np.linalg.inv(pb.S))      # zeta = sqrt(tau) L w, ||w|| = 1
    W = rng.standard_normal((200000, pb.NX))
    W /= np.linalg.norm(W, axis=1, keepdims=True)
    Z = np.sqrt(pb.tau) * W @ L.T
    assert np.allclose(np.einsum("ni,ij,nj->n", Z, pb.S, Z), pb.tau)
    for j in range(pb.ng):
        soc = np.linalg.norm(pb.Ahat[j] @ kv + pb.bhat[j])
        vals = Z @ C[j]
        assert vals.max() <= soc + 1e-9
        assert vals.max() >= 0.9 * soc


def test_Qv_definition():
    """1/2 k_v^T Q_v k_v = sum_k ||R_K^k K_k||_F^2."""
    shape, data = tiny("franka", T=2)
    rng = np.random.default_rng(1)
    RK = rng.standard_normal((shape.T, shape.n_u, shape.n_u))
    data = dict(data); data["W_K"] = np.einsum("kji,kjl->kil", RK, RK)
    pb = DenseProblem(shape, data)
    for _ in range(10):
        kv = rng.standard_normal(pb.NK)
        K = unvec_cm(kv.reshape(shape.T, -1), shape.n_u, shape.n_x)
        fro = sum(np.linalg.norm(RK[k] @ K[k]) ** 2 for k in range(shape.T))
        assert 0.5 * kv @ pb.Qv @ kv == pytest.approx(fro, rel=1e-12)
