"""oracle.structured (ragged, per-timestep) == oracle.dense (literal matrices).

The structured tier is what the GPU parity tests compare against at c1-c3
sizes; here it is pinned iterate-by-iterate to the dense tier, which is in
turn pinned by test_oracle_construction / test_oracle_admm.
"""
import numpy as np
import pytest

from oracle import dense
from oracle import structured as st
from oracle.params import make_params
from tests.helpers import tiny, relerr, ragged_from_dense

CASES = [("uni", 4, 0), ("quad", 2, 1), ("franka", 2, 2)]


@pytest.mark.parametrize("kind,T,seed", CASES)
def test_setup_and_maps(kind, T, seed):
    shape, data = tiny(kind, T=T, seed=seed)
    pb = dense.DenseProblem(shape, data)
    sp = st.StructuredProblem(shape, data)
    np.testing.assert_allclose(sp.bhat_flat(), ragged_from_dense(shape, pb.nx, pb.bhat), atol=1e-15)
    rng = np.random.default_rng(seed)
    kv = rng.standard_normal(pb.NK)
    full = np.stack([pb.Ahat[j] @ kv + pb.bhat[j] for j in range(pb.ng)])
    np.testing.assert_allclose(sp.fwd(kv), ragged_from_dense(shape, pb.nx, full), atol=1e-14)
    # zero tails: nothing outside the ragged support
    mask = np.zeros_like(full, bool)
    for j in range(pb.ng):
        k = shape.cone_knot[j]
        if shape.cone_kind[j] == 0:
            mask[j, :(k + 1) * pb.nx] = True
        else:
            mask[j, k * pb.nx:(k + 1) * pb.nx] = True
    assert np.all(full[~mask] == 0)
    e = rng.standard_normal(sp.E)
    ed = np.zeros((pb.ng, pb.NX)); ed[mask] = 0
    for j in range(pb.ng):
        sl = e[sp.off[j]:sp.off[j + 1]]
        k = shape.cone_knot[j]
        if shape.cone_kind[j] == 0:
            ed[j, :len(sl)] = sl
        else:
            ed[j, k * pb.nx:(k + 1) * pb.nx] = sl
    np.testing.assert_allclose(sp.adj(e), sum(pb.Ahat[j].T @ ed[j] for j in range(pb.ng)), atol=1e-13)
    H = sp.gram_blocks(10.0, 0.5)
    Hd = pb.Qv + 0.5 * np.eye(pb.NK) + 10.0 * sum(pb.Ahat[j].T @ pb.Ahat[j] for j in range(pb.ng))
    n = shape.n_u * shape.n_x
    for k in range(T):
        np.testing.assert_allclose(H[k], Hd[k * n:(k + 1) * n, k * n:(k + 1) * n], rtol=1e-12, atol=1e-14)
    off = Hd.copy()
    for k in range(T):
        off[k * n:(k + 1) * n, k * n:(k + 1) * n] = 0
    assert np.abs(off).max() <= 1e-15 * np.abs(Hd).max()       # block diagonal


@pytest.mark.parametrize("kind,T,seed", CASES)
def test_riccati_qp_equals_dense_qp(kind, T, seed):
    shape, data = tiny(kind, T=T, seed=seed, r_trust=0.3)
    pb = dense.DenseProblem(shape, data)
    sp = st.StructuredProblem(shape, data)
    qd = dense.DenseQP(pb, 10.0, 1.0, 1e-6, 1.6)
    qs = st.RiccatiQP(sp, 10.0, 1.0, 1e-6, 1.6)
    rng = np.random.default_rng(seed)
    for call in range(4):
        v = rng.uniform(-0.2, 0.5, pb.ng)
        a = qd.solve(v, 7)
        b = qs.solve(v, 7)
        assert relerr(b[0], a[0]) < 1e-11 and relerr(b[1], a[1]) < 1e-11


@pytest.mark.parametrize("kind,T,seed", CASES)
def test_fulladmm_iterates(kind, T, seed):
    shape, data = tiny(kind, T=T, seed=seed, r_trust=0.3)
    pb = dense.DenseProblem(shape, data)
    sp = st.StructuredProblem(shape, data)
    prm = make_params(max_iter=12, fixed_iters=1)
    td, ts = [], []
    rd = dense.fulladmm(pb, prm, trace=td)
    rs = st.fulladmm(sp, prm, trace=ts)
    for a, b in zip(td, ts):
        for key in ("kv", "pt", "p", "du", "lam_p"):
            # lam_p accumulates p - p~ (cancellation): scale by ||p|| as well
            den = np.linalg.norm(a[key]) + (np.linalg.norm(a["p"]) if key == "lam_p" else 0)
            assert np.linalg.norm(b[key] - a[key]) <= 1e-10 * den + 1e-14, key
        nu_r = ragged_from_dense(shape, pb.nx, a["nu"])
        assert relerr(b["nu"], nu_r) < 1e-10
        # lam_nu accumulates a(k) - nu (cancellation): floor at ||nu||
        lam_r = ragged_from_dense(shape, pb.nx, a["lam_nu"])
        assert np.linalg.norm(b["lam_nu"] - lam_r) <= 1e-10 * (np.linalg.norm(lam_r) + np.linalg.norm(nu_r))
    for key in ("objective", "r_p", "r_d"):
        assert rs[key] == pytest.approx(rd[key], rel=1e-9, abs=1e-14)
    np.testing.assert_allclose(rs["margin_cone"], rd["margin_cone"], atol=1e-10)
    np.testing.assert_allclose(rs["margin_lin"], rd["margin_lin"], atol=1e-10)


@pytest.mark.parametrize("kind,T,seed", CASES[:2])
def test_dr_engine_iterates(kind, T, seed):
    shape, data = tiny(kind, T=T, seed=seed, r_trust=0.3)
    pb = dense.DenseProblem(shape, data)
    sp = st.StructuredProblem(shape, data)
    prm = make_params(max_admm_iter=4, max_dr_iter=9, fixed_iters=1)
    td, ts = [], []
    rd = dense.nrto_admm_dr(pb, prm, trace=td)
    rs = st.nrto_admm_dr(sp, prm, trace=ts)
    NX = pb.NX
    for a, b in zip(td, ts):
        for key in ("kv", "pt", "p", "du", "lam"):
            den = np.linalg.norm(a[key]) + (40 * np.linalg.norm(a["p"]) if key == "lam" else 0)
            assert np.linalg.norm(b[key] - a[key]) <= 1e-10 * den + 1e-14, key
        S = a["st"].reshape(pb.ng, 1 + NX)
        np.testing.assert_allclose(b["tt"], S[:, 0], atol=1e-11)
        assert relerr(b["et"], ragged_from_dense(shape, pb.nx, S[:, 1:])) < 1e-10
        assert b["r_dr"] == pytest.approx(a.get("r_dr", b["r_dr"]), rel=1e-9)
    assert rs["objective"] == pytest.approx(rd["objective"], rel=1e-9)


def test_early_termination_same_iteration():
    shape, data = tiny("uni", T=4, seed=3, r_trust=0.3)
    pb = dense.DenseProblem(shape, data)
    sp = st.StructuredProblem(shape, data)
    prm = make_params(max_iter=400, eps_p=1e-4, eps_d=1e-4)
    rd = dense.fulladmm(pb, prm)
    rs = st.fulladmm(sp, prm)
    assert rd["status"] == rs["status"] and rd["iters"] == rs["iters"]
