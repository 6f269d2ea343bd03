"""GPU parity of the general-uncertainty-set path (nrto_setup_general, SURVEY §8f
NEXT-4: zeta = Gamma z, dense S) against the dense oracle
(oracle.dense.DenseProblem with the same Gamma, S; its pins are in
tests/test_oracle_general.py): iterates normwise and element-wise at fixed
iteration counts, termination, and the interior-point optimum of Problem 2."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen import make_instance, stack_instances
from gen.problems import make_quad, make_unicycle
from oracle import dense, ip
from oracle.params import make_params
from tests.helpers import close, elementwise, relerr
from tests.test_oracle_general import general_set, general_instance

from paper_2603_02642_b200 import nrto
from tests.test_gpu_parity import _require_gpu


def _psi(S):
    return np.linalg.cholesky(np.linalg.inv(S)).T          # upper, Psi^T Psi = S^-1


def gpu_general(shape, datas, Gammas, Ss, **pkw):
    _require_gpu()
    _, batch = stack_instances([(shape, d) for d in datas])
    dd = nrto.to_tensors(batch, device="cuda")
    G = torch.tensor(np.stack(Gammas), dtype=torch.float64, device="cuda")
    P = torch.tensor(np.stack([_psi(S) for S in Ss]), dtype=torch.float64, device="cuda")
    s = nrto.InnerSolver(shape, dd, Gamma=G, Psi=P, **pkw)
    out = s.solve(nrto.NRTO_FULLADMM)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    s.close()
    return res


def check(g, o, i=0, tol=1e-9):
    ng = len(o["p"])
    sc = np.linalg.norm(o["p"]) + np.linalg.norm(o["p_tilde"])
    for k in ("kv", "du"):
        assert close(g[k][i], o[k], tol=tol), k
    assert close(g["p"][i], o["p"], sc, tol=tol) and close(g["p_tilde"][i], o["p_tilde"], sc, tol=tol)
    assert close(g["lam_p"][i], o["lam_p"], sc, tol=tol)
    nu_g = g["nu"][i].reshape(ng, -1)
    assert close(nu_g, o["nu"], tol=tol), "nu"
    assert close(g["lam_nu"][i].reshape(ng, -1), o["lam_nu"], np.linalg.norm(o["nu"]), tol=tol), "lam_nu"
    assert elementwise(g["kv"][i], o["kv"]) <= 1e-8
    assert g["objective"][i] == pytest.approx(o["objective"], rel=1e-7, abs=1e-12)
    assert close(g["margin_cone"][i], o["margin_cone"], sc, tol=1e-7)


@pytest.mark.parametrize("L", [1, 5, 30])
def test_general_c1_fixed(L):
    shape, data = make_instance("c1")
    Gamma, S = general_set(shape, 30, 11)
    g = gpu_general(shape, [data], [Gamma], [S], max_iter=L, fixed_iters=1)
    pb = dense.DenseProblem(shape, data, S=S, Gamma=Gamma)
    o = dense.fulladmm(pb, make_params(max_iter=L, fixed_iters=1))
    check(g, o)


def test_general_batch_quad():
    items = [make_quad(2, i, T=6, n_obs=2) for i in range(3)]
    shape = items[0][0]
    sets = [general_set(shape, 40, 20 + i) for i in range(3)]
    g = gpu_general(shape, [d for _, d in items], [s[0] for s in sets], [s[1] for s in sets],
                    max_iter=12, fixed_iters=1)
    for i, (_, d) in enumerate(items):
        pb = dense.DenseProblem(shape, d, S=sets[i][1], Gamma=sets[i][0])
        check(g, dense.fulladmm(pb, make_params(max_iter=12, fixed_iters=1)), i=i)


def test_general_converges_to_ip_optimum():
    shape, data, Gamma, S, pb = general_instance(seed=0)
    kw = dict(max_iter=2500, fixed_iters=1, qp_iters=20)
    g = gpu_general(shape, [data], [Gamma], [S], **kw)
    sol = ip.solve_problem2(pb)
    assert g["objective"][0] == pytest.approx(sol["objective"], rel=1e-7)
    assert relerr(g["kv"][0], sol["kv"]) < 1e-5 and relerr(g["du"][0], sol["du"]) < 1e-5


def test_general_termination_matches_oracle():
    shape, data = make_unicycle(1, 3)
    Gamma, S = general_set(shape, 25, 5)
    kw = dict(max_iter=300, eps_p=1e-5, eps_d=1e-5, check_every=2)
    g = gpu_general(shape, [data], [Gamma], [S], **kw)
    o = dense.fulladmm(dense.DenseProblem(shape, data, S=S, Gamma=Gamma), make_params(**kw))
    assert int(g["iters"][0]) == o["iters"] and int(g["status"][0]) == o["status"]
    check(g, o)
