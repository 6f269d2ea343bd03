"""Debug of the general-set path: compare its internal arrays (W, b_hat, Cholesky
factor, ragged costates / b rows) with the dense oracle's quantities."""
import ctypes as C, faulthandler, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(60, repeat=True)
import numpy as np, torch
from gen import make_instance, stack_instances
from tests.test_oracle_general import general_set
from paper_2603_02642_b200 import nrto
from oracle import dense
from oracle.params import make_params
shape, data = make_instance("c1")
Gamma, S = general_set(shape, 30, 11)
_, batch = stack_instances([(shape, data)])
dd = nrto.to_tensors(batch, device="cuda")
G = torch.tensor(np.stack([Gamma]), dtype=torch.float64, device="cuda")
Psi = np.linalg.cholesky(np.linalg.inv(S)).T
P = torch.tensor(np.stack([Psi]), dtype=torch.float64, device="cuda")
s = nrto.InnerSolver(shape, dd, Gamma=G, Psi=P, max_iter=1, fixed_iters=1)
out = s.solve(nrto.NRTO_FULLADMM)
torch.cuda.synchronize()
pb = dense.DenseProblem(shape, data, S=S, Gamma=Gamma)
o = dense.fulladmm(pb, make_params(max_iter=1, fixed_iters=1))
print("kv err", np.abs(out["kv"].cpu().numpy()[0] - o["kv"]).max(), "kv max", np.abs(o["kv"]).max())
L = nrto.lib()
L.nrto_debug_gen_copy.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
nx, nu, T, ng, nz = pb.nx, pb.nu, pb.T, pb.ng, pb.nz
NX, NK = pb.NX, pb.NK
def get(which, shp):
    a = np.zeros(shp)
    r = L.nrto_debug_gen_copy(s.handle, which, a.ctypes.data, a.size)
    assert r == 0, r
    return a
tau = float(data["tau"])
W = np.sqrt(tau) * Psi @ Gamma.T
Wg = get(0, (nz, NX)); print("W err", np.abs(Wg - W).max(), np.abs(W).max())
Bh = get(1, (ng, nz)); print("bhat err", np.abs(Bh - pb.bhat).max(), np.abs(pb.bhat).max())
Lg = np.tril(get(2, (NK, NK)))
Minv = pb.Qv + 10.0 * sum(pb.Ahat[j].T @ pb.Ahat[j] for j in range(ng))
print("LL^T err", np.abs(Lg @ Lg.T - Minv).max(), np.abs(Minv).max())
E = s.E // nz * 0
print("nu err", np.abs(out["nu"].cpu().numpy()[0].reshape(ng, -1) - o["nu"]).max(), np.abs(o["nu"]).max())
print("pt err", np.abs(out["p_tilde"].cpu().numpy()[0] - o["p_tilde"]).max())
