"""Reproduce tests/test_gpu_general.py::test_general_c1_fixed[1] step by step with
tracebacks dumped if it stalls."""
import faulthandler, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(45, repeat=True)
import numpy as np, torch
from gen import make_instance, stack_instances
from tests.test_oracle_general import general_set
from paper_2603_02642_b200 import nrto
shape, data = make_instance("c1")
t0 = time.time()
Gamma, S = general_set(shape, 30, 11)
print("general_set", time.time() - t0, flush=True)
_, batch = stack_instances([(shape, data)])
dd = nrto.to_tensors(batch, device="cuda")
G = torch.tensor(np.stack([Gamma]), dtype=torch.float64, device="cuda")
P = torch.tensor(np.stack([np.linalg.cholesky(np.linalg.inv(S)).T]), dtype=torch.float64, device="cuda")
print("tensors", time.time() - t0, flush=True)
s = nrto.InnerSolver(shape, dd, Gamma=G, Psi=P, max_iter=1, fixed_iters=1)
torch.cuda.synchronize(); print("setup", time.time() - t0, flush=True)
out = s.solve(nrto.NRTO_FULLADMM)
torch.cuda.synchronize(); print("solve", time.time() - t0, flush=True)
from oracle import dense
from oracle.params import make_params
pb = dense.DenseProblem(shape, data, S=S, Gamma=Gamma)
print("dense problem", time.time() - t0, flush=True)
o = dense.fulladmm(pb, make_params(max_iter=1, fixed_iters=1))
print("oracle", time.time() - t0, flush=True)
print("kv err", np.abs(out["kv"].cpu().numpy()[0] - o["kv"]).max())
