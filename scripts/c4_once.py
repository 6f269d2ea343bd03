"""One c4 quadcopter point solve (for launch lists).  usage: c4_once.py T n_obs engine [L]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen.problems import make_quad, stack_instances, CONFIGS
T, nobs, eng = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
L = int(sys.argv[4]) if len(sys.argv) > 4 else 2
shp, d = make_quad(CONFIGS["c4"], 0, T=T, n_obs=nobs)
dd = nrto.to_tensors(stack_instances([(shp, d)])[1], device="cuda")
kw = dict(max_iter=L) if eng == 0 else dict(max_admm_iter=1, max_dr_iter=L)
s = nrto.InnerSolver(shp, dd, fixed_iters=1, **kw)
o = nrto.alloc_out(shp, 1, s.E, device="cuda", full=False)
s.solve(eng, out=o); torch.cuda.synchronize()
print("ok")
