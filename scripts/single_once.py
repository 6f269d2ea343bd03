"""One fixed-iteration single-instance solve (for launch lists).
usage: single_once.py cfg engine(0 FullADMM, 1 DR) [L]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_instance
from gen.problems import stack_instances
cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
eng = int(sys.argv[2]) if len(sys.argv) > 2 else 0
L = int(sys.argv[3]) if len(sys.argv) > 3 else 4
shp, d = make_instance(cfg)
dd = nrto.to_tensors(stack_instances([(shp, d)])[1], device="cuda")
kw = dict(max_iter=L) if eng == 0 else dict(max_admm_iter=L)
s = nrto.InnerSolver(shp, dd, fixed_iters=1, **kw)
o = nrto.alloc_out(shp, 1, s.E, device="cuda", full=False)
s.solve(eng, out=o); torch.cuda.synchronize()
print("ok")
