"""One NRTO-DR solve of c2 (for launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_instance
from gen.problems import stack_instances
shp, d = make_instance("c2")
dd = nrto.to_tensors(stack_instances([(shp, d)])[1], device="cuda")
La = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s = nrto.InnerSolver(shp, dd, fixed_iters=1, max_admm_iter=La)
o = nrto.alloc_out(shp, 1, s.E, device="cuda", full=False)
s.solve(nrto.NRTO_DR, out=o); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); s.solve(nrto.NRTO_DR, out=o); e1.record(); torch.cuda.synchronize()
print("DR solve ms", e0.elapsed_time(e1), "per DR iteration us", 1000 * e0.elapsed_time(e1) / (La * 100))
