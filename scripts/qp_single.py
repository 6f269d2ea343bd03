import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_instance, stack_instances
shape, data = make_instance("c3")
_, b = stack_instances([(shape, data)])
s = nrto.InnerSolver(shape, nrto.to_tensors(b), max_iter=3, fixed_iters=1)
out = nrto.alloc_out(shape, 1, s.E, full=False)
for _ in range(2): s.solve(nrto.NRTO_FULLADMM, out=out)
torch.cuda.synchronize()
