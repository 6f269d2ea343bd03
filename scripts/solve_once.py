"""One FullADMM solve of the bench batch (for ncu launch lists).
usage: solve_once.py [B] [L] [qp_iters]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_batch
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
L = int(sys.argv[2]) if len(sys.argv) > 2 else 50
qpi = int(sys.argv[3]) if len(sys.argv) > 3 else 10
shape, batch = make_batch("c5", B)
dd = nrto.to_tensors(batch, device="cuda")
s = nrto.InnerSolver(shape, dd, max_iter=L, fixed_iters=1, qp_iters=qpi)
od = nrto.alloc_out(shape, B, s.E, device="cuda", full=False)
s.pass_bytes()
s.solve(nrto.NRTO_FULLADMM, out=od); torch.cuda.synchronize()
print("pass bytes per launch (avg):", s.pass_bytes() / L)
s.close()
