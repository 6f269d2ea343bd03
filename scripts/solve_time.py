"""Device time of fixed-L FullADMM solves of the bench wave (probe).
usage: solve_time.py [B] [L]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_batch
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
L = int(sys.argv[2]) if len(sys.argv) > 2 else 50
shape, batch = make_batch("c5", B)
dd = nrto.to_tensors(batch, device="cuda")
s = nrto.InnerSolver(shape, dd, max_iter=L, fixed_iters=1)
od = nrto.alloc_out(shape, B, s.E, device="cuda", full=False)
for _ in range(2):
    s.solve(nrto.NRTO_FULLADMM, out=od)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    s.solve(nrto.NRTO_FULLADMM, out=od)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"solve B={B} L={L}: {ms:.1f} ms  ({ms / L:.2f} ms/iteration, {B * L / ms * 1000:.0f} inst-it/s)")
s.profile(True); s.profile_read()
s.solve(nrto.NRTO_FULLADMM, out=od); torch.cuda.synchronize()
print("  classes:", {k: round(v[0], 1) for k, v in s.profile_read().items()})
s.close()
