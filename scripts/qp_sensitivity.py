"""Sensitivity of the overlapped FullADMM loop to the QP's share: solve time and
per-class device time for several qp_iters (a probe, not a bench number).
usage: qp_sensitivity.py [B] [L] [qp_iters,...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_batch
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
L = int(sys.argv[2]) if len(sys.argv) > 2 else 50
qps = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "10,5,1").split(",")]
shape, batch = make_batch("c5", B)
dd = nrto.to_tensors(batch, device="cuda")
for qpi in qps:
    s = nrto.InnerSolver(shape, dd, max_iter=L, fixed_iters=1, qp_iters=qpi)
    od = nrto.alloc_out(shape, B, s.E, device="cuda", full=False)
    s.solve(nrto.NRTO_FULLADMM, out=od); torch.cuda.synchronize()
    s.profile(True); s.profile_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.solve(nrto.NRTO_FULLADMM, out=od)
    e1.record(); torch.cuda.synchronize()
    prof = s.profile_read()
    print(f"qp_iters {qpi}: solve {e0.elapsed_time(e1):.1f} ms;",
          ", ".join(f"{k} {v[0]:.1f}" for k, v in prof.items()), flush=True)
    s.close()
