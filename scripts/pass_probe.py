"""Per-class device time of one FullADMM solve for different QP loads."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_batch
B = 512
shape, batch = make_batch("c5", B)
dd = nrto.to_tensors(batch, device="cuda")
for qpi in (10, 0):
    s = nrto.InnerSolver(shape, dd, max_iter=50, fixed_iters=1, qp_iters=qpi)
    od = nrto.alloc_out(shape, B, s.E, device="cuda", full=False)
    s.solve(nrto.NRTO_FULLADMM, out=od); torch.cuda.synchronize()
    s.profile(True); s.profile_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.pass_bytes()
    e0.record(); s.solve(nrto.NRTO_FULLADMM, out=od); e1.record(); torch.cuda.synchronize()
    p = s.profile_read()
    pb = s.pass_bytes()
    print(f"pass bytes/launch {pb/50/1e9:.2f} GB -> {pb/ (p['pass'][0]*1e-3) / 1e9:.0f} GB/s")
    print(f"qp_iters={qpi}: solve {e0.elapsed_time(e1):.1f} ms; " + ", ".join(f"{k} {v[0]:.1f}ms/{v[1]}" for k, v in p.items()))
    s.profile(False); s.close()
