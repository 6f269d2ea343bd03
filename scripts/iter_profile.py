"""Per-class device time of the first L iterations (fixed_iters, bench batch) for
several L, to see where in the solve each kernel class spends its time (probe).
usage: iter_profile.py [B] [L,...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_batch
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
Ls = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,3,5,10,20,50").split(",")]
shape, batch = make_batch("c5", B)
dd = nrto.to_tensors(batch, device="cuda")
for L in Ls:
    s = nrto.InnerSolver(shape, dd, max_iter=L, fixed_iters=1)
    od = nrto.alloc_out(shape, B, s.E, device="cuda", full=False)
    s.solve(nrto.NRTO_FULLADMM, out=od); torch.cuda.synchronize()
    s.profile(True); s.profile_read()
    s.pass_bytes()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.solve(nrto.NRTO_FULLADMM, out=od)
    e1.record(); torch.cuda.synchronize()
    prof = s.profile_read()
    print(f"L {L}: solve {e0.elapsed_time(e1):.1f} ms; pass GB {s.pass_bytes() / 1e9:.2f};",
          ", ".join(f"{k} {v[0]:.2f}" for k, v in prof.items()), flush=True)
    s.close()
