"""Per-class device time of one NRTO-DR solve of c2 (bench's secondary line), probe.
usage: dr_profile.py [La]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_instance
from gen.problems import stack_instances
shp, d = make_instance("c2")
dd = nrto.to_tensors(stack_instances([(shp, d)])[1], device="cuda")
La = int(sys.argv[1]) if len(sys.argv) > 1 else 40
s = nrto.InnerSolver(shp, dd, fixed_iters=1, max_admm_iter=La)
o = nrto.alloc_out(shp, 1, s.E, device="cuda", full=False)
s.solve(nrto.NRTO_DR, out=o); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); s.solve(nrto.NRTO_DR, out=o); e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1)
s.profile(True); s.profile_read()
s.solve(nrto.NRTO_DR, out=o); torch.cuda.synchronize()
prof = s.profile_read()
print(f"DR solve {t:.1f} ms ({1000 * t / (La * 100):.1f} us per DR iteration); launches/solve {s.launches()}")
print("profiled:", ", ".join(f"{k} {v[0]:.1f} ms/{v[1]}" for k, v in prof.items()))
