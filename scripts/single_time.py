"""Single-instance timings (as bench.py's dr_engine / single_instance lines):
c1 FullADMM, c1 DR, c2 DR, c3 FullADMM; one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import make_instance, stack_instances
from paper_2603_02642_b200 import nrto

res = {}
for cfg, eng, name in (("c1", 0, "c1_fa"), ("c1", 1, "c1_dr"), ("c2", 1, "c2_dr"), ("c3", 0, "c3_fa")):
    shp, d = make_instance(cfg)
    dd = nrto.to_tensors(stack_instances([(shp, d)])[1], device="cuda")
    s = nrto.InnerSolver(shp, dd, fixed_iters=1)
    o = nrto.alloc_out(shp, 1, s.E, device="cuda", full=False)
    for _ in range(2):
        s.solve(eng, out=o)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        s.solve(eng, out=o)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    its = s.params.max_iter if eng == 0 else s.params.max_admm_iter * s.params.max_dr_iter
    res[name] = round(1000 * ms / its, 2)      # us per (DR) iteration
    s.close()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("NRTO_")}, "us_per_iter": res}))
