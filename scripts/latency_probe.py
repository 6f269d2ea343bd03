"""Single-instance latency of the inner solve (c1, c2 DR, c3)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_instance, stack_instances
def run(cfg, engine, **kw):
    shape, data = make_instance(cfg)
    _, b = stack_instances([(shape, data)])
    s = nrto.InnerSolver(shape, nrto.to_tensors(b), **kw)
    out = nrto.alloc_out(shape, 1, s.E, full=False)
    s.solve(engine, out=out); torch.cuda.synchronize()
    s.profile(True); s.profile_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = s.launches()
    t = time.perf_counter(); e0.record(); s.solve(engine, out=out); e1.record(); torch.cuda.synchronize()
    wall = (time.perf_counter() - t) * 1e3
    p = s.profile_read()
    print(f"{cfg} engine={engine} {kw}: {e0.elapsed_time(e1):.2f} ms device, {wall:.2f} ms wall, iters={out['iters'].item()}, "
          f"status={out['status'].item()}, launches={s.launches()-l0}; " + ", ".join(f"{k} {v[0]:.2f}/{v[1]}" for k, v in p.items()))
    s.close()
run("c1", 0, max_iter=40, fixed_iters=1)
run("c3", 0, max_iter=50, fixed_iters=1)
run("c2", 1, max_admm_iter=40, max_dr_iter=100, fixed_iters=1)
run("c2", 1)
run("c3", 0, max_iter=200)
