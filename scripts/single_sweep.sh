#!/bin/bash
# single-instance FullADMM timing under launch knobs (probe only)
cd "$(dirname "$0")/.."
for cfg in "$@"; do
  echo "$cfg" >> gpurun_out/single_sweep.txt
  env $cfg timeout 300 python - >> gpurun_out/single_sweep.txt 2>&1 <<'PY'
import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2603_02642_b200 import nrto
from gen import make_instance
from gen.problems import stack_instances
for cfg in ("c1", "c3"):
    shp, d = make_instance(cfg)
    dd = nrto.to_tensors(stack_instances([(shp, d)])[1], device="cuda")
    s = nrto.InnerSolver(shp, dd, fixed_iters=1, max_iter=40)
    o = nrto.alloc_out(shp, 1, s.E, device="cuda", full=False)
    for _ in range(2): s.solve(nrto.NRTO_FULLADMM, out=o)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): s.solve(nrto.NRTO_FULLADMM, out=o)
    b.record(); torch.cuda.synchronize()
    print(cfg, "us/it %.1f" % (1000 * a.elapsed_time(b) / 3 / 40))
    s.close()
PY
done
