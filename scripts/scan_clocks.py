"""Phase clocks (SM cycles) of the chunked-scan QP, QP iteration 1 of the last launch,
instance 0.  usage: scan_clocks.py cfg [engine]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import make_instance, stack_instances
from paper_2603_02642_b200 import nrto
names = ["r_u", "a_k", "bwd local", "bwd chain", "bwd interior", "kff", "e_k", "fwd local",
         "fwd chain", "fwd interior", "du~", "rows", "ball"]
for cfg in sys.argv[1:] or ["c1", "c3"]:
    shp, d = make_instance(cfg)
    dd = nrto.to_tensors(stack_instances([(shp, d)])[1], device="cuda")
    s = nrto.InnerSolver(shp, dd, fixed_iters=1, max_iter=3)
    s.solve(0); torch.cuda.synchronize()
    buf = (C.c_longlong * 64)()
    nrto.lib().nrto_debug_qp_clocks(buf)
    a = np.array(buf[32:46], dtype=np.float64)
    dt = np.diff(a)
    print(cfg, "total %.0f cycles:" % (a[13] - a[0]), ", ".join("%s %.0f" % (n, x) for n, x in zip(names, dt)))
    s.close()
