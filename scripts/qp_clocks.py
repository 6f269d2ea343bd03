"""Phase timing (clock64, SM cycles) of one k_qp_sparse CTA inside a bench-size solve.
Prints, per QP iteration, the cycles from the iteration start to each recorded
phase boundary (0 = not recorded by this kernel variant).
usage: qp_clocks.py [B]"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_02642_b200 import nrto
from gen import make_batch
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
shape, batch = make_batch("c5", B)
dd = nrto.to_tensors(batch, device="cuda")
names = {2: "r_u", 3: "r_x", 4: "bwd rec", 5: "kff", 6: "e_k", 7: "fwd rec", 8: "du~", 9: "rows", 10: "ball"}
s = nrto.InnerSolver(shape, dd, max_iter=50, fixed_iters=1)
od = nrto.alloc_out(shape, B, s.E, device="cuda", full=False)
s.solve(nrto.NRTO_FULLADMM, out=od); torch.cuda.synchronize()
c = (ctypes.c_longlong * 64)()
nrto.lib().nrto_debug_qp_clocks(c)
c = np.array(c[:])
print("B", B, "prologue", c[1] - c[0])
for it in (0, 1):
    start = c[1] if it == 0 else c[10]
    row = c[it * 32: it * 32 + 11]
    print(f" it{it}:", ", ".join(f"{names[p]} +{row[p] - start}" for p in range(2, 11) if row[p] > 0))
    r = c[it * 32: it * 32 + 32]
    if r[12] or r[16]:
        print(f"   bwd: chunk-wait {r[12]}, a_k spin {r[13]}, step {r[14]};  fwd: e-wait {r[16]}, chunk-wait {r[17]}, step {r[18]}")
s.close()
