"""Phase timing (clock64, SM cycles) of one k_qp_sparse CTA inside a bench-size solve.
usage: qp_clocks.py [B]"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_02642_b200 import nrto
from gen import make_batch
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
shape, batch = make_batch("c5", B)
dd = nrto.to_tensors(batch, device="cuda")
names = ["zero", "prologue", "r_u", "r_x", "bwd rec", "kff", "e_k", "fwd rec", "du~", "rows", "ball"]
for L in (50,):
    s = nrto.InnerSolver(shape, dd, max_iter=L, fixed_iters=1)
    od = nrto.alloc_out(shape, B, s.E, device="cuda", full=False)
    s.solve(nrto.NRTO_FULLADMM, out=od); torch.cuda.synchronize()
    c = (ctypes.c_longlong * 64)()
    nrto.lib().nrto_debug_qp_clocks(c)
    c = np.array(c[:])
    t0 = c[0]
    print("B", B, "cycles since CTA start (it0 / it1):")
    for it in (0, 1):
        row = c[it * 32: it * 32 + 11]
        prev = c[1] if it == 0 else c[10]
        seq = []
        for ph in range(2, 11):
            seq.append(f"{names[ph]} {row[ph] - (row[ph-1] if ph > 2 else prev)}")
        print(f" it{it}:", ", ".join(seq))
    print(" prologue", c[1] - c[0])
    s.close()
