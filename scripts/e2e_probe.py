"""Time the pieces of the host-buffer (e2e) path vs the device path."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_batch
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
shape, batch = make_batch("c5", B)
dd = nrto.to_tensors(batch, device="cuda")
dh = nrto.to_tensors(batch, device="cpu", pinned=True)
print("pinned:", all(t.is_pinned() for t in dh.values()))
s = nrto.InnerSolver(shape, dd, max_iter=50, fixed_iters=1)
od = nrto.alloc_out(shape, B, s.E, device="cuda"); od.pop("nu"); od.pop("lam_nu")
oh = nrto.alloc_out(shape, B, s.E, device="cpu", pinned=True); oh.pop("nu"); oh.pop("lam_nu")
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / n * 1e3
print("refresh dev  %.1f ms" % t(lambda: s.refresh(dd)))
print("refresh host %.1f ms" % t(lambda: s.refresh(dh, memory=nrto.NRTO_MEM_HOST)))
print("solve dev    %.1f ms" % t(lambda: s.solve(nrto.NRTO_FULLADMM, out=od)))
print("solve host   %.1f ms" % t(lambda: s.solve(nrto.NRTO_FULLADMM, out=oh, memory=nrto.NRTO_MEM_HOST)))
x = torch.empty(sum(v.numel() for v in dh.values()), dtype=torch.float64, device="cuda")
src = torch.empty(x.numel(), dtype=torch.float64).pin_memory()
print("raw H2D %.1f ms for %.0f MB" % (t(lambda: x.copy_(src, non_blocking=True)), x.numel() * 8 / 1e6))
