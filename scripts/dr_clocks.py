"""Phase clocks of the persistent DR loop (CTA 0, globaltimer ns), iterations 2..5."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import make_instance, stack_instances
from paper_2603_02642_b200 import nrto
for cfg in sys.argv[1:] or ["c1", "c2"]:
    shp, d = make_instance(cfg)
    dd = nrto.to_tensors(stack_instances([(shp, d)])[1], device="cuda")
    s = nrto.InnerSolver(shp, dd, fixed_iters=1, max_admm_iter=2, max_dr_iter=20)
    o = nrto.alloc_out(shp, 1, s.E, device="cuda", full=False)
    s.solve(nrto.NRTO_DR, out=o); torch.cuda.synchronize()
    s.solve(nrto.NRTO_DR, out=o); torch.cuda.synchronize()
    buf = (C.c_ulonglong * 64)()
    nrto.lib().nrto_debug_dr_clocks(buf)
    a = np.array(buf[:32], dtype=np.float64).reshape(4, 8)
    for it in range(4):
        t = a[it]
        print(cfg, "iter", it + 2, "head %.2f G %.2f bar1 %.2f P %.2f bar2 %.2f us" % (
            (t[5] - t[0]) / 1e3, (t[1] - t[5]) / 1e3, (t[2] - t[1]) / 1e3, (t[3] - t[2]) / 1e3, (t[4] - t[3]) / 1e3))
    s.close()
    buf2 = (C.c_ulonglong * 2048)()
    s = nrto.InnerSolver(shp, dd, fixed_iters=1, max_admm_iter=1, max_dr_iter=5)
    o = nrto.alloc_out(shp, 1, s.E, device="cuda", full=False)
    s.solve(nrto.NRTO_DR, out=o); torch.cuda.synchronize()
    nrto.lib().nrto_debug_dr_pclocks(buf2)
    pc = np.array(buf2[:], dtype=np.float64).reshape(1024, 2) / 1e3
    n = int((pc[:, 1] > 0).sum())
    P, Gt = pc[:n, 0], pc[:n, 1]
    print(cfg, "CTAs", n, "P us: max %.2f mean %.2f argmax %d | G us: max %.2f mean %.2f" % (P.max(), P.mean(), P.argmax(), Gt.max(), Gt.mean()))
    print(cfg, "P per CTA:", " ".join("%.1f" % x for x in P))
    s.close()
    buf3 = (C.c_ulonglong * 8192)()
    nrto.lib().nrto_debug_dr_sub(buf3)
    sb = np.array(buf3[:], dtype=np.float64).reshape(1024, 8)
    for cta in (0, n // 2, int(P.argmax())):
        t = sb[cta]
        base = t[0] - pc[cta, 0] * 1e3 + (t[5] - t[0]) * 0   # approximate
        print(cfg, "CTA", cta, "Cload->sync %.2f flat1 %.2f red1 %.2f flat2 %.2f zpart+red2 %.2f" % tuple(
            (t[i + 1] - t[i]) / 1e3 for i in range(5)))
