"""c4 constraint/horizon scaling sweep (BASELINE configs[3]): one
quadcopter instance per point, T x obstacle count, both engines, fixed iteration
counts; prints one JSON line per point (device time by CUDA events, after one
warm-up solve that also captures the CUDA graph).
usage: sweep_c4.py [T,... [obs,...]]"""
import json, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen.problems import make_quad, stack_instances, CONFIGS
Ts = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "50,100,200,400,800").split(",")]
OBS = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "10,20,50,100,200").split(",")]
budget_e = float(os.environ.get("C4_MAX_E", 4e8))       # skip points above this many cone elements
for T in Ts:
    for nobs in OBS:
        t0 = time.time()
        shp, d = make_quad(CONFIGS["c4"], 0, T=T, n_obs=nobs)
        E, _ = nrto.nrto_layout(shp, 1)
        if E > budget_e:
            print(json.dumps({"T": T, "n_obs": nobs, "E": int(E), "skipped": "E above C4_MAX_E"}), flush=True)
            continue
        dd = nrto.to_tensors(stack_instances([(shp, d)])[1], device="cuda")
        row = {"T": T, "n_obs": nobs, "n_g": int(shp.n_g), "E": int(E)}
        for eng, kw, name in ((nrto.NRTO_FULLADMM, dict(max_iter=10), "fulladmm"),
                              (nrto.NRTO_DR, dict(max_admm_iter=2, max_dr_iter=10), "dr")):
            s = nrto.InnerSolver(shp, dd, fixed_iters=1, **kw)
            o = nrto.alloc_out(shp, 1, s.E, device="cuda", full=False)
            s.solve(eng, out=o); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); s.solve(eng, out=o); b.record(); torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            its = kw.get("max_iter", 0) or kw["max_admm_iter"] * kw["max_dr_iter"]
            row[name] = {"us_per_iteration": 1000 * ms / its, "cone_elements_per_s": E * its / (ms / 1e3)}
            s.close()
        row["wall_s"] = round(time.time() - t0, 1)
        print(json.dumps(row), flush=True)
