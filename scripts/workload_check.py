"""Convergence and projection-case mix of the bench workload, by the ORACLE only.

For c3 instance 0 and c5 instances {0, 137, 300, 511} this runs the structured
oracle's FullADMM (Algorithm 1) with termination on (eps_p = eps_d =
1e-3, P:1439 / DESIGN R6, checked every iteration) up to L_max = 600 and records
  * the iteration at which it stops (r_p <= eps_p and r_d <= eps_d),
  * the three-case histogram of the SOC projection (SM Eq.(18)) per
    iteration, summarised as the case-3 share over iterations 6..stop (SURVEY
    §8d: a run is representative only if case 3 >= 5 % after iteration 5),
  * final objective and r_p / r_d.
Output: tests/golden/workload_c3_c5.json (read by the GPU tests and bench.py).
Calls gen/ and oracle/ only.
"""
from __future__ import annotations

import json
import os
import sys
from multiprocessing import Pool

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [("c3", 0), ("c5", 0), ("c5", 137), ("c5", 300), ("c5", 511)]
L_MAX = 600


def run(case):
    import numpy as np
    from threadpoolctl import threadpool_limits
    from gen import make_instance
    from oracle.structured import StructuredProblem, fulladmm
    from oracle.params import make_params
    cfg, i = case
    with threadpool_limits(limits=1):
        shape, data = make_instance(cfg, i)
        sp = StructuredProblem(shape, data)
        r = fulladmm(sp, make_params(max_iter=L_MAX, fixed_iters=0, check_every=1), hist=True)
    C = np.asarray(r["cases"])
    after = C[5:] if len(C) > 5 else C
    return {"cfg": cfg, "instance": i, "n_g": shape.n_g, "iters": int(r["iters"]),
            "status": int(r["status"]), "r_p": float(r["r_p"]), "r_d": float(r["r_d"]),
            "objective": float(r["objective"]),
            "g0_max": float(np.max(data["g0"])),
            "case_share_after5": [float(x) for x in after.sum(0) / after.sum()],
            "cases_first5": C[:5].tolist()}


if __name__ == "__main__":
    with Pool(len(CASES)) as p:
        res = p.map(run, CASES)
    out = {"script": "scripts/workload_check.py", "eps_p": 1e-3, "eps_d": 1e-3, "L_max": L_MAX,
           "rule": "case-3 share over iterations 6..stop >= 0.05 (SURVEY 8d)", "cases": res}
    path = os.path.join(ROOT, "tests", "golden", "workload_c3_c5.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    for r in res:
        print(r["cfg"], r["instance"], "iters", r["iters"], "status", r["status"],
              "case3 %.1f%%" % (100 * r["case_share_after5"][2]), "g0_max %.3f" % r["g0_max"])
