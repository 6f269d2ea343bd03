"""Tiny solves through every kernel path, for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck).  usage: sanitize_cases.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02642_b200 import nrto
from gen import make_instance, stack_instances
from gen.problems import make_franka, make_quad


def run(name, shape, batch, engine, **kw):
    s = nrto.InnerSolver(shape, nrto.to_tensors(batch, device="cuda"), **kw)
    s.solve(engine)
    s.solve(engine)                  # second solve: graph replay where the path uses one
    torch.cuda.synchronize()
    s.close()
    print("ok", name, flush=True)


one = lambda sh, d: stack_instances([(sh, d)])[1]
sh, d = make_instance("c1")
run("c1 FullADMM (whole-loop k_fa_small, scan QP staged + resident)", sh, one(sh, d), nrto.NRTO_FULLADMM,
    max_iter=3, fixed_iters=1)
run("c1 FullADMM termination", sh, one(sh, d), nrto.NRTO_FULLADMM, max_iter=6)
run("c1 DR (persistent k_dr_loop, graph)", sh, one(sh, d), nrto.NRTO_DR, max_admm_iter=2, max_dr_iter=3,
    fixed_iters=1)
run("c1 DR early stop (in-kernel stop test)", sh, one(sh, d), nrto.NRTO_DR, max_admm_iter=2, max_dr_iter=40,
    eps_dr=1e-3)
sh2, d2 = make_instance("c2")
run("c2 DR (persistent loop, chunks)", sh2, one(sh2, d2), nrto.NRTO_DR, max_admm_iter=1, max_dr_iter=3,
    fixed_iters=1)
items = [make_quad(2, i, T=16, n_obs=4) for i in range(5)]
sh5, b5 = stack_instances(items)
run("quad batch 5 DR (several tasks per CTA)", sh5, b5, nrto.NRTO_DR, max_admm_iter=2, max_dr_iter=3,
    fixed_iters=1)
sh, d = make_franka(3, 0, T=12)
run("c3s FullADMM (TMA pass, pipelined sparse QP)", sh, one(sh, d), nrto.NRTO_FULLADMM, max_iter=3, fixed_iters=1)
run("c3s DR", sh, one(sh, d), nrto.NRTO_DR, max_admm_iter=2, max_dr_iter=3, fixed_iters=1)
items = [make_franka(5, i, T=12, jitter=True) for i in range(160)]
sh, b = stack_instances(items)
run("B=160 overlapped (QP beside pass, persistent grid)", sh, b, nrto.NRTO_FULLADMM, max_iter=3, fixed_iters=1)
sh, d = make_quad(4, 3, T=450, n_obs=1)
run("quad T=450 FullADMM (generic pass)", sh, one(sh, d), nrto.NRTO_FULLADMM, max_iter=2, fixed_iters=1)
run("quad T=450 DR (long-cone pass)", sh, one(sh, d), nrto.NRTO_DR, max_admm_iter=1, max_dr_iter=2, fixed_iters=1)
