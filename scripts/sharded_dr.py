"""Cone-sharded NRTO-DR of ONE large instance over the ranks.
One process per GPU (torchrun, NCCL): every rank sets up the whole quadcopter
instance, streams only its cone range in the DR pass, and the ranks allreduce the
T n_u n_x adjoint after every pass and pi before every QP.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
      scripts/sharded_dr.py --T 800 --obs 200 --admm 2 --dr 10
Prints one JSON line on rank 0: ms per DR iteration (max over ranks)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from gen.problems import make_quad, stack_instances, CONFIGS
from paper_2603_02642_b200 import nrto
from paper_2603_02642_b200.dist import cone_range, sharded_dr_solve

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=800)
ap.add_argument("--obs", type=int, default=200)
ap.add_argument("--admm", type=int, default=2)
ap.add_argument("--dr", type=int, default=10)
a = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl")
shape, data = make_quad(CONFIGS["c4"], 0, T=a.T, n_obs=a.obs)
t = nrto.to_tensors(stack_instances([(shape, data)])[1], device="cuda")
lo, hi = cone_range(rank, world, shape)
allreduce = (lambda x: dist.all_reduce(x)) if world > 1 else None
times = []
for rep in range(2):                                   # first: warm-up (graph-free path)
    s = nrto.InnerSolver(shape, t, fixed_iters=1, max_admm_iter=a.admm, max_dr_iter=a.dr)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = sharded_dr_solve(s, lo, hi, allreduce)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
    s.close()
ms = torch.tensor([times[-1]], dtype=torch.float64, device="cuda")
if world > 1:
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
if rank == 0:
    print(json.dumps({"config": f"c4 quadcopter T={a.T}, {a.obs} obstacles, n_g={shape.n_g}",
                      "ranks": world, "cones_rank0": [lo, hi], "admm": a.admm, "dr": a.dr,
                      "ms_per_solve": ms.item(), "ms_per_dr_iteration": ms.item() / (a.admm * a.dr)}))
if world > 1:
    dist.destroy_process_group()
