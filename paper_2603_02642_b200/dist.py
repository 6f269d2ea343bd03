"""Multi-GPU plumbing for the instance-sharded inner solve.

Instances are independent: rank r of N owns a contiguous range
of instances and its own nrto handle; no data-path collective exists.  The
collectives are the batch-wide termination test inside the loop (allreduce MAX
of the 4 residual flags every check_every outer iterations, `solve_collective`),
the max-over-ranks step time and the final residual statistics (max r_p,
#unconverged, any diverged), done through torch.distributed (NCCL over NVLink
on the GPU box, gloo in CPU tests).
"""
from __future__ import annotations


def instance_range(rank: int, world: int, per_rank: int):
    """(first instance, count) of rank `rank` under weak scaling."""
    if not (0 <= rank < world) or per_rank < 1:
        raise ValueError("bad rank/world/per_rank")
    return rank * per_rank, per_rank


def strong_range(rank: int, world: int, total: int):
    """(first, count) of a contiguous split of `total` instances (strong scaling)."""
    base, rem = divmod(total, world)
    first = rank * base + min(rank, rem)
    return first, base + (1 if rank < rem else 0)


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def batch_stats(r_p, status, device=None):
    """Batch-wide residual reduction: (max r_p, #unconverged, any diverged)."""
    import torch
    import torch.distributed as dist
    r_p = torch.as_tensor(r_p, device=device)
    status = torch.as_tensor(status, device=device)
    mx = torch.tensor([r_p.max().item() if r_p.numel() else 0.0], dtype=torch.float64,
                      device=device)
    cnt = torch.tensor([float((status != 0).sum().item()), float((status == 2).any().item())],
                       dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    return float(mx.item()), int(cnt[0].item()), bool(cnt[1].item() > 0)


def collective_loop(iterate, read_flags, allreduce, L: int, check_every: int):
    """Host loop of the multi-rank termination test (Algorithm 1 line 9, P:522;
    SURVEY §8e).  `iterate(n)` runs up to n more outer iterations and returns the
    number run so far; `read_flags()` returns the 4-vector [max r_p/eps_p,
    max r_d/eps_d, #active, any diverged] of this rank; `allreduce(flags)`
    reduces it in place with MAX over ranks (None: single rank).  Stops once no
    instance on any rank is active or after L iterations.  Returns (iterations
    run, collectives issued)."""
    if check_every < 1:
        raise ValueError("check_every must be >= 1")
    done, ncoll = 0, 0
    while done < L:
        done = iterate(check_every)
        flags = read_flags()
        if allreduce is not None:
            allreduce(flags)
            ncoll += 1
        if float(flags[2]) == 0.0:
            break
    return done, ncoll


def nccl_max(flags):
    """allreduce(MAX) of a flags tensor over the default process group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(flags, op=dist.ReduceOp.MAX)


def solve_collective(solver, engine, out=None, check_every=None, allreduce=nccl_max):
    """Termination-mode inner solve of this rank's shard through the incremental
    C ABI (nrto_solve_begin / _iterate / _flags / _end), with the batch-wide
    allreduce(MAX) of the residual flags between chunks of check_every outer
    iterations.  Returns (out, iterations run, collectives issued)."""
    import torch
    from . import nrto
    if out is None:
        out = nrto.alloc_out(solver.shape, solver.batch, solver.E, device="cuda")
    ce = int(check_every or solver.params.check_every)
    L = solver.params.max_iter if engine == nrto.NRTO_FULLADMM else solver.params.max_admm_iter
    flags = torch.zeros(4, dtype=torch.float64, device="cuda")

    def read_flags():
        nrto.nrto_solve_flags(solver.handle, flags, solver.stream)
        return flags

    nrto.nrto_solve_begin(solver.handle, engine, solver.stream)
    done, ncoll = collective_loop(lambda n: nrto.nrto_solve_iterate(solver.handle, n, solver.stream),
                                  read_flags, allreduce, L, ce)
    nrto.nrto_solve_end(solver.handle, out, solver.stream)
    return out, done, ncoll


# ---------------------------------------------------------------------------
# Cone sharding of ONE instance over ranks (nrto.h
# nrto_shard_cones): every rank holds the whole problem, streams only its cones in
# the DR pass, and the ranks sum the T n_u n_x adjoint after every pass and gather
# pi before every QP.
def cone_range(rank: int, world: int, shape):
    """Contiguous cone range of `rank`, balanced by cone elements (L_j =
    (k_j + 1) n_x for state cones, n_x for control cones)."""
    import numpy as np
    knot = np.asarray(shape.cone_knot, np.int64)
    kind = np.asarray(shape.cone_kind)
    L = np.where(kind == 0, (knot + 1) * shape.n_x, shape.n_x)
    cum = np.concatenate([[0], np.cumsum(L)])
    tot = cum[-1]
    lo = int(np.searchsorted(cum, tot * rank / world, side="left")) if rank else 0
    hi = int(np.searchsorted(cum, tot * (rank + 1) / world, side="left")) if rank + 1 < world else len(L)
    return min(lo, len(L)), min(max(hi, lo), len(L))


def sharded_dr_solve(solver, cone_lo, cone_hi, allreduce, out=None, stream=None):
    """NRTO-ADMM + DR (fixed iteration counts) on a cone-sharded handle.
    `allreduce(t)` sums a float64 CUDA tensor in place over the ranks (None: one
    rank).  Returns the output dict of nrto_solve_end."""
    from . import nrto
    h = solver.handle
    nrto.nrto_shard_cones(h, cone_lo, cone_hi)
    prm = solver.params
    Z = nrto.nrto_buffer(h, 0)
    pi = nrto.nrto_buffer(h, 1)
    ng = solver.shape.n_g
    B = solver.batch
    nrto.nrto_solve_begin(h, nrto.NRTO_DR, stream)
    for l in range(1, prm.max_admm_iter + 1):
        nrto.nrto_dr_step(h, 0, l, stream)
        for _ in range(prm.max_dr_iter):
            nrto.nrto_dr_step(h, 1, l, stream)
            nrto.nrto_dr_step(h, 2, l, stream)
            if allreduce is not None:
                allreduce(Z)
        if allreduce is not None:
            p2 = pi.view(B, ng)
            p2[:, :cone_lo] = 0.0
            p2[:, cone_hi:] = 0.0
            allreduce(pi)
        nrto.nrto_dr_step(h, 3, l, stream)
    if out is None:
        out = nrto.alloc_out(solver.shape, B, solver.E, device="cuda")
    nrto.nrto_solve_end(h, out, stream)
    return out
