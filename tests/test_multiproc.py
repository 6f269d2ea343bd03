"""World-size-2 gloo test of the instance-sharded multi-rank path (CPU).

Each rank takes its instance range, solves its shard with the CPU oracle
(standing in for the per-rank GPU handle), and the ranks meet only in the
max-over-ranks time and the batch residual statistics -- the same calls
bench.py makes over NCCL.  The sharded result must equal the unsharded one.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_02642_b200.dist import instance_range, max_over_ranks, batch_stats
    from gen.problems import make_unicycle
    from oracle import structured as st
    from oracle.params import make_params
    first, count = instance_range(rank, world, per_rank)
    r_p, status = [], []
    for i in range(first, first + count):
        shape, data = make_unicycle(1, i, T=6)
        r = st.fulladmm(st.StructuredProblem(shape, data), make_params(max_iter=15, fixed_iters=1))
        r_p.append(r["r_p"]); status.append(r["status"])
    t = max_over_ranks(float(rank + 1))
    stats = batch_stats(np.array(r_p), np.array(status))
    out[rank] = (first, count, r_p, t, stats)
    dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    world, per_rank = 2, 3
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, per_rank, out), nprocs=world, join=True)
    firsts = sorted(out[r][0] for r in range(world))
    assert firsts == [0, per_rank]                            # disjoint, covering ranges
    assert all(out[r][3] == 2.0 for r in range(world))        # max over ranks
    all_rp = out[0][2] + out[1][2]
    for r in range(world):
        mx, nun, div = out[r][4]
        assert mx == pytest.approx(max(all_rp))
        assert nun == world * per_rank and not div
    # sharded results equal the unsharded computation instance by instance
    from gen.problems import make_unicycle
    from oracle import structured as st
    from oracle.params import make_params
    for i in range(world * per_rank):
        shape, data = make_unicycle(1, i, T=6)
        r = st.fulladmm(st.StructuredProblem(shape, data), make_params(max_iter=15, fixed_iters=1))
        assert all_rp[i] == r["r_p"]


def test_ranges():
    from paper_2603_02642_b200.dist import instance_range, strong_range
    assert instance_range(3, 8, 512) == (1536, 512)
    cover = [strong_range(r, 3, 10) for r in range(3)]
    assert cover == [(0, 4), (4, 3), (7, 3)]
    with pytest.raises(ValueError):
        instance_range(2, 2, 4)


def _loop_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_02642_b200.dist import collective_loop, nccl_max
    stop_at = [7, 12][rank]          # this rank's last active instance stops here
    state = {"l": 0}

    def iterate(n):
        state["l"] = min(40, state["l"] + n)
        return state["l"]

    def read_flags():
        active = 1.0 if state["l"] < stop_at else 0.0
        return torch.tensor([10.0 / (rank + 1), 1.0 * rank, active, 0.0], dtype=torch.float64)

    box = {}

    def allreduce(f):
        nccl_max(f)
        box["f"] = f.clone()

    done, ncoll = collective_loop(iterate, read_flags, allreduce, 40, 5)
    out[rank] = (done, ncoll, box["f"].tolist())
    dist.destroy_process_group()


def test_two_rank_collective_termination_loop():
    """The in-loop batch-wide termination test: both ranks keep
    iterating until the LAST active instance on ANY rank has stopped (rank 1
    at 12 -> both stop after the chunk ending at 15), with one allreduce(MAX)
    of the flags per chunk of check_every = 5 iterations."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_loop_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        done, ncoll, f = out[r]
        assert done == 15 and ncoll == 3
        assert f == [10.0, 1.0, 0.0, 0.0]       # MAX over ranks of the last flags


def test_collective_loop_single_rank():
    from paper_2603_02642_b200.dist import collective_loop
    st = {"l": 0}

    def it(n):
        st["l"] = min(23, st["l"] + n)
        return st["l"]
    done, ncoll = collective_loop(it, lambda: [0.0, 0.0, 1.0, 0.0], None, 23, 4)
    assert done == 23 and ncoll == 0
    with pytest.raises(ValueError):
        collective_loop(it, lambda: [0, 0, 0, 0], None, 5, 0)


def test_cone_range_partition():
    """Cone sharding of one instance (NEXT-3(i)): the ranks' contiguous cone ranges
    cover every cone once and balance the cone elements."""
    import numpy as np
    from gen import make_instance
    from paper_2603_02642_b200.dist import cone_range
    shape, _ = make_instance("c2")
    knot = np.asarray(shape.cone_knot); kind = np.asarray(shape.cone_kind)
    L = np.where(kind == 0, (knot + 1) * shape.n_x, shape.n_x)
    for world in (1, 2, 3, 8):
        rs = [cone_range(r, world, shape) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == shape.n_g
        assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
        work = [L[a:b].sum() for a, b in rs]
        assert max(work) - min(work) <= L.max() + 1, work
