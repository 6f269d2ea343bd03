#!/usr/bin/env python
"""Benchmark of the NRTO inner solve (one JSON line on rank 0).

Workload: config c5 of BASELINE.json -- a batch of 4096
independent Franka-shaped SOCP subproblems (n_x=14, n_u=7, T=100, n_g=4306
cones, E=2.12M ragged cone elements each), FullADMM engine, L=50 iterations
with fixed_iters, STRONG scaling: rank r of N owns 4096/N instances
and runs them in waves of <= 512 resident instances (one handle; the 4096
instances' primitives stay resident in HBM, ~1 MB each).  One step = one
SL-iteration subproblem for the whole batch: per wave nrto_refresh (setup
S0-S2 from the device-resident primitives) + nrto_inner_solve (S3-S10).
The working set (~35 GB per wave) is >> the 126 MB L2: no flush is needed.

`--impl reference` times the CPU oracle (oracle/, as it stands) on a bounded
sample of the same workload, one instance per host core per step.
`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N processes (one per GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

METRIC = "inner DR/ADMM iters/sec and SOC projections/sec per GPU; SL-iteration wall-clock"
UNIT = "instance-iterations/s"
NOMINAL_HBM_GBS = 8000.0       # B200 HBM3e nominal (north_star's "~8 TB/s")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--instances", type=int, default=4096, help="total instances (strong scaling)")
    ap.add_argument("--wave", type=int, default=512, help="max resident instances per wave")
    ap.add_argument("--pipe", type=int, default=1, help="handles the waves alternate between (2: setup of wave w+1 beside the solve of wave w; measured slower, 58.6 k vs 61.8 k)")
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--conv-max-iter", type=int, default=600)
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-conv", action="store_true")
    ap.add_argument("--no-dr", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev, self.rows, self.stop = dev, [], threading.Event()

    def _run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def shape_stats(shape):
    """E, E_s, E_B (state rows), n_ctrl -- SURVEY §8(d) notation."""
    nx, nu = shape.n_x, shape.n_u
    knot = np.asarray(shape.cone_knot, np.int64)
    st = np.asarray(shape.cone_kind) == 0
    E_s = int(((knot[st] + 1) * nx).sum())
    n_ctrl = int((~st).sum())
    E = E_s + n_ctrl * nx
    E_B = int((knot[st] * nu).sum())
    return E, E_s, E_B, n_ctrl


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def _gen_chunk(args):
    cfg, first, n = args
    from gen import make_batch
    return make_batch(cfg, n, start=first)


def make_shard(cfg, first, count, procs=None):
    """The rank's instances (gen/, seeded per instance), generated in a process pool."""
    from gen import stack_instances  # noqa: F401  (import check)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    procs = procs or max(1, min(16, (os.cpu_count() or 1) // world))
    chunks = []
    step = max(1, (count + procs - 1) // procs)
    for a in range(first, first + count, step):
        chunks.append((cfg, a, min(step, first + count - a)))
    if len(chunks) == 1:
        return _gen_chunk(chunks[0])
    import multiprocessing as mp
    with mp.get_context("spawn").Pool(min(procs, len(chunks))) as pool:
        parts = pool.map(_gen_chunk, chunks)
    shape = parts[0][0]
    batch = {k: np.concatenate([p[1][k] for p in parts]) for k in parts[0][1]}
    return shape, batch


def _oracle_worker(args):
    cfg, i, L = args
    from threadpoolctl import threadpool_limits
    from gen import make_instance
    from oracle import structured as st
    from oracle.params import make_params
    with threadpool_limits(limits=1):
        shape, data = make_instance(cfg, i)
        t0 = time.perf_counter()
        sp = st.StructuredProblem(shape, data)
        st.fulladmm(sp, make_params(max_iter=L, fixed_iters=1))
        return time.perf_counter() - t0


def cpu_oracle_sample(cfg, L, seed0=0, cores=None):
    """The oracle as it stands, one single-threaded process per host core, each
    solving one instance x L FullADMM iterations (setup included).  Returns
    (instance-iterations/s over the wall time, wall s, cores used, 1-core rate)."""
    cores = cores or max(1, min(32, os.cpu_count() or 1))
    jobs = [(cfg, seed0 + i, L) for i in range(cores)]
    import multiprocessing as mp
    t0 = time.perf_counter()
    if cores == 1:
        per = [_oracle_worker(jobs[0])]
    else:
        with mp.get_context("spawn").Pool(cores) as pool:
            per = pool.map(_oracle_worker, jobs)
    wall = time.perf_counter() - t0
    return cores * L / wall, wall, cores, L / float(np.mean(per))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def workload_config(args, world, shape, E, per_rank, wave):
    return {"workload": f"{args.workload}: {args.instances} Franka-shaped SOCP subproblems "
                        f"(n_x=14, n_u=7, T=100, n_g={shape.n_g}, E={E}) sharded over "
                        f"{world} GPU(s), FullADMM, L={args.iters} fixed iterations; "
                        f"{per_rank} instances/GPU in waves of {wave}",
            "global_batch": args.instances, "parallelism": f"instances sharded dp{world}",
            "l2": "inputs larger than L2 (working set ~%.0f GB per wave)"
                  % (wave * 8 * (3 * E + E) / 1e9)}


# -------------------------------------------------------------- reference
def run_reference(args, rank, world):
    if rank != 0:
        return
    L = args.iters
    cfg = args.workload
    cpu_oracle_sample(cfg, L, seed0=0, cores=1)          # warm the interpreter / imports
    walls, rates, cores = [], [], 1
    for s in range(args.steps):
        v, wall, cores, _ = cpu_oracle_sample(cfg, L, seed0=1000 + s * 64)
        walls.append(wall)
        rates.append(v)
    ms = 1000.0 * float(np.mean(walls))
    value = cores * L / (ms / 1000.0)
    sample = (f"bounded sample: {cores} {cfg} instances x {L} FullADMM iterations (+ setup) per "
              f"step, one single-threaded oracle process per host core ({cores} of "
              f"{os.cpu_count()} cores, {cpu_model()})")
    from gen import make_instance
    shape, _ = make_instance(cfg, 0)
    E = shape_stats(shape)[0]
    per_rank = args.instances // max(1, world)
    config = workload_config(args, world, shape, E, per_rank, min(args.wave, per_rank))
    config["sample"] = sample
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (gen/, seeded PCG64)",
            "config": config,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2603_02642_b200.build import build as _build, needs_build
    if needs_build():
        if rank == 0:
            _build()
        if world > 1:
            dist.barrier()
    from paper_2603_02642_b200 import nrto
    from paper_2603_02642_b200.dist import (strong_range, max_over_ranks, batch_stats,
                                            solve_collective, nccl_max)

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L = args.iters
    first, count = strong_range(rank, world, args.instances)
    nw = max(1, -(-count // args.wave))
    wave = -(-count // nw)
    waves = [(a, min(wave, count - a)) for a in range(0, count, wave)]
    shape, batch = make_shard(args.workload, first, count)
    E, E_s, E_B, n_ctrl = shape_stats(shape)
    data_dev = nrto.to_tensors(batch, device=dev)            # primitives of every instance, resident
    sl = lambda d, a, n: {k: v[a:a + n] for k, v in d.items()}
    # wave pipeline: consecutive waves alternate between `pipe` handles on their own
    # streams, so the setup (S0-S2) of wave w+1 runs while wave w is still solving
    # (nrto_refresh blocks only the host thread, on its own stream)
    pipe = max(1, min(args.pipe, len(waves)))
    torch.cuda.synchronize()                                  # primitives resident before any setup
    stream = torch.cuda.current_stream()
    pstreams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(pipe - 1)]
    psolvers = [dict() for _ in range(pipe)]
    for i in range(pipe):
        for a, n in waves:                                    # one handle per distinct wave size
            if n not in psolvers[i]:
                psolvers[i][n] = nrto.InnerSolver(shape, sl(data_dev, a, n), max_iter=L, fixed_iters=1,
                                                  stream=None if i == 0 else pstreams[i])
    solvers = psolvers[0]                                     # the current stream's handles
    out = nrto.alloc_out(shape, count, solvers[wave].E, device=dev, full=True, ragged=False)

    def step():
        ev = torch.cuda.Event()
        ev.record(stream)
        for st in pstreams[1:]:
            st.wait_event(ev)
        for w, (a, n) in enumerate(waves):
            s = psolvers[w % pipe][n]
            s.refresh(sl(data_dev, a, n))
            s.solve(nrto.NRTO_FULLADMM, out=sl(out, a, n))
        for st in pstreams[1:]:
            e2 = torch.cuda.Event()
            e2.record(st)
            stream.wait_event(e2)

    def barrier():
        if world > 1:
            dist.barrier()

    def launches():
        return sum(s.launches() for ps in psolvers for s in ps.values())

    # ---- headline: device-resident inputs, profiler OFF (production launch path)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    l0 = launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    n_launch = launches() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_max = max_over_ranks(ms, device=dev)
    value = args.instances * L / (ms_max / 1000.0)

    # ---- profiled pass (separate, 1 step): per-kernel-class device time (CUDA events on
    # each launching stream), the pass kernel's own byte counter, projection-case mix
    for s in solvers.values():
        s.profile(True); s.profile_read(); s.pass_bytes(); s.case_stats(True)
    torch.cuda.synchronize()
    case_tot = np.zeros((L, 3), np.int64)
    for a, n in waves:
        s = solvers[n]
        s.refresh(sl(data_dev, a, n))
        s.solve(nrto.NRTO_FULLADMM, out=sl(out, a, n))
        case_tot += s.case_stats_read(L)
    torch.cuda.synchronize()
    prof = {}
    moved = 0
    for s in solvers.values():
        for k, (t_ms, n_l) in s.profile_read().items():
            a0, b0 = prof.get(k, (0.0, 0))
            prof[k] = (a0 + t_ms, b0 + n_l)
        moved += s.pass_bytes()
        s.profile(False); s.case_stats(False)

    # batch-wide residual statistics of the fixed-L solve (allreduce over ranks)
    max_rp, n_unconv, any_div = batch_stats(out["r_p"], out["status"], device=dev)

    # ---- end to end through the C ABI with HOST buffers (H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        data_host = nrto.to_tensors(batch, device="cpu", pinned=True)
        out_h = nrto.alloc_out(shape, count, solvers[wave].E, device="cpu", pinned=True, full=True,
                               ragged=False)
        h2d = sum(v.numel() * v.element_size() for v in data_host.values())
        d2h = sum(v.numel() * v.element_size() for v in out_h.values())

        def step_e2e():
            for a, n in waves:
                s = solvers[n]
                s.refresh(sl(data_host, a, n), memory=nrto.NRTO_MEM_HOST)
                s.solve(nrto.NRTO_FULLADMM, out=sl(out_h, a, n), memory=nrto.NRTO_MEM_HOST)

        step_e2e()
        torch.cuda.synchronize()
        barrier()
        ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev2.record(stream)
        for _ in range(args.steps):
            step_e2e()
        ev3.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = max_over_ranks(ev2.elapsed_time(ev3) / args.steps, device=dev)
        e2e = {"value": args.instances * L / (ems / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
               "ms_per_step": ems,
               "note": "refresh from pinned host primitives + fixed-L solve + D2H of every "
                       "output, per wave, all ranks; bytes summed over ranks"}

    # ---- SL-iteration wall-clock to CONVERGENCE (termination on, eps_p = eps_d = 1e-3,
    # L_max = conv-max-iter): host pinned inputs -> refresh -> solve to convergence with
    # the batch-wide allreduce(MAX) of the residual flags every iteration (SURVEY §8e,
    # nrto_solve_* incremental ABI) -> D2H of the outputs; device events, max over ranks
    conv = None
    if not args.no_conv:
        for sv in solvers.values():           # free the fixed-L handles (HBM) first
            sv.close()
        csol = {}
        for a, n in waves:
            if n not in csol:
                csol[n] = nrto.InnerSolver(shape, sl(data_dev, a, n), max_iter=args.conv_max_iter,
                                           eps_p=1e-3, eps_d=1e-3, check_every=1)
        data_host = data_host if e2e else nrto.to_tensors(batch, device="cpu", pinned=True)
        Ew = nrto.nrto_layout(shape, 1)[0]
        out_c = nrto.alloc_out(shape, count, Ew, device="cpu", pinned=True, full=True, ragged=False)
        out_cd = nrto.alloc_out(shape, count, Ew, device=dev, full=True, ragged=False)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev4, ev5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev4.record(stream)
        ncoll, iters_run = 0, 0
        for a, n in waves:
            s = csol[n]
            s.refresh(sl(data_host, a, n), memory=nrto.NRTO_MEM_HOST)
            o, done, nc = solve_collective(s, nrto.NRTO_FULLADMM, out=sl(out_cd, a, n),
                                           allreduce=nccl_max if world > 1 else None)
            ncoll += nc
            iters_run += done
            for k in out_c:
                out_c[k][a:a + n].copy_(o[k], non_blocking=True)
        ev5.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        cms = max_over_ranks(ev4.elapsed_time(ev5), device=dev)
        wall = max_over_ranks(wall * 1000.0, device=dev)
        its = out_c["iters"].numpy().astype(np.float64)
        stt = out_c["status"].numpy()
        if world > 1:
            g_its = [None] * world
            dist.all_gather_object(g_its, (its.tolist(), stt.tolist()))
            its = np.concatenate([np.asarray(x[0]) for x in g_its])
            stt = np.concatenate([np.asarray(x[1]) for x in g_its])
        inst_its = float(its.sum())
        conv = {"eps_p": 1e-3, "eps_d": 1e-3, "max_iter": args.conv_max_iter, "check_every": 1,
                "iters_to_converge": {"p50": float(np.median(its)), "max": float(its.max()),
                                      "min": float(its.min()), "mean": float(its.mean())},
                "converged": int((stt == 0).sum()), "instances": int(len(stt)),
                "diverged": int((stt == 2).sum()),
                "sl_iteration_wall_clock_ms": cms, "host_wall_ms": wall,
                "instance_iterations_per_s": inst_its / (cms / 1000.0),
                "collectives_per_rank": ncoll,
                "note": "one SL iteration for the whole batch: H2D of the primitives, setup, "
                        "inner solve to convergence (per-instance freeze, batch-wide "
                        "termination allreduce every iteration), D2H of the outputs"}
        for s in csol.values():
            s.close()

    # secondary lines (rank 0): NRTO-DR engine on c2 (configs[1]) and single-instance
    # latency of c1 (both engines) and c3 -- CUDA-graph replay of the fixed loop
    dr, singles = None, None
    if not args.no_dr and rank == 0:
        from gen import make_instance, stack_instances
        shp2, d2 = make_instance("c2")
        dd2 = nrto.to_tensors(stack_instances([(shp2, d2)])[1], device=dev)
        s2 = nrto.InnerSolver(shp2, dd2, fixed_iters=1)
        o2 = nrto.alloc_out(shp2, 1, s2.E, device=dev, full=False)
        s2.solve(nrto.NRTO_DR, out=o2)
        torch.cuda.synchronize()
        e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e4.record(stream)
        for _ in range(2):
            s2.solve(nrto.NRTO_DR, out=o2)
        e5.record(stream)
        torch.cuda.synchronize()
        dms = e4.elapsed_time(e5) / 2
        La, Ld = s2.params.max_admm_iter, s2.params.max_dr_iter
        dr = {"workload": "c2: quadcopter NRTO-DR, 1 instance (n_x=12, n_u=4, T=50, n_g=%d), "
                          "%d NRTO-ADMM x %d DR iterations, fixed" % (shp2.n_g, La, Ld),
              "dr_iters_per_s": La * Ld / (dms / 1000.0),
              "admm_iters_per_s": La / (dms / 1000.0), "ms_per_solve": dms}
        s2.close()
        singles = {}
        for cfg, eng, name in (("c1", nrto.NRTO_FULLADMM, "c1_fulladmm"), ("c1", nrto.NRTO_DR, "c1_dr"),
                               ("c3", nrto.NRTO_FULLADMM, "c3_fulladmm")):
            shp3, d3 = make_instance(cfg)
            dd3 = nrto.to_tensors(stack_instances([(shp3, d3)])[1], device=dev)
            s3 = nrto.InnerSolver(shp3, dd3, fixed_iters=1)
            o3 = nrto.alloc_out(shp3, 1, s3.E, device=dev, full=False)
            for _ in range(2):
                s3.solve(eng, out=o3)
            torch.cuda.synchronize()
            e6, e7 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e6.record(stream)
            for _ in range(3):
                s3.solve(eng, out=o3)
            e7.record(stream)
            torch.cuda.synchronize()
            sms = e6.elapsed_time(e7) / 3
            if eng == nrto.NRTO_FULLADMM:
                it = s3.params.max_iter
                singles[name] = {"workload": "%s, 1 instance (n_x=%d, n_u=%d, T=%d, n_g=%d), FullADMM, %d iterations, fixed"
                                 % (cfg, shp3.n_x, shp3.n_u, shp3.T, shp3.n_g, it),
                                 "inner_iters_per_s": it / (sms / 1000.0), "us_per_iteration": 1000 * sms / it,
                                 "ms_per_solve": sms}
            else:
                La, Ld = s3.params.max_admm_iter, s3.params.max_dr_iter
                singles[name] = {"workload": "%s, 1 instance (n_x=%d, n_u=%d, T=%d, n_g=%d), NRTO-DR, %d x %d, fixed"
                                 % (cfg, shp3.n_x, shp3.n_u, shp3.T, shp3.n_g, La, Ld),
                                 "dr_iters_per_s": La * Ld / (sms / 1000.0), "us_per_dr_iteration": 1000 * sms / (La * Ld),
                                 "ms_per_solve": sms}
            s3.close()

    # c4 constraint / horizon scaling points (BASELINE configs[3]; one quadcopter instance
    # each, both engines, fixed iterations) with their SURVEY §8(d) bytes and fraction
    c4 = None
    if not args.no_c4 and rank == 0:
        from gen.problems import make_quad, stack_instances, CONFIGS
        peak_c4, _ = load_peaks()
        c4 = []
        for T4, nobs in ((50, 10), (200, 50), (800, 200)):
            shp4, d4 = make_quad(CONFIGS["c4"], 0, T=T4, n_obs=nobs)
            E4, E4s, E4B, _ = shape_stats(shp4)
            dd4 = nrto.to_tensors(stack_instances([(shp4, d4)])[1], device=dev)
            bytes_it = 8 * (2 * E4 + E4s + E4B)
            row = {"T": T4, "n_obs": nobs, "n_g": int(shp4.n_g), "E": int(E4),
                   "alg_bytes_per_iteration": bytes_it}
            for eng, kw4, name in ((nrto.NRTO_FULLADMM, dict(max_iter=10), "fulladmm"),
                                   (nrto.NRTO_DR, dict(max_admm_iter=2, max_dr_iter=10), "dr")):
                s4 = nrto.InnerSolver(shp4, dd4, fixed_iters=1, **kw4)
                o4 = nrto.alloc_out(shp4, 1, s4.E, device=dev, full=False)
                s4.solve(eng, out=o4)
                torch.cuda.synchronize()
                a4, b4 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a4.record(stream); s4.solve(eng, out=o4); b4.record(stream)
                torch.cuda.synchronize()
                ms4 = a4.elapsed_time(b4)
                its = kw4.get("max_iter", 0) or kw4["max_admm_iter"] * kw4["max_dr_iter"]
                gbs = bytes_it * its / (ms4 / 1e3) / 1e9
                row[name] = {"us_per_iteration": 1000 * ms4 / its, "achieved_gbs_8d": gbs,
                             "frac_8d": gbs / peak_c4, "iterations": its}
                s4.close()
            del dd4
            c4.append(row)

    # case mix over all ranks (SURVEY §8d representativeness rule: case 3 >= 5 % after l = 5)
    ct = torch.as_tensor(case_tot, dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ct)
    case_tot = ct.cpu().numpy()
    if rank != 0:
        return
    after = case_tot[5:].sum(0)
    share = after / max(after.sum(), 1.0)
    first5 = case_tot[:5].sum(0) / max(case_tot[:5].sum(), 1.0)
    case_mix = {"after_iter5": {"case1": float(share[0]), "case2": float(share[1]), "case3": float(share[2])},
                "iters_1_to_5": {"case1": float(first5[0]), "case2": float(first5[1]), "case3": float(first5[2])},
                "representative": bool(share[2] >= 0.05),
                "rule": "case 3 >= 5 % of projections after iteration 5 (SURVEY §8d)"}

    peak, peak_kind = load_peaks()
    # roofline of the dominant kernel k_fa_tma (state cones):
    #   achieved (§8d) = SURVEY §8(d) algorithmic bytes of the state-cone stream per
    #     instance-iteration, 8 (2 E_s + E_s + E_B), x the instances of a launch, / its
    #     event-timed average duration in the profiled step (same launch path as the headline)
    #   dram = the bytes the kernel itself counts (lazy y: b_hat + b + y where read /
    #     stored), same time -- what HBM actually carries (ncu agrees, `traffic`)
    pms, pn = prof["pass"]
    bytes8d = 8 * (3 * E_s + E_B)
    inst_per_launch = float(count) / max(1, len(waves))
    t_launch = (pms / pn) / 1000.0 if pn else None
    achieved = bytes8d * inst_per_launch / t_launch / 1e9 if t_launch else None
    dram_gbs = (moved / pn) / t_launch / 1e9 if t_launch else None
    traffic = None
    tf = os.path.join(ROOT, "profiles", "pass_traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            if tj.get("wave") == wave and tj.get("iters") == L:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            pass
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v_all, wall, cores, v1 = cpu_oracle_sample(args.workload, L, seed0=0)
        cpu = {"value": v_all, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{cores} {args.workload} instances x {L} FullADMM iterations incl. setup, "
                         f"one single-threaded oracle process per core ({wall:.1f} s wall)",
               "value_1core": v1, "cpu_model": cpu_model(), "nproc": os.cpu_count()}
    kernel_ms = {k: (v[0]) for k, v in prof.items()}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen/, seeded PCG64; no datasets or trained weights)",
        "config": workload_config(args, world, shape, E, count, wave),
        "value_per_gpu": value / world,
        "soc_projections_per_s": value * shape.n_g,
        "cone_elements_per_s": value * E,
        "sl_iteration_wall_clock_ms": (conv or {}).get("sl_iteration_wall_clock_ms"),
        "convergence": conv,
        "case_mix": case_mix,
        "kernel_ms_per_step": kernel_ms,
        "kernel_ms_note": ("one separate profiled step (CUDA events per kernel class on its launching "
                           "stream); qp (low-priority stream) and ctrl (second high-priority stream) "
                           "run concurrently with pass / adjoint / gain, so classes overlap and do not "
                           "add up to the step; the headline steps run with the profiler off"),
        "roofline": {"bound": "hbm",
                     "kernel": "k_fa_tma: fused state-cone pass (S3 forward map + S4 SOC norms + "
                               "S5 state update)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "peak_kind": peak_kind,
                     "frac_vs_nominal_8tbs": (achieved / NOMINAL_HBM_GBS) if achieved else None,
                     "algorithmic_bytes_per_launch": bytes8d * inst_per_launch,
                     "algorithmic_bytes_def": "SURVEY 8(d): 8 (2 E_s + E_s + E_B) per instance-iteration "
                                              "(state-cone row read+write, b_hat, b) x instances per launch",
                     "dram_achieved": dram_gbs,
                     "dram_frac": (dram_gbs / peak) if dram_gbs else None,
                     "dram_bytes_per_launch": (moved / pn) if pn else None,
                     "dram_def": "bytes the kernel moves (lazy y: b_hat + b of every block, y^{l-1} "
                                 "read / y^l stored only where needed), counted by the kernel",
                     "avg_launch_ms": (pms / pn) if pn else None, "launches": pn},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(n_launch),
        "clocks": clk.summary(),
        "dr_engine": dr,
        "single_instance": singles,
        "c4_sweep": c4,
        "residuals": {"max_r_p_at_L": max_rp, "unconverged_at_L": n_unconv,
                      "any_diverged": any_div},
    }
    print(json.dumps(line), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
