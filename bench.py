#!/usr/bin/env python
"""Benchmark of the NRTO inner solve (one JSON line on rank 0).

Workload: c5 -- a batch of Franka-shaped SOCP subproblems
(n_x=14, n_u=7, T=100, n_g=4306 cones, E=2.12M ragged cone elements each),
FullADMM engine, L_max=50 iterations with fixed_iters, per-GPU batch
fixed (weak scaling; N=8 x 512 = 4096 = c5).  One step = one SL-iteration
subproblem for the whole batch: nrto_refresh (setup S0-S2 from
device-resident primitives) + nrto_inner_solve (S3-S10).  Working set per GPU
is ~22 GB >> 126 MB L2, so no L2 flush is needed between steps.

`--impl reference` times the CPU oracle (oracle/, as it stands) on a bounded
sample of the same workload (one instance per step).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

METRIC = "inner DR/ADMM iters/sec and SOC projections/sec per GPU; SL-iteration wall-clock"
UNIT = "instance-iterations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch-per-gpu", type=int, default=512)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dr", action="store_true")
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


def workload_shape_stats(shape):
    nx, nu = shape.n_x, shape.n_u
    knot = np.asarray(shape.cone_knot, np.int64)
    kind = np.asarray(shape.cone_kind)
    st = kind == 0
    E_s = int(((knot[st] + 1) * nx).sum())
    E = E_s + int((~st).sum()) * nx
    E_B = int((knot[st] * nu).sum()) + int((~st).sum()) * nu
    return E, E_s, E_B


def cpu_oracle_sample(cfg, L, n_inst=1, seed0=0):
    """Time the oracle (as it stands) on n_inst instances x L iterations, 1 thread."""
    from threadpoolctl import threadpool_limits
    from gen import make_instance
    from oracle import structured as st
    from oracle.params import make_params
    items = [make_instance(cfg, seed0 + i) for i in range(n_inst)]
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        for shape, data in items:
            sp = st.StructuredProblem(shape, data)
            st.fulladmm(sp, make_params(max_iter=L, fixed_iters=1))
        dt = time.perf_counter() - t0
    return n_inst * L / dt, dt


def workload_config(args, world, shape, E, E_B):
    """The `config` of both arms (ours and --impl reference)."""
    B, L = args.batch_per_gpu, args.iters
    return {"workload": f"{args.workload}: batch of Franka-shaped SOCP subproblems "
                        f"(n_x=14, n_u=7, T=100, n_g={shape.n_g}, E={E}), FullADMM, "
                        f"L={L} fixed iterations, {B} instances/GPU",
            "global_batch": world * B, "parallelism": f"instances sharded dp{world}",
            "l2": "inputs larger than L2 (working set ~%.0f GB/GPU)" % (B * 8 * (2 * E + E_B) / 1e9)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# -------------------------------------------------------------- reference
def run_reference(args, rank, world):
    if rank != 0:
        return
    L = args.iters
    cfg = "c5" if args.workload == "c5" else args.workload
    for _ in range(args.warmup):
        cpu_oracle_sample(cfg, L, 1, seed0=0)
    times = []
    for s in range(args.steps):
        v, dt = cpu_oracle_sample(cfg, L, 1, seed0=s + 1)
        times.append(dt)
    ms = 1000.0 * float(np.mean(times))
    value = L / (ms / 1000.0)
    sample = (f"bounded sample: 1 {cfg} instance x {L} FullADMM iterations (+ setup) per step "
              f"(of the {args.batch_per_gpu} instances/GPU of the workload), 1 host thread")
    from gen import make_instance
    shape, _ = make_instance(cfg, 0)
    E, _, E_B = workload_shape_stats(shape)
    config = workload_config(args, world, shape, E, E_B)
    config["sample"] = sample
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (gen/, seeded PCG64)",
            "config": config,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": sample},
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
    from paper_2603_02642_b200.dist import instance_range, max_over_ranks, batch_stats
    from gen import make_batch

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    B, L = args.batch_per_gpu, args.iters
    first, count = instance_range(rank, world, B)
    shape, batch = make_batch(args.workload, count, start=first)
    E, E_s, E_B = workload_shape_stats(shape)
    data_dev = nrto.to_tensors(batch, device=dev)
    solver = nrto.InnerSolver(shape, data_dev, max_iter=L, fixed_iters=1)
    out = nrto.alloc_out(shape, B, solver.E, device=dev, full=True)
    out.pop("nu"); out.pop("lam_nu")          # optional ragged outputs not requested
    stream = torch.cuda.current_stream()

    def step():
        solver.refresh(data_dev)
        solver.solve(nrto.NRTO_FULLADMM, out=out)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    solver.profile(True)
    solver.profile_read()                      # clear
    solver.pass_bytes()                        # clear the pass byte counter
    l0 = solver.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = solver.launches() - l0
    prof = solver.profile_read()
    moved = solver.pass_bytes()                # algorithmic bytes of k_fa_tma in the timed steps
    solver.profile(False)
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_max = max_over_ranks(ms, device=dev)
    value = world * B * L / (ms_max / 1000.0)

    # ---- end to end through the C ABI with HOST buffers (H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        data_host = nrto.to_tensors(batch, device="cpu", pinned=True)
        out_h = nrto.alloc_out(shape, B, solver.E, device="cpu", pinned=True, full=True)
        out_h.pop("nu"); out_h.pop("lam_nu")
        h2d = sum(v.numel() * v.element_size() for v in data_host.values())
        d2h = sum(v.numel() * v.element_size() for v in out_h.values())

        def step_e2e():
            solver.refresh(data_host, memory=nrto.NRTO_MEM_HOST)
            solver.solve(nrto.NRTO_FULLADMM, out=out_h, memory=nrto.NRTO_MEM_HOST)

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
        e2e = {"value": world * B * L / (ems / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "sl_iteration_wall_clock_ms": ems}

    # secondary line: the NRTO-DR engine on its own config (c2 quadcopter, one
    # instance, 40 NRTO-ADMM x 100 DR iterations, fixed) -- latency-bound, reported
    # as DR iterations/s (S3-S8 per DR iteration) and NRTO-ADMM iterations/s
    dr = None
    if not args.no_dr and rank == 0:
        from gen import make_instance
        from gen.problems import stack_instances
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

    # single-instance lines of the other configs (latency-bound; CUDA-graph replay of
    # the fixed-iteration loop): c1 unicycle (both engines), c3 Franka FullADMM
    singles = None
    if not args.no_dr and rank == 0:
        from gen import make_instance
        from gen.problems import stack_instances
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

    # batch-wide residual statistics over NVLink (the only collective)
    max_rp, n_unconv, any_div = batch_stats(out["r_p"], out["status"], device=dev)

    if rank != 0:
        return
    peak, peak_kind = load_peaks()
    # roofline of k_fa_tma: algorithmic bytes = b_hat + b of every state-cone
    # block, y^{l-1} of cones with s^{l-1} != 1, y^l where stored -- counted by the
    # kernel itself (nrto_pass_bytes) -- over its event-timed device time in the steps
    pms, pn = prof["pass"]
    bytes_per_launch = moved / pn if pn else None
    achieved = moved / (pms / 1000.0) / 1e9 if pms else None
    traffic = None
    tf = os.path.join(ROOT, "profiles", "pass_traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            if tj.get("batch") == B and tj.get("iters") == L:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            pass
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v1, dt = cpu_oracle_sample(args.workload, L, 1, seed0=0)
        cpu = {"value": v1, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"1 {args.workload} instance x {L} FullADMM iterations incl. setup "
                         f"({dt:.1f} s, 1 host thread)"}
    kernel_ms = {k: (v[0] / args.steps) for k, v in prof.items()}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen/, seeded PCG64; no datasets or trained weights)",
        "config": workload_config(args, world, shape, E, E_B),
        "soc_projections_per_s": value * shape.n_g,
        "cone_elements_per_s": value * E,
        "sl_iteration_wall_clock_ms": (e2e or {}).get("sl_iteration_wall_clock_ms"),
        "kernel_ms_per_step": kernel_ms,
        "kernel_ms_note": ("CUDA-event time per kernel class on its own stream; qp (low-priority "
                           "stream) and ctrl (second high-priority stream) run concurrently with "
                           "pass / adjoint / gain, so the classes overlap and do not add up to the step"),
        "roofline": {"bound": "hbm", "kernel": "k_fa_tma: fused state-cone pass (S3 forward map + "
                                                "S4 SOC norms + S5 state update)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": bytes_per_launch},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "dr_engine": dr,
        "single_instance": singles,
        "residuals": {"max_r_p": max_rp, "unconverged_instances": n_unconv,
                      "any_diverged": any_div},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
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
