"""Key metrics of every kernel in an ncu report (ncu -i ... --page details/raw), as CSV rows."""
import csv, io, subprocess, sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy", "Registers Per Thread",
        "Issue Slots Busy", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum",
       "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
       "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]


def run(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout


for rep in sys.argv[1:]:
    det = list(csv.reader(io.StringIO(run(rep, "details"))))
    h = det[0]
    rows = {}
    for r in det[1:]:
        d = dict(zip(h, r))
        key = (d.get("ID"), d.get("Kernel Name", "")[:60])
        if d.get("Metric Name") in KEYS:
            rows.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"] + " " + d.get("Metric Unit", "")
    raw = list(csv.reader(io.StringIO(run(rep, "raw"))))
    if raw:
        rh = raw[0]
        for r in raw[2:]:
            d = dict(zip(rh, r))
            key = (d.get("ID"), d.get("Kernel Name", "")[:60])
            for k in RAW:
                if k in d and d[k] not in ("", "n/a"):
                    rows.setdefault(key, {})[k] = d[k]
    for (i, name), m in rows.items():
        print(f"{rep.split('/')[-1]},{i},\"{name}\"," + ",".join(f"{k}={m[k]}" for k in KEYS + RAW if k in m))
