"""profiles/pass_traffic.json from an ncu launch list of one bench-size solve
(scripts/solve_once.py under `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum`): mean DRAM bytes per k_fa_tma launch vs the kernel's own
algorithmic byte count.  usage: pass_traffic.py launches.csv solve_once.log B L"""
import csv, json, os, sys
csvf, logf, B, L = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
rows = list(csv.reader(open(csvf)))
h_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[h_i]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
per = {}
for r in rows[h_i + 1:]:
    if 'k_fa_tma' in r[ki]:
        per.setdefault(r[ii], {})[r[mi]] = float(r[vi].replace(',', ''))
dram = [m['dram__bytes_read.sum'] + m['dram__bytes_write.sum'] for m in per.values()]
tms = [m['gpu__time_duration.sum'] for m in per.values()]
alg = None
for line in open(logf):
    if line.startswith("pass bytes per launch"):
        alg = float(line.split(":")[1])
out = {"batch": B, "iters": L, "launches": len(dram),
       "dram_bytes_per_launch": sum(dram) / len(dram),
       "algorithmic_bytes_per_launch": alg,
       "traffic_over_algorithmic": (sum(dram) / len(dram)) / alg if alg else None,
       "ncu_mean_launch_ms": sum(tms) / len(tms) / 1e6,
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (serialised, cold) of "
                 "scripts/solve_once.py %d %d" % (B, L)}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
json.dump(out, open(os.path.join(root, "profiles", "pass_traffic.json"), "w"), indent=1)
print(out)
