"""Summarise an ncu --csv launch list (time + dram bytes per kernel).
usage: launch_summary.py launches.csv [kernel-substring-for-per-launch-listing]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr_i]; data = rows[hdr_i + 1:]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
L = collections.OrderedDict()
for r in data:
    L.setdefault((r[ii], r[ki].split('(')[0][:48]), {})[r[mi]] = float(r[vi].replace(',', ''))
tot = collections.defaultdict(lambda: [0.0, 0.0, 0])
for (i, k), m in L.items():
    t = tot[k]; t[0] += m.get('gpu__time_duration.sum', 0) / 1e6
    t[1] += (m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)) / 1e9; t[2] += 1
S = sum(v[0] for v in tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1][0]):
    print(f"{v[0]:9.2f} ms {100*v[0]/S:5.1f}% {v[2]:5d} launches {v[1]:8.2f} GB  {k}")
if len(sys.argv) > 2:
    for (i, k), m in L.items():
        if sys.argv[2] in k:
            t = m['gpu__time_duration.sum'] / 1e6
            b = (m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)) / 1e9
            print(f"  {t:.3f} ms {b:6.2f} GB {b/t:6.0f} GB/s")
