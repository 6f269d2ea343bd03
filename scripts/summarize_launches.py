import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv')))
hdr = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hdr]; data = rows[hdr + 1:]
ki, mi, vi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
agg = collections.defaultdict(list)
for r in data:
    if len(r) > vi and r[mi] == 'gpu__time_duration.sum':
        agg[r[ki].split('(')[0]].append(float(r[vi].replace(',', '')))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:42s} n={len(v):4d} sum={sum(v)/1e6:9.3f} ms  mean={sum(v)/len(v)/1e3:9.1f} us  share={sum(v)/tot*100:5.1f}%")
