"""Hot source lines / stall reasons / opcode mix of one kernel in an .ncu-rep.
usage: ncu_hot.py report.ncu-rep [nlines]"""
import csv, collections, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(det))); h = r[0]
si, ni, vi, ui = h.index('Section Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
want = {'Duration', 'DRAM Throughput', 'Memory Throughput', 'Executed Ipc Active', 'Issue Slots Busy',
        'Registers Per Thread', 'Achieved Active Warps Per SM', 'Warp Cycles Per Issued Instruction',
        'Eligible Warps Per Scheduler', 'L2 Hit Rate', 'L1/TEX Hit Rate'}
for x in r[1:]:
    if x[ni] in want: print(f"{x[ni]:40s} {x[vi]} {x[ui]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
cur = None; out = []; sass = []; hdr = None
for x in rows:
    if x and x[0] == "File Path": cur = x[1].split('/')[-1]; continue
    if x and x[0] == "Line No": hdr = x; continue
    if hdr and len(x) > 8:
        try:
            if x[0] not in ("",) and x[2] == "-": out.append((int(x[7]), int(x[4]), cur, x[0], x[1][:90]))
            elif x[0] == "" and x[2] != "-": sass.append(x)
        except ValueError: pass
tot = sum(o[0] for o in out); tots = sum(o[1] for o in out)
print(f"instructions {tot/1e6:.1f}M  samples {tots}")
for o in sorted(out, key=lambda o: -o[1])[:N]:
    print(f"{o[0]/1e6:8.1f}M {100*o[1]/max(tots,1):5.1f}% {o[2]}:{o[3]:>4} {o[4]}")
if hdr:
    sc = [i for i, c in enumerate(hdr) if c.startswith('stall_') and 'Not Issued' not in c]
    agg = collections.Counter()
    op = collections.Counter()
    for x in sass:
        for i in sc:
            try: agg[hdr[i]] += int(x[i] or 0)
            except ValueError: pass
        t = x[3].split()
        if t:
            o = t[1] if t[0].startswith('@') and len(t) > 1 else t[0]
            try: op[o.split('.')[0]] += int(x[7])
            except ValueError: pass
    print("stalls:", agg.most_common(10))
    print("opcodes:", [(k, round(v / 1e6, 1)) for k, v in op.most_common(16)])
