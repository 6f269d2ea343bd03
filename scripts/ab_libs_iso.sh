#!/bin/bash
# A/B: bench + isolated (ncu-serialised) pass launch times per library variant
cd "$(dirname "$0")/.."
for f in ablibs/lib_*.so; do
  cp "$f" paper_2603_02642_b200/libnrto.so
  echo "== $f"
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-dr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['kernel_ms_per_step'].items()})"
  timeout 600 ncu --metrics gpu__time_duration.sum -k regex:k_fa_tma --csv --log-file /tmp/iso.csv python scripts/solve_once.py 512 50 10 > /dev/null 2>&1
  python scripts/launch_summary.py /tmp/iso.csv k_fa_tma | sed -n '1p;26,28p'
done
