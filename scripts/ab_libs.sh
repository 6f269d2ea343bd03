#!/bin/bash
# A/B the bench (and isolated QP phase clocks) across prebuilt library variants ablibs/lib_*.so
cd "$(dirname "$0")/.."
for f in ablibs/lib_*.so; do
  cp "$f" paper_2603_02642_b200/libnrto.so
  echo "== $f"
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['kernel_ms_per_step'].items()})"
  if [ -n "$QPCLK" ]; then
    ncu --metrics gpu__time_duration.sum -k regex:k_qp_sparse --csv --log-file /tmp/qpiso.csv python scripts/qp_clocks.py 512 | grep -v "^==PROF" | grep "it1"
  fi
done
