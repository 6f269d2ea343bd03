#!/bin/bash
# QP compile-time variant probe: build each variant, per-phase QP clocks + solve timing.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out/qp_variants_${TAG:-x}.txt
for v in "$@"; do
  python paper_2603_02642_b200/build.py $v > gpurun_out/build_var.log 2>&1 || { echo "build failed: $v" >> $OUT; continue; }
  echo "=== variant: $v" >> $OUT
  timeout 300 python scripts/qp_clocks.py 512 >> $OUT 2>&1
  timeout 300 python scripts/solve_time.py 512 50 >> $OUT 2>&1
  timeout 300 python scripts/solve_time.py 1 40 >> $OUT 2>&1
done
python paper_2603_02642_b200/build.py > gpurun_out/build.log 2>&1
