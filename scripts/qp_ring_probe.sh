#!/bin/bash
# QP recurrence ring-depth probe: per-phase clocks of one QP CTA in a bench-size solve.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "-DQP_RING=8" "-DQP_RING=16" "-DQP_RING=32" "-DQP_RING=32 -DNRTO_NOOVERLAP"; do
  python paper_2603_02642_b200/build.py $v > gpurun_out/build_var.log 2>&1 || { echo "build failed: $v" >> gpurun_out/qp_ring.txt; continue; }
  echo "variant: $v" >> gpurun_out/qp_ring.txt
  timeout 300 python scripts/qp_clocks.py 512 >> gpurun_out/qp_ring.txt 2>&1
  timeout 300 python scripts/solve_time.py 512 50 >> gpurun_out/qp_ring.txt 2>&1
done
python paper_2603_02642_b200/build.py > gpurun_out/build.log 2>&1
