#!/bin/bash
# QP CTA-shape variants (compile-time knobs), each built and timed on the bench batch (probe only).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  python paper_2603_02642_b200/build.py $v > gpurun_out/build_var.log 2>&1 || { echo "build failed: $v" >> gpurun_out/qp_variants.txt; continue; }
  echo "variant: $v" >> gpurun_out/qp_variants.txt
  timeout 300 python scripts/iter_profile.py 512 50 >> gpurun_out/qp_variants.txt 2>&1
done
python paper_2603_02642_b200/build.py > gpurun_out/build.log 2>&1
