#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2e}
python paper_2603_02642_b200/build.py > gpurun_out/build_${TAG}.log 2>&1
timeout 150 python scripts/debug_general.py > gpurun_out/dbg_general_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qp_scan -s 2 -c 1 \
   -o gpurun_out/prof_scan_${TAG} python scripts/single_once.py c3 0 4 > gpurun_out/ncu_scan_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dr_loop -s 1 -c 1 \
   -o gpurun_out/prof_drloop_${TAG} python scripts/single_once.py c2 1 2 > gpurun_out/ncu_drloop_${TAG}.log 2>&1
cat gpurun_out/dbg_general_${TAG}.log
