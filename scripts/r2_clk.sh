#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2g}
python paper_2603_02642_b200/build.py > gpurun_out/build_${TAG}.log 2>&1
timeout 120 python scripts/dr_clocks.py c1 c2 > gpurun_out/drclk_${TAG}.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
   --log-file gpurun_out/launch_${TAG}_c3_e0.csv python scripts/single_once.py c3 0 10 > gpurun_out/ncu_${TAG}_c3.log 2>&1
python scripts/summarize_launches.py gpurun_out/launch_${TAG}_c3_e0.csv > gpurun_out/launch_${TAG}_c3_e0_summary.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_persist.py -q --timeout 240 -k scan > gpurun_out/pytest_${TAG}.log 2>&1
cat gpurun_out/drclk_${TAG}.log; head -4 gpurun_out/launch_${TAG}_c3_e0_summary.txt; tail -2 gpurun_out/pytest_${TAG}.log
