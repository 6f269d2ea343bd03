#!/bin/bash
# ncu --set full of the dominant kernel in the exact bench launch configuration (B=512),
# plus the serialised launch list of one bench step.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python paper_2603_02642_b200/build.py > gpurun_out/build.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fa_tma -s 10 -c 1 \
   -o gpurun_out/prof_tma512 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
   > gpurun_out/ncu_tma512.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 420 --csv \
   --log-file gpurun_out/launches512.csv python bench.py --steps 1 --warmup 3 --no-e2e \
   --no-cpu-baseline > gpurun_out/ncu_launch512.log 2>&1
ls -la gpurun_out | head -30
