#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python paper_2603_02642_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${CNT:-800} --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --batch-per-gpu ${B:-512} \
   --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
tail -2 gpurun_out/ncu_bench.log
