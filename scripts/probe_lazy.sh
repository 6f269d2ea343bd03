#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/pass_probe.py > gpurun_out/pass_probe.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/solve_launches.csv python scripts/solve_once.py 512 50 10 > gpurun_out/solve_once.log 2>&1
echo "ncu exit $?" >> gpurun_out/solve_once.log
