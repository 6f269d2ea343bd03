#!/bin/bash
# ncu --set full of one lazy-y k_fa_tma launch (iteration 20 of a bench-size solve).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fa_tma -s 19 -c 1 \
   -o gpurun_out/prof_tma_lazy python scripts/solve_once.py 512 50 10 > gpurun_out/ncu_tma_lazy.log 2>&1
echo "exit $?" >> gpurun_out/ncu_tma_lazy.log
tail -3 gpurun_out/ncu_tma_lazy.log
