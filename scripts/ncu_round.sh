#!/bin/bash
# Round profile set: launch list of one bench step (time + DRAM bytes), full ncu
# captures of the pass and the QP at iteration 20 of a bench-size solve.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python paper_2603_02642_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none --csv --log-file gpurun_out/solve_launches.csv \
   python scripts/solve_once.py 512 50 10 > gpurun_out/solve_once.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fa_tma -s 20 -c 1 \
   -o gpurun_out/prof_pass python scripts/solve_once.py 512 50 10 > gpurun_out/ncu_pass.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qp_sparse -s 20 -c 1 \
   -o gpurun_out/prof_qp python scripts/solve_once.py 512 50 10 > gpurun_out/ncu_qp.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zlist_mma -s 30 -c 1 \
   -o gpurun_out/prof_zlist python scripts/solve_once.py 512 50 10 > gpurun_out/ncu_zlist.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
ls -la gpurun_out | head -40
