#!/bin/bash
# Round-2 re-entry check: GPU tests, smoke, bench line, launch list of one bench solve.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2b}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
python paper_2603_02642_b200/build.py > gpurun_out/build_${TAG}.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2> gpurun_out/bench_${TAG}.err
echo "bench exit $?" >> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
   --log-file gpurun_out/launches_${TAG}.csv python scripts/solve_once.py 512 50 > gpurun_out/ncu_list_${TAG}.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_${TAG}.csv > gpurun_out/launches_${TAG}_summary.txt 2>&1
tail -3 gpurun_out/pytest_${TAG}.log; tail -2 gpurun_out/smoke_${TAG}.log; tail -1 gpurun_out/bench_${TAG}.log
