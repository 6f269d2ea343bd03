#!/bin/bash
# Full round-2 evidence run: GPU tests (per-test timeout), smoke, bench line, launch
# lists (bench-wave solve, single instances), ncu --set full of the top kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2o}
python paper_2603_02642_b200/build.py > gpurun_out/build_${TAG}.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread --durations=15 > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
if [ -z "$NOBENCH" ]; then
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2> gpurun_out/bench_${TAG}.err
echo "bench exit $?" >> gpurun_out/bench_${TAG}.err
fi
if [ -n "$PROF" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
   --log-file gpurun_out/launches_${TAG}.csv python scripts/solve_once.py 512 50 > gpurun_out/ncu_list_${TAG}.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_${TAG}.csv > gpurun_out/launches_${TAG}_summary.txt 2>&1
TAG=${TAG} bash scripts/single_profile.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fa_tma|k_qp_sparse" -s 40 -c 2 \
   -o gpurun_out/prof_batch_${TAG} python scripts/solve_once.py 512 50 > gpurun_out/ncu_full_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dr_loop -s 1 -c 1 \
   -o gpurun_out/prof_drloop_${TAG} python scripts/single_once.py c2 1 2 > gpurun_out/ncu_drloop_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qp_scan -s 2 -c 1 \
   -o gpurun_out/prof_scan_${TAG} python scripts/single_once.py c3 0 4 > gpurun_out/ncu_scan_${TAG}.log 2>&1
fi
tail -25 gpurun_out/pytest_${TAG}.log; tail -2 gpurun_out/smoke_${TAG}.log
