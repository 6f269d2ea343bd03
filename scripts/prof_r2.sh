#!/bin/bash
# Round-2 profiling pass: bench line, QP phase clocks, ncu launch list of one
# bench-wave solve (B=512, L=50), ncu --set full of the pass and the QP.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2> gpurun_out/bench_${TAG}.err
timeout 300 python scripts/qp_clocks.py 512 > gpurun_out/qpclk_${TAG}.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
   --log-file gpurun_out/launches_${TAG}.csv python scripts/solve_once.py 512 50 > gpurun_out/ncu_list_${TAG}.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_${TAG}.csv > gpurun_out/launches_${TAG}_summary.txt 2>&1
if [ -n "$FULL" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fa_tma|k_qp_sparse" -s 40 -c 4 \
   -o gpurun_out/prof_${TAG} python scripts/solve_once.py 512 50 > gpurun_out/ncu_full_${TAG}.log 2>&1
fi
