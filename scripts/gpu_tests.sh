#!/bin/bash
# GPU tests + smoke + ncu launch list and full capture of the pass kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python paper_2603_02642_b200/build.py > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --batch-per-gpu 128 \
     --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fa_pass -s 20 -c 2 \
     -o gpurun_out/prof_pass python bench.py --steps 1 --warmup 3 --batch-per-gpu 128 --no-e2e \
     --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_adjoint|k_qp" -s 20 -c 2 \
     -o gpurun_out/prof_adj_qp python bench.py --steps 1 --warmup 3 --batch-per-gpu 128 --no-e2e \
     --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
