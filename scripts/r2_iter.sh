#!/bin/bash
# Round-2 iteration check: general-path debug, new/affected GPU tests, bench A/B of the batch QP.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2c}
python paper_2603_02642_b200/build.py > gpurun_out/build_${TAG}.log 2>&1
timeout 150 python scripts/debug_general.py > gpurun_out/dbg_general_${TAG}.log 2>&1
echo "exit $?" >> gpurun_out/dbg_general_${TAG}.log
timeout 900 python -m pytest tests/test_gpu_persist.py tests/test_gpu_parity.py -q --timeout 240 ${PYTEST_ARGS} > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
for P in 0 2; do
NRTO_QP_PIPE=$P timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-conv --no-c4 > gpurun_out/bench_${TAG}_pipe$P.log 2> gpurun_out/bench_${TAG}_pipe$P.err
done
tail -3 gpurun_out/pytest_${TAG}.log; tail -3 gpurun_out/dbg_general_${TAG}.log
