#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2d}
python paper_2603_02642_b200/build.py > gpurun_out/build_${TAG}.log 2>&1
timeout 600 python -m pytest tests/test_gpu_persist.py tests/test_gpu_parity.py -q -x --timeout 240 -k "dr or DR or persist or scan" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
timeout 300 python -m pytest tests/test_gpu_general.py -q -x --timeout 120 > gpurun_out/pytest_general_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_general_${TAG}.log
TAG=${TAG} bash scripts/single_profile.sh
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-conv --no-c4 > gpurun_out/bench_${TAG}.log 2> gpurun_out/bench_${TAG}.err
tail -2 gpurun_out/pytest_${TAG}.log
