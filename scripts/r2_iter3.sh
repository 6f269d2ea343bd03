#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2f}
python paper_2603_02642_b200/build.py > gpurun_out/build_${TAG}.log 2>&1
timeout 900 python -m pytest tests/test_gpu_persist.py tests/test_gpu_general.py tests/test_gpu_parity.py -q --timeout 240 -k "dr or DR or persist or scan or general" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
for spec in "c1 1 4" "c2 1 4"; do
  set -- $spec
  n="${1}_e${2}"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
     --log-file gpurun_out/launch_${TAG}_${n}.csv python scripts/single_once.py $1 $2 $3 > gpurun_out/ncu_${TAG}_${n}.log 2>&1
  python scripts/summarize_launches.py gpurun_out/launch_${TAG}_${n}.csv > gpurun_out/launch_${TAG}_${n}_summary.txt 2>&1
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-conv --no-c4 > gpurun_out/bench_${TAG}.log 2> gpurun_out/bench_${TAG}.err
tail -3 gpurun_out/pytest_${TAG}.log; head -3 gpurun_out/launch_${TAG}_c2_e1_summary.txt
