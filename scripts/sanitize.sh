#!/bin/bash
# compute-sanitizer over every kernel path (tiny configs); logs in gpurun_out/sanitize_*.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export NRTO_GRAPH=${NRTO_GRAPH:-1}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_cases.py \
    > gpurun_out/sanitize_${tool}.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${tool}.log
done
