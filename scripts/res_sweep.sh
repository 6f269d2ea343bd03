#!/bin/bash
# Sweep of launch-shape knobs of the overlapped loop (probe only).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() { echo "$*" >> gpurun_out/res_sweep.txt; env "$@" timeout 300 python scripts/iter_profile.py 512 ${LS:-5,50} >> gpurun_out/res_sweep.txt 2>&1; }
for cfg in "${@}"; do run $cfg; done
