#!/bin/bash
# DR (c2) launch-knob sweep (probe only)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in "$@"; do echo "$cfg" >> gpurun_out/dr_sweep.txt; env $cfg timeout 300 python scripts/dr_profile.py 40 >> gpurun_out/dr_sweep.txt 2>&1; done
