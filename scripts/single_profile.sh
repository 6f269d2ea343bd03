#!/bin/bash
# Launch lists (ncu, per-kernel durations) of single-instance solves: c1 FullADMM,
# c1 DR, c2 DR, c3 FullADMM (scripts/single_once.py), summarised per kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-sp}
for spec in "c1 0 20" "c1 1 4" "c2 1 4" "c3 0 10"; do
  set -- $spec
  n="${1}_e${2}"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
     --log-file gpurun_out/launch_${TAG}_${n}.csv python scripts/single_once.py $1 $2 $3 > gpurun_out/ncu_${TAG}_${n}.log 2>&1
  python scripts/summarize_launches.py gpurun_out/launch_${TAG}_${n}.csv > gpurun_out/launch_${TAG}_${n}_summary.txt 2>&1
done
