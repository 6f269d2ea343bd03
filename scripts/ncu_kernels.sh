#!/bin/bash
# ncu capture of the hot kernels on the bench workload (reduced batch).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python paper_2603_02642_b200/build.py > gpurun_out/build.log 2>&1
B=${B:-128}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --batch-per-gpu $B \
   --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_fa_fused|k_qp_staged}" -s ${SKIP:-40} -c ${CNT:-2} \
   -o gpurun_out/prof_hot python bench.py --steps 1 --warmup 3 --batch-per-gpu $B --no-e2e \
   --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
