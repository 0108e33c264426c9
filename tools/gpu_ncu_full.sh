#!/bin/bash
# One `ncu --set full` capture of the rollout kernel (K1) at a config.
# Usage: bash tools/gpu_ncu_full.sh TAG CFG [K] [extra env assignments...]
TAG=${1:-r01}; CFG=${2:-c1}; K=${3:-0}
mkdir -p gpurun_out
timeout 300 python tools/ncu_target.py $CFG $K 2 > gpurun_out/plain_$TAG.log 2>&1 || { cat gpurun_out/plain_$TAG.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout -s 1 -c 1 \
  -o gpurun_out/k1_${CFG}_$TAG -f python tools/ncu_target.py $CFG $K 2 > gpurun_out/ncu_full_$TAG.log 2>&1
ncu -i gpurun_out/k1_${CFG}_$TAG.ncu-rep --page raw --csv > gpurun_out/k1_${CFG}_${TAG}_raw.csv 2>&1
ncu -i gpurun_out/k1_${CFG}_$TAG.ncu-rep --page details --csv > gpurun_out/k1_${CFG}_${TAG}_details.csv 2>&1
ncu -i gpurun_out/k1_${CFG}_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/k1_${CFG}_${TAG}_source.csv 2>&1
tail -3 gpurun_out/ncu_full_$TAG.log
