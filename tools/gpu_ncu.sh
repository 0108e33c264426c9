#!/bin/bash
# ncu evidence for the bench workload (run under gpurun, one GPU):
#  1. the launch list of a short bench run (per-launch durations, serialised)
#  2. one `--set full` capture of the rollout kernel (K1) at the bench config
# Usage: bash tools/gpu_ncu.sh [tag] [cfg] [K]
TAG=${1:-r01}; CFG=${2:-c1}; K=${3:-0}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain_$TAG.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout -s 3 -c 1 \
  -o gpurun_out/k1_${CFG}_$TAG -f python tools/ncu_target.py $CFG $K 5 > gpurun_out/ncu_full_$TAG.log 2>&1
ncu -i gpurun_out/k1_${CFG}_$TAG.ncu-rep --page raw --csv > gpurun_out/k1_${CFG}_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/k1_${CFG}_$TAG.ncu-rep --page details --csv > gpurun_out/k1_${CFG}_${TAG}_details.csv 2>/dev/null
ncu -i gpurun_out/k1_${CFG}_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/k1_${CFG}_${TAG}_source.csv 2>/dev/null
ls -la gpurun_out
