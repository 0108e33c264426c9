#!/bin/bash
# One `ncu --set full` capture of one kernel at a config (default: K1).
# Usage: bash tools/gpu_ncu_full.sh TAG CFG [K] [KERNEL_REGEX]
#   extra environment (e.g. MPPI_KERNEL=umma) is passed through to the target.
TAG=${1:-r02}; CFG=${2:-c1}; K=${3:-0}; KR=${4:-rollout}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python tools/ncu_target.py $CFG $K 2 > $O/plain_${CFG}.log 2>&1 || { cat $O/plain_${CFG}.log; exit 1; }
N=$O/ncu_full_${KR//[^a-z_]/}_${CFG}_K$K
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KR -s 2 -c 1 \
  -o $N -f python tools/ncu_target.py $CFG $K 4 > $N.log 2>&1
ncu -i $N.ncu-rep --page raw --csv > ${N}_raw.csv 2>&1
ncu -i $N.ncu-rep --page details --csv > ${N}_details.csv 2>&1
ncu -i $N.ncu-rep --page source --csv --print-source sass > ${N}_source.csv 2>&1
tail -3 $N.log
