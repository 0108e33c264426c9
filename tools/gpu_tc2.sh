#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/accuracy.py > gpurun_out/accuracy.log 2>&1
bash tools/gpu_ncu_full.sh tc1 c1 0
MPPI_TC_MT=2 bash tools/gpu_ncu_full.sh tc2 c4 262144
cat gpurun_out/accuracy.log
