#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/accuracy.py > gpurun_out/accuracy.log 2>&1
bash tools/gpu_ncu_full.sh tc1v2 c1 0
cat gpurun_out/accuracy.log
