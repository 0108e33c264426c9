#!/bin/bash
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c1b.csv python tools/ncu_target.py c1 0 6 > /dev/null 2>&1
bash tools/gpu_ncu_full.sh tc1v3 c1 0
