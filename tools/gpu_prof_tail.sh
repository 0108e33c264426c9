#!/bin/bash
mkdir -p gpurun_out
for K in merge_chunks epilogue; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/tail_$K -f python tools/ncu_target.py c1 0 4 > gpurun_out/ncu_tail_$K.log 2>&1
ncu -i gpurun_out/tail_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/tail_${K}_source.csv 2>&1
ncu -i gpurun_out/tail_$K.ncu-rep --page details --csv > gpurun_out/tail_${K}_details.csv 2>&1
done
