#!/bin/bash
# Quick timing pass: config sweep (iteration + K1 ms) and the ncu launch list of a short c1 bench.
# Usage (under gpurun): bash tools/gpu_quick.sh TAG
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python tools/sweep.py envs '[["c0",1920,{}],["c1",16384,{}],["c2",65536,{}],["c4",1024,{}],["c4",65536,{}],["c4",262144,{}],["c4",1048576,{}]]' > gpurun_out/sweep_$TAG.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launch_$TAG.log 2>&1
cat gpurun_out/sweep_$TAG.jsonl
python tools/launch_summary.py gpurun_out/launches_$TAG.csv
