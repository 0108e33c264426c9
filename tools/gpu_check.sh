#!/bin/bash
# One GPU-box pass: gpu tests, smoke, a short bench, the kernel-variant sweep.
# Usage (from the repo root, under gpurun): bash tools/gpu_check.sh [sweep]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ "$1" = "sweep" ]; then timeout 900 python tools/sweep.py > gpurun_out/sweep.log 2>&1; fi
tail -n 30 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log
