#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_tc.log
timeout 900 python tools/sweep.py tc > gpurun_out/sweep_tc.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_tc.log 2>&1
tail -n 15 gpurun_out/pytest_gpu_tc.log; cat gpurun_out/sweep_tc.log gpurun_out/bench_tc.log
