#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_tc.log
timeout 600 python tools/accuracy.py > gpurun_out/accuracy.log 2>&1
timeout 900 python tools/sweep.py tc > gpurun_out/sweep_tc.log 2>&1
tail -n 15 gpurun_out/pytest_gpu_tc.log; cat gpurun_out/accuracy.log gpurun_out/sweep_tc.log
