#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_tc.log
timeout 900 python tools/sweep.py tc > gpurun_out/sweep_tc.log 2>&1
tail -n 25 gpurun_out/pytest_gpu_tc.log; cat gpurun_out/sweep_tc.log
