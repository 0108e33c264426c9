#!/bin/bash
# tests, a short sweep of the default variants, the bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python tools/sweep.py envs '[["c1",16384,{}],["c0",1920,{}],["c4",262144,{}],["c2",65536,{}]]' 2>&1 | cut -c1-330
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.log 2>&1; cut -c1-900 gpurun_out/bench.log
