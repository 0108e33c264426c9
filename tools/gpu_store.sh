#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_tc.log 2>&1; tail -3 gpurun_out/pytest_gpu_tc.log
python tools/sweep.py envs '[["c1",16384,{"MPPI_TC_STORE":"0"}],["c1",16384,{"MPPI_TC_STORE":"1"}],["c0",1920,{"MPPI_TC_STORE":"0"}],["c0",1920,{"MPPI_TC_STORE":"1"}],["c1",16384,{"MPPI_TC_MT":"2","MPPI_TC_STORE":"1"}]]' 2>&1 | cut -c1-400
