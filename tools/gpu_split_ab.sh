#!/bin/bash
# A/B of the sample-split K1 (MPPI_TC_SPLIT=1) against the default K1:
# bit-identity tests, then the config sweep.  Usage: bash tools/gpu_split_ab.sh [CFG_JSON]
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "split_kernel" > gpurun_out/split_test.log 2>&1; echo "rc=$?" >> gpurun_out/split_test.log
CFGS=${1:-'[["c0",1920,{}],["c0",1920,{"MPPI_TC_SPLIT":"1"}],["c4",1024,{}],["c4",1024,{"MPPI_TC_SPLIT":"1"}],["c4",4096,{}],["c4",4096,{"MPPI_TC_SPLIT":"1"}]]'}
timeout 900 python tools/sweep.py envs "$CFGS" > gpurun_out/split_sweep.jsonl 2>&1
tail -3 gpurun_out/split_test.log; cut -c1-330 gpurun_out/split_sweep.jsonl
