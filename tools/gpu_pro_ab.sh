#!/bin/bash
# A/B of the eps'-prologue build (lib/pro, -DMPPI_TC_PRO=1) of the single-warp
# K1 against the default build, then its bit-identity tests.
mkdir -p gpurun_out
CFGS='[["c1",16384,{}],["c4",6144,{"MPPI_TC_SPLIT":"0"}],["c4",8192,{}],["c4",11264,{}],["c4",12288,{}]]' bash tools/gpu_libvariants.sh pro
L=paper_1707_02342_b200/lib
cp $L/libmppi_gpu.so /tmp/keep.so; cp $L/pro/libmppi_gpu.so $L/libmppi_gpu.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "regenerated_eps or split_kernel or pair_kernel or full_iteration_parity_c1" > gpurun_out/pro_test.log 2>&1; echo "rc=$?" >> gpurun_out/pro_test.log
cp /tmp/keep.so $L/libmppi_gpu.so
tail -3 gpurun_out/pro_test.log
