#!/bin/bash
# Sweep c0/c1/c4 over alternative library builds (paper_1707_02342_b200/lib/<v>/libmppi_gpu.so),
# swapping each in for the default one on the (scratch) GPU-box copy of the repo.
# Usage: bash tools/gpu_libvariants.sh v1 v2 ...   (the default build is measured as "default")
mkdir -p gpurun_out
L=paper_1707_02342_b200/lib
cp $L/libmppi_gpu.so /tmp/libmppi_gpu_default.so
CFGS='[["c1",16384,{}],["c0",1920,{}],["c4",262144,{}],["c2",65536,{}]]'
for v in default "$@"; do
  if [ "$v" = default ]; then cp /tmp/libmppi_gpu_default.so $L/libmppi_gpu.so; else cp $L/$v/libmppi_gpu.so $L/libmppi_gpu.so; fi
  echo "== $v" >> gpurun_out/libvariants.log
  timeout 300 python tools/sweep.py envs "$CFGS" >> gpurun_out/libvariants.log 2>&1
done
cp /tmp/libmppi_gpu_default.so $L/libmppi_gpu.so
