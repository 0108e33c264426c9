#!/bin/bash
# The GPU tests and tools/sanitize_target.py on the debug build with device-side
# index checks (-DMPPI_DEVICE_CHECKS: every global write of K1, the group merge
# and the tail traps on an out-of-range index).  compute-sanitizer is closed on
# this GPU pool.  Build first:  make -C paper_1707_02342_b200 dchk
mkdir -p gpurun_out
L=paper_1707_02342_b200/lib
cp $L/libmppi_gpu.so /tmp/libmppi_gpu_default.so
cp $L/dchk/libmppi_gpu.so $L/libmppi_gpu.so
strings $L/libmppi_gpu.so | grep -c "MPPI_DCHECK failed" > gpurun_out/device_checks.log
timeout 900 python tools/sanitize_target.py >> gpurun_out/device_checks.log 2>&1; echo "sanitize_target rc=$?" >> gpurun_out/device_checks.log
timeout 1500 python -m pytest tests -m gpu -q >> gpurun_out/device_checks.log 2>&1; echo "pytest rc=$?" >> gpurun_out/device_checks.log
cp /tmp/libmppi_gpu_default.so $L/libmppi_gpu.so
tail -8 gpurun_out/device_checks.log
