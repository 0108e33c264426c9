#!/bin/bash
# A/B of the split K1's two-steps-ahead L2 costmap prefetch (default build)
# against no prefetch (lib/p0, -DMPPI_SPLIT_PF=0) + the split bit-identity tests.
mkdir -p gpurun_out
rm -f gpurun_out/libvariants.log
CFGS='[["c0",1920,{}],["c4",4096,{}],["c4",1024,{}]]' bash tools/gpu_libvariants.sh p0
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "split_kernel" > gpurun_out/pf_test.log 2>&1; echo "rc=$?" >> gpurun_out/pf_test.log
tail -2 gpurun_out/pf_test.log
