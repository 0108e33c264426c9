#!/bin/bash
# A/B of the owner/mirror split Philox draws (default build) against the
# per-pair draws (lib/p0, -DMPPI_TC_PHX4=0) + the bit-identity tests.
mkdir -p gpurun_out
rm -f gpurun_out/libvariants.log
CFGS='[["c1",16384,{}],["c4",11264,{}],["c4",24576,{}],["c4",8192,{}]]' bash tools/gpu_libvariants.sh p0
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "regenerated_eps or split_kernel or pair_kernel or full_iteration_parity_c1 or philox or tail_grid" > gpurun_out/phx4_test.log 2>&1; echo "rc=$?" >> gpurun_out/phx4_test.log
tail -3 gpurun_out/phx4_test.log
