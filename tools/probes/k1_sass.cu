// SASS probe: one instantiation of the tensor-core rollout kernel (c1's
// variant), for checking the instruction mix with cuobjdump without building
// the whole library.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -cubin \
//   -I paper_1707_02342_b200/csrc -o /tmp/k1.cubin tools/probes/k1_sass.cu
#include "rollout_tc.cuh"
template __global__ void mppi_dev::rollout_tc_kernel<32, 1, 4, mppi_dev::kPhilox, false, true, false>(
    const __grid_constant__ mppi_dev::RolloutArgs<float>, const uint32_t* __restrict__,
    const __grid_constant__ mppi_dev::TailArgs);
