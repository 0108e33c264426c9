// SASS probe: the warp-pair tensor-core rollout (rollout_tc_pair.cuh), c1's variant.
#include "rollout_tc_pair.cuh"
template __global__ void mppi_dev::rollout_tc_pair_kernel<1, mppi_dev::kPhilox, false>(
    const __grid_constant__ mppi_dev::RolloutArgs<float>, const uint32_t* __restrict__);
