// ws_launch.hpp — launchers of the warp-specialised fp32 rollout kernel
// (rollout_ws.cuh), compiled in their own translation units (ws_h32.cu,
// ws_h64.cu) so the per-(H, L, noise) instantiations build in parallel.
#pragma once

#include <cuda_runtime.h>

#include "model.cuh"
#include "rollout.cuh"

namespace mppi_host {

cudaError_t launch_rollout_ws_h32(const mppi_dev::RolloutArgs<float>& a, const mppi_dev::WeightHolder<float, 32>& w,
                                  int mode, int L, bool smem_weights, dim3 grid, size_t smem, cudaStream_t stream);
cudaError_t launch_rollout_ws_h64(const mppi_dev::RolloutArgs<float>& a, const mppi_dev::WeightHolder<float, 64>& w,
                                  int mode, int L, bool smem_weights, dim3 grid, size_t smem, cudaStream_t stream);

}  // namespace mppi_host
