// ws_h32.cu — instantiations of rollout_ws_kernel for H = 32.
#include "rollout_ws.cuh"
#include "ws_launch.hpp"

namespace mppi_host {

namespace {
template <int L, int Mode>
cudaError_t go(const mppi_dev::RolloutArgs<float>& a, const mppi_dev::WeightHolder<float, 32>& w, dim3 grid,
               size_t smem, cudaStream_t stream) {
  auto kern = mppi_dev::rollout_ws_kernel<32, L, Mode>;
  if (smem > 32 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  kern<<<grid, 32 * L, smem, stream>>>(a, w);
  return cudaGetLastError();
}
template <int Mode>
cudaError_t by_l(const mppi_dev::RolloutArgs<float>& a, const mppi_dev::WeightHolder<float, 32>& w, int L, dim3 grid,
                 size_t smem, cudaStream_t stream) {
  switch (L) {
    case 1: return go<1, Mode>(a, w, grid, smem, stream);
    case 2: return go<2, Mode>(a, w, grid, smem, stream);
    case 4: return go<4, Mode>(a, w, grid, smem, stream);
    default: return go<8, Mode>(a, w, grid, smem, stream);
  }
}
}  // namespace

cudaError_t launch_rollout_ws_h32(const mppi_dev::RolloutArgs<float>& a, const mppi_dev::WeightHolder<float, 32>& w,
                                  int mode, int L, dim3 grid, size_t smem, cudaStream_t stream) {
  switch (mode) {
    case mppi_dev::kInjected: return by_l<mppi_dev::kInjected>(a, w, L, grid, smem, stream);
    case mppi_dev::kRefSplitmix: return by_l<mppi_dev::kRefSplitmix>(a, w, L, grid, smem, stream);
    default: return by_l<mppi_dev::kPhilox>(a, w, L, grid, smem, stream);
  }
}

}  // namespace mppi_host
