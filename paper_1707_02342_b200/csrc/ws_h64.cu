// ws_h64.cu — instantiations of rollout_ws_kernel for H = 64.
#include "rollout_ws.cuh"
#include "ws_launch.hpp"

namespace mppi_host {

namespace {
template <int L, int Mode, bool SW>
cudaError_t go(const mppi_dev::RolloutArgs<float>& a, const mppi_dev::WeightHolder<float, 64>& w, dim3 grid,
               size_t smem, cudaStream_t stream) {
  auto kern = mppi_dev::rollout_ws_kernel<64, L, Mode, SW>;
  if (smem > 32 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  kern<<<grid, 32 * L, smem, stream>>>(a, w);
  return cudaGetLastError();
}
template <int L, int Mode>
cudaError_t by_sw(const mppi_dev::RolloutArgs<float>& a, const mppi_dev::WeightHolder<float, 64>& w, bool sw, dim3 grid,
                  size_t smem, cudaStream_t stream) {
  return sw ? go<L, Mode, true>(a, w, grid, smem, stream) : go<L, Mode, false>(a, w, grid, smem, stream);
}
template <int Mode>
cudaError_t by_l(const mppi_dev::RolloutArgs<float>& a, const mppi_dev::WeightHolder<float, 64>& w, int L, bool sw,
                 dim3 grid, size_t smem, cudaStream_t stream) {
  switch (L) {  // H = 64 always splits the hidden layer over >= 2 warps
    case 1:
    case 2: return by_sw<2, Mode>(a, w, sw, grid, smem, stream);
    case 4: return by_sw<4, Mode>(a, w, sw, grid, smem, stream);
    default: return by_sw<8, Mode>(a, w, sw, grid, smem, stream);
  }
}
}  // namespace

cudaError_t launch_rollout_ws_h64(const mppi_dev::RolloutArgs<float>& a, const mppi_dev::WeightHolder<float, 64>& w,
                                  int mode, int L, bool sw, dim3 grid, size_t smem, cudaStream_t stream) {
  switch (mode) {
    case mppi_dev::kInjected: return by_l<mppi_dev::kInjected>(a, w, L, sw, grid, smem, stream);
    case mppi_dev::kRefSplitmix: return by_l<mppi_dev::kRefSplitmix>(a, w, L, sw, grid, smem, stream);
    default: return by_l<mppi_dev::kPhilox>(a, w, L, sw, grid, smem, stream);
  }
}

}  // namespace mppi_host
