// tc_dispatch.cu — host dispatch of the tensor-core rollout over (H, noise
// mode): each (H, mode) set of kernel instantiations lives in its own
// translation unit (tc_h{32,64}_{phx,ref,inj}.cu) so they compile in
// parallel; plus the element-parallel merge launcher.
#include <algorithm>

#include "tail.cuh"
#include "ws_launch.hpp"

namespace mppi_host {

namespace tc_detail {
int g_tc_last_pair = 0;
}

template <int H>
cudaError_t launch_rollout_tc(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag,
                              const mppi_dev::TailArgs& tail, int mode, int mt, int n_chunks, int ctrls,
                              cudaStream_t stream) {
  switch (mode) {
    case mppi_dev::kInjected: return tc_detail::by_stab<H, mppi_dev::kInjected>(a, frag, tail, mt, n_chunks, ctrls, stream);
    case mppi_dev::kRefSplitmix: return tc_detail::by_stab<H, mppi_dev::kRefSplitmix>(a, frag, tail, mt, n_chunks, ctrls, stream);
    default: return tc_detail::by_stab<H, mppi_dev::kPhilox>(a, frag, tail, mt, n_chunks, ctrls, stream);
  }
}

template cudaError_t launch_rollout_tc<32>(const mppi_dev::RolloutArgs<float>&, const uint32_t*,
                                           const mppi_dev::TailArgs&, int, int, int, int, cudaStream_t);
template cudaError_t launch_rollout_tc<64>(const mppi_dev::RolloutArgs<float>&, const uint32_t*,
                                           const mppi_dev::TailArgs&, int, int, int, int, cudaStream_t);

cudaError_t launch_merge_elements(const mppi_dev::Acc* partials, int n, int stride, long long ctrl_stride,
                                  double lambda, mppi_dev::Acc* merged, int ctrls, cudaStream_t stream) {
  const size_t smem = mppi_dev::merge_smem_bytes(n);
  auto kern = mppi_dev::merge_elements_kernel<>;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const dim3 grid(std::min(stride, 296), ctrls);
  kern<<<grid, mppi_dev::kMergeBlock, smem, stream>>>(partials, n, stride, ctrl_stride, lambda, merged);
  return cudaGetLastError();
}

}  // namespace mppi_host
