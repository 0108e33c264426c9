// tc_dispatch.cu — host dispatch of the tensor-core rollout over (H, noise
// mode): each (H, mode) set of kernel instantiations lives in its own
// translation unit (tc_h{32,64}_{phx,ref,inj}.cu) so they compile in
// parallel; plus the fixed-group merge launcher (group.cuh).
#include <algorithm>

#include "tail.cuh"
#include "group.cuh"
#include "ws_launch.hpp"

namespace mppi_host {

namespace tc_detail {
int g_tc_last_pair = 0;
}

template <int H>
cudaError_t launch_rollout_tc(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, int mode, int mt,
                              int n_chunks, int ctrls, cudaStream_t stream) {
  switch (mode) {
    case mppi_dev::kInjected: return tc_detail::by_stab<H, mppi_dev::kInjected>(a, frag, mt, n_chunks, ctrls, stream);
    case mppi_dev::kRefSplitmix: return tc_detail::by_stab<H, mppi_dev::kRefSplitmix>(a, frag, mt, n_chunks, ctrls, stream);
    default: return tc_detail::by_stab<H, mppi_dev::kPhilox>(a, frag, mt, n_chunks, ctrls, stream);
  }
}

template cudaError_t launch_rollout_tc<32>(const mppi_dev::RolloutArgs<float>&, const uint32_t*, int, int, int, int,
                                           cudaStream_t);
template cudaError_t launch_rollout_tc<64>(const mppi_dev::RolloutArgs<float>&, const uint32_t*, int, int, int, int,
                                           cudaStream_t);

cudaError_t launch_group_merge(const mppi_dev::Acc* partials, long long partials_ctrl_stride, int n_chunks,
                               int n_groups, int g0, int n_local, int stride, double lambda, mppi_dev::Acc* groups,
                               long long groups_ctrl_stride, int ctrls, bool pdl, cudaStream_t stream) {
  if (n_local <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_local, (stride + mppi_dev::kGroupElems - 1) / mppi_dev::kGroupElems, ctrls);
  cfg.blockDim = dim3(mppi_dev::kGroupBlock);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, mppi_dev::group_merge_kernel<>, partials, partials_ctrl_stride, n_chunks, n_groups,
                            g0, stride, lambda, groups, groups_ctrl_stride);
}

}  // namespace mppi_host
