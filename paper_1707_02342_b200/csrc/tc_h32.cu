// tc_h32.cu — the tensor-core rollout kernel and tail for H = 32 (fp32 path),
// plus the element-parallel merge kernel launcher.
#define TC_H 32
#include "tc_launch.cuh"

namespace mppi_host {

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
