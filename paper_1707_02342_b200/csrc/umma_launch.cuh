// umma_launch.cuh — launcher of the tcgen05 / TMEM rollout (rollout_umma.cuh)
// for hidden width UMMA_H; instantiated by umma_h32.cu / umma_h64.cu so the
// two widths build in parallel.
#include "rollout_umma.cuh"
#include "ws_launch.hpp"

namespace mppi_host {
namespace {

constexpr int H = UMMA_H;
template <int Mode, bool STAB, bool TRACE>
cudaError_t go_umma(const mppi_dev::RolloutArgs<float>& a, const unsigned char* wimg, int n_chunks, int ctrls,
                    cudaStream_t stream) {
  auto kern = mppi_dev::rollout_umma_kernel<H, Mode, STAB, TRACE>;
  const size_t smem = mppi_dev::umma_smem_bytes<H>(a.T);
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  constexpr int TPC = mppi_dev::umma_tiles_per_cta<H>();
  cfg.gridDim = dim3((n_chunks + TPC - 1) / TPC, ctrls);
  cfg.blockDim = dim3(mppi_dev::kUmmaThreads * TPC);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a, wimg);
}
template <int Mode, bool STAB>
cudaError_t by_trace(const mppi_dev::RolloutArgs<float>& a, const unsigned char* wimg, int n_chunks, int ctrls,
                     cudaStream_t stream) {
  return a.trace_states ? go_umma<Mode, STAB, true>(a, wimg, n_chunks, ctrls, stream)
                        : go_umma<Mode, STAB, false>(a, wimg, n_chunks, ctrls, stream);
}
template <int Mode>
cudaError_t by_stab_umma(const mppi_dev::RolloutArgs<float>& a, const unsigned char* wimg, int n_chunks, int ctrls,
                         cudaStream_t stream) {
  return a.sys.cost.alpha_stab != 0.f ? by_trace<Mode, true>(a, wimg, n_chunks, ctrls, stream)
                                      : by_trace<Mode, false>(a, wimg, n_chunks, ctrls, stream);
}

}  // namespace

template <>
cudaError_t launch_rollout_umma<UMMA_H>(const mppi_dev::RolloutArgs<float>& a, const unsigned char* wimg, int mode,
                                        int n_chunks, int ctrls, cudaStream_t stream) {
  switch (mode) {
    case mppi_dev::kInjected: return by_stab_umma<mppi_dev::kInjected>(a, wimg, n_chunks, ctrls, stream);
    case mppi_dev::kRefSplitmix: return by_stab_umma<mppi_dev::kRefSplitmix>(a, wimg, n_chunks, ctrls, stream);
    default: return by_stab_umma<mppi_dev::kPhilox>(a, wimg, n_chunks, ctrls, stream);
  }
}

}  // namespace mppi_host
