// umma_launch.cuh — launcher of the tcgen05 / TMEM rollout (rollout_umma.cuh)
// for hidden width UMMA_H; instantiated by umma_h32.cu / umma_h64.cu so the
// two widths build in parallel.
#include "rollout_umma.cuh"
#include "ws_launch.hpp"

#include <cstdlib>

namespace mppi_host {
namespace {

constexpr int H = UMMA_H;
template <int Mode, bool STAB, bool TRACE, int TPC = mppi_dev::umma_tiles_per_cta<H>()>
cudaError_t go_umma(const mppi_dev::RolloutArgs<float>& a, const unsigned char* wimg, int n_chunks, int ctrls,
                    cudaStream_t stream) {
  auto kern = mppi_dev::rollout_umma_kernel<H, Mode, STAB, TRACE, TPC>;
  const size_t smem = mppi_dev::umma_smem_bytes<H, TPC>(a.T);
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
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
// H = 64: two-tile CTAs (one shared weight copy, four tiles per SM instead
// of three) when that fits the grid in one wave and single tiles do not —
// the c2 band (c2 K1 1165 -> 1118 us; larger grids lose with them,
// rollout_umma.cuh).  MPPI_UMMA_TPC2=0 / 1 forces the choice.
bool umma_two_tiles(long long tiles) {
  if constexpr (H != 64 || mppi_dev::umma_tiles_per_cta<H>() != 1) {
    return false;
  } else {
    static const int sms = [] {
      int dev = 0, n = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
      return n;
    }();
    if (const char* e = std::getenv("MPPI_UMMA_TPC2")) return std::atoi(e) != 0;
    const long long one = static_cast<long long>(mppi_dev::umma_min_ctas<H, 1>()) * sms;
    const long long two = 2LL * mppi_dev::umma_min_ctas<H, 2>() * sms;
    return tiles > one && tiles <= two;
  }
}
template <int Mode, bool STAB>
cudaError_t by_trace(const mppi_dev::RolloutArgs<float>& a, const unsigned char* wimg, int n_chunks, int ctrls,
                     cudaStream_t stream) {
  if constexpr (H == 64 && mppi_dev::umma_tiles_per_cta<H>() == 1) {
    if (!a.trace_states && umma_two_tiles(static_cast<long long>(n_chunks) * ctrls))
      return go_umma<Mode, STAB, false, 2>(a, wimg, n_chunks, ctrls, stream);
  }
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
