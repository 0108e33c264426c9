// tc_h32.cu — instantiations and launcher of the tensor-core rollout kernel
// (rollout_tc.cuh), H = 32, fp32 path.
#include "rollout_tc.cuh"
#include "ws_launch.hpp"

#include <cstdlib>

namespace mppi_host {

namespace {
constexpr int kTcWarps = 4;  // warps (chunks) per CTA

template <int MT, int Mode, bool STAB, bool STORE, bool TRACE>
cudaError_t go_trace(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, const mppi_dev::TailArgs& tail,
                     int n_chunks, int ctrls, size_t smem, cudaStream_t stream) {
  auto kern = mppi_dev::rollout_tc_kernel<MT, kTcWarps, Mode, STAB, STORE, TRACE>;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const dim3 grid((n_chunks + kTcWarps - 1) / kTcWarps, ctrls);
  kern<<<grid, 32 * kTcWarps, smem, stream>>>(a, frag, tail);
  return cudaGetLastError();
}
// the per-step state trace (parity: mppi_gpu_rollout_states) is its own instantiation
template <int MT, int Mode, bool STAB, bool STORE>
cudaError_t go_store(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, const mppi_dev::TailArgs& tail,
                     int n_chunks, int ctrls, size_t smem, cudaStream_t stream) {
  if (a.trace_states) return go_trace<MT, Mode, STAB, STORE, true>(a, frag, tail, n_chunks, ctrls, smem, stream);
  return go_trace<MT, Mode, STAB, STORE, false>(a, frag, tail, n_chunks, ctrls, smem, stream);
}
// eps' stays on chip when the grid still fits one wave with that footprint
// (2 CTAs of 4 warps per SM); larger launches regenerate it from the counters.
template <int MT, int Mode, bool STAB>
cudaError_t go(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, const mppi_dev::TailArgs& tail,
               int n_chunks, int ctrls, cudaStream_t stream) {
  const size_t plan_bytes = (sizeof(float) * (2 * a.T + 2) + 15) & ~size_t(15);
  const size_t base = plan_bytes + sizeof(double) * kTcWarps * 2 * mppi_dev::kTcTB * mppi_dev::kTcRedStride;
  const size_t eps_bytes = sizeof(float2) * kTcWarps * a.T * 16 * MT;
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const long long ctas = static_cast<long long>((n_chunks + kTcWarps - 1) / kTcWarps) * ctrls;
  const bool store = std::getenv("MPPI_TC_STORE") ? std::atoi(std::getenv("MPPI_TC_STORE")) != 0
                                                   : (base + eps_bytes <= 110 * 1024 && ctas <= 2LL * sms);
  if (store) return go_store<MT, Mode, STAB, true>(a, frag, tail, n_chunks, ctrls, base + eps_bytes, stream);
  return go_store<MT, Mode, STAB, false>(a, frag, tail, n_chunks, ctrls, base, stream);
}
template <int Mode, bool STAB>
cudaError_t by_mt(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, const mppi_dev::TailArgs& tail, int mt,
                  int n_chunks, int ctrls, cudaStream_t stream) {
  return mt == 1 ? go<1, Mode, STAB>(a, frag, tail, n_chunks, ctrls, stream)
                 : go<2, Mode, STAB>(a, frag, tail, n_chunks, ctrls, stream);
}
template <int Mode>
cudaError_t by_stab(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, const mppi_dev::TailArgs& tail,
                    int mt, int n_chunks, int ctrls, cudaStream_t stream) {
  // the side-slip term (atan) is compiled in only when its weight is nonzero
  return a.sys.cost.alpha_stab != 0.f ? by_mt<Mode, true>(a, frag, tail, mt, n_chunks, ctrls, stream)
                                      : by_mt<Mode, false>(a, frag, tail, mt, n_chunks, ctrls, stream);
}
}  // namespace

cudaError_t launch_rollout_tc_h32(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag,
                                  const mppi_dev::TailArgs& tail, int mode, int mt, int n_chunks, int ctrls,
                                  cudaStream_t stream) {
  switch (mode) {
    case mppi_dev::kInjected: return by_stab<mppi_dev::kInjected>(a, frag, tail, mt, n_chunks, ctrls, stream);
    case mppi_dev::kRefSplitmix: return by_stab<mppi_dev::kRefSplitmix>(a, frag, tail, mt, n_chunks, ctrls, stream);
    default: return by_stab<mppi_dev::kPhilox>(a, frag, tail, mt, n_chunks, ctrls, stream);
  }
}

cudaError_t launch_tail_final(const mppi_dev::TailArgs& tail, int T, int partial_stride, double lambda, int ctrls,
                              cudaStream_t stream) {
  const size_t smem = sizeof(double) * 32 * mppi_dev::kRedStride;
  mppi_dev::tail_final_kernel<><<<ctrls, 32, smem, stream>>>(tail, T, partial_stride, lambda);
  return cudaGetLastError();
}

}  // namespace mppi_host
