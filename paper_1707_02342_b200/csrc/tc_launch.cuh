// tc_launch.cuh — launchers of the tensor-core rollout kernel (rollout_tc.cuh)
// and its tail, templated on the hidden width H; instantiated once per H by
// tc_h32.cu / tc_h64.cu (define TC_H before including) so the variants build
// in parallel.
#include "rollout_tc.cuh"
#include "rollout_tc_pair.cuh"
#include "rollout_tc_split.cuh"
#include "ws_launch.hpp"

#include <algorithm>
#include <cstdlib>

namespace mppi_host {
namespace tc_detail {
constexpr int kTcWarps = 4;  // warps (chunks) per CTA

// K1 launch, as a programmatic dependent of the previous kernel when a.pdl
// (the step graph's x0 fetch: K1 stages its weights and plan while the state
// crosses PCIe, and waits for it in cudaGridDependencySynchronize)
template <class Kern>
cudaError_t launch_k1(Kern kern, dim3 grid, int threads, size_t smem, cudaStream_t stream,
                      const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a, frag);
}

template <int H, int MT, int Mode, bool STAB, bool STORE, bool TRACE, bool PST = false>
cudaError_t go_trace(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, int n_chunks, int ctrls, size_t smem,
                     cudaStream_t stream) {
  auto kern = mppi_dev::rollout_tc_kernel<H, MT, kTcWarps, Mode, STAB, STORE, TRACE, PST>;
  // (static + dynamic shared memory may pass 48 KB even when `smem` does not:
  // the H = 64 kernel holds its layer-2 fragments in 16 KB of static smem)
  {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const dim3 grid((n_chunks + kTcWarps - 1) / kTcWarps, ctrls);
  return launch_k1(kern, grid, 32 * kTcWarps, smem, stream, a, frag);
}
// the per-step state trace (parity: mppi_gpu_rollout_states) is its own instantiation
template <int H, int MT, int Mode, bool STAB, bool STORE>
cudaError_t go_store(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, int n_chunks, int ctrls, size_t smem,
                     cudaStream_t stream) {
  // (a trace is a parity call: no on-chip eps' variant is compiled for it)
  if constexpr (!STORE) {
    if (a.trace_states) return go_trace<H, MT, Mode, STAB, false, true>(a, frag, n_chunks, ctrls, smem, stream);
  }
  // predicated stage stores at <= 1 warp per scheduler (H = 32, MT = 1;
  // rollout_tc_kernel's PST), the C++ branch above that
  if constexpr (H == 32 && MT == 1) {
    static const int schedulers = [] {
      int dev = 0, n = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
      return 4 * n;
    }();
    if (static_cast<long long>(n_chunks) * ctrls <= schedulers)
      return go_trace<H, MT, Mode, STAB, STORE, false, true>(a, frag, n_chunks, ctrls, smem, stream);
  }
  return go_trace<H, MT, Mode, STAB, STORE, false>(a, frag, n_chunks, ctrls, smem, stream);
}
// The warp-pair kernel (rollout_tc_pair.cuh): H = 32, eps' on chip, no trace.
// Opt-in (MPPI_TC_PAIR=1, when its grid is resident at once): it was the
// default at <= 1 chunk per SM (c0: K1 -5 % against the branch-store
// single-warp kernel) until the single-warp kernel's predicated stage stores
// (PST) made that kernel faster there too (c0 K1 89.7 -> 87.2 us); with more
// chunks per SM its barrier handoffs cost more than the shorter per-warp
// chain saves (c1: +24 %, profiles/README.md).
constexpr int kTcPairs = 1;  // warp pairs (chunks) per CTA
template <int Mode, bool STAB>
bool pair_fits(int T, int n_chunks, int ctrls) {
  const char* e = std::getenv("MPPI_TC_PAIR");
  if (!e || std::atoi(e) == 0) return false;
  auto kern = mppi_dev::rollout_tc_pair_kernel<kTcPairs, Mode, STAB>;
  const size_t smem = mppi_dev::tc_pair_smem_bytes(T, kTcPairs);
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 64 * kTcPairs, smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const long long ctas = static_cast<long long>((n_chunks + kTcPairs - 1) / kTcPairs) * ctrls;
  if (!(e && std::atoi(e) == 1) && static_cast<long long>(n_chunks) * ctrls > sms) return false;
  return ctas <= static_cast<long long>(per_sm) * sms;
}
template <int Mode, bool STAB>
cudaError_t go_pair(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, int n_chunks, int ctrls,
                    cudaStream_t stream) {
  auto kern = mppi_dev::rollout_tc_pair_kernel<kTcPairs, Mode, STAB>;
  const size_t smem = mppi_dev::tc_pair_smem_bytes(a.T, kTcPairs);
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const dim3 grid((n_chunks + kTcPairs - 1) / kTcPairs, ctrls);
  g_tc_last_pair = 1;
  return launch_k1(kern, grid, 64 * kTcPairs, smem, stream, a, frag);
}
// The sample-split warp pair (rollout_tc_split.cuh): H = 32, eps' on chip,
// no trace.  Default while its warps fit one per scheduler (2 chunks' worth
// of warps per 4 schedulers of an SM): there a warp's step is its own chain
// and the split halves the MLP part of it (c0 K1 86.8 -> 72.2 us, K = 4096
// 86.6 -> 73.2); with two warps on a scheduler the single-warp kernel's
// lower instruction count per sample wins (K = 6144 +5 %, K = 8192 +5 %,
// profiles/r02d).  MPPI_TC_SPLIT=0 disables it, =1 uses it whenever the
// grid is resident at once.
constexpr int kTcSplitPairs = 1;  // warp pairs (chunks) per CTA
template <int Mode, bool STAB>
bool split_fits(int T, int n_chunks, int ctrls) {
  const char* e = std::getenv("MPPI_TC_SPLIT");
  const int mode = e ? std::atoi(e) : -1;
  if (mode == 0) return false;
  auto kern = mppi_dev::rollout_tc_split_kernel<kTcSplitPairs, Mode, STAB, false>;
  const size_t smem = mppi_dev::tc_split_smem_bytes(T, kTcSplitPairs);
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long ctas = static_cast<long long>((n_chunks + kTcSplitPairs - 1) / kTcSplitPairs) * ctrls;
  if (mode != 1 && 2LL * kTcSplitPairs * ctas > 4LL * sms) return false;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 64 * kTcSplitPairs, smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return ctas <= static_cast<long long>(per_sm) * sms;
}
// The split K1's two-steps-ahead L2 costmap prefetch pays while the samples
// are sparse over the map (K1: c0 73.2 -> 67.1 us, K = 1024 -7.5 %, 2048
// -8 %, 3072 -5.5 %) and costs where they are dense enough to keep the lines
// warm (K = 4096 +4.2 %): on up to kSplitPfChunks chunks per controller
// (profiles/r02d/pf_sweep.jsonl).  MPPI_SPLIT_PF=0 / 1 forces.
constexpr int kSplitPfChunks = 192;
template <int Mode, bool STAB, bool PF>
cudaError_t go_split_pf(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, int n_chunks, int ctrls,
                        cudaStream_t stream) {
  auto kern = mppi_dev::rollout_tc_split_kernel<kTcSplitPairs, Mode, STAB, PF>;
  const size_t smem = mppi_dev::tc_split_smem_bytes(a.T, kTcSplitPairs);
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const dim3 grid((n_chunks + kTcSplitPairs - 1) / kTcSplitPairs, ctrls);
  g_tc_last_pair = 2;
  return launch_k1(kern, grid, 64 * kTcSplitPairs, smem, stream, a, frag);
}
template <int Mode, bool STAB>
cudaError_t go_split(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, int n_chunks, int ctrls,
                     cudaStream_t stream) {
  const char* e = std::getenv("MPPI_SPLIT_PF");
  const bool pf = e ? std::atoi(e) != 0 : n_chunks <= kSplitPfChunks;
  return pf ? go_split_pf<Mode, STAB, true>(a, frag, n_chunks, ctrls, stream)
            : go_split_pf<Mode, STAB, false>(a, frag, n_chunks, ctrls, stream);
}
// eps' stays on chip when the grid still fits one wave with that footprint
// (tc_min_ctas CTAs of 4 warps per SM); larger launches regenerate it from
// the counters.
template <int H, int MT, int Mode, bool STAB>
cudaError_t go(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, int n_chunks, int ctrls,
               cudaStream_t stream) {
  const size_t plan_bytes = (sizeof(float) * (2 * a.T + 2) + 15) & ~size_t(15);
  const size_t base = plan_bytes + sizeof(double) * kTcWarps * mppi_dev::tc_red_doubles(false);
  const size_t base_store = plan_bytes + sizeof(double) * kTcWarps * mppi_dev::tc_red_doubles(true);
  const size_t eps_bytes = sizeof(float2) * kTcWarps * a.T * 16 * MT;
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const long long ctas = static_cast<long long>((n_chunks + kTcWarps - 1) / kTcWarps) * ctrls;
  constexpr int per_sm = mppi_dev::tc_min_ctas<H, MT>();
  const bool store = std::getenv("MPPI_TC_STORE") ? std::atoi(std::getenv("MPPI_TC_STORE")) != 0
                                                   : (per_sm * (base_store + eps_bytes) <= 220 * 1024 &&
                                                      ctas <= per_sm * static_cast<long long>(sms));
  g_tc_last_pair = 0;
  if constexpr (H == 32 && MT == 1) {
    if (!a.trace_states && split_fits<Mode, STAB>(a.T, n_chunks, ctrls))
      return go_split<Mode, STAB>(a, frag, n_chunks, ctrls, stream);
    if (!a.trace_states && pair_fits<Mode, STAB>(a.T, n_chunks, ctrls))
      return go_pair<Mode, STAB>(a, frag, n_chunks, ctrls, stream);
  }
  // (MT = 2 serves K > 32768, whose grid never fits one wave: no on-chip eps')
  if constexpr (MT == 1) {
    if (store && !a.trace_states)
      return go_store<H, MT, Mode, STAB, true>(a, frag, n_chunks, ctrls, base_store + eps_bytes, stream);
  }
  return go_store<H, MT, Mode, STAB, false>(a, frag, n_chunks, ctrls, base, stream);
}
template <int H, int Mode, bool STAB>
cudaError_t by_mt(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, int mt, int n_chunks, int ctrls,
                  cudaStream_t stream) {
  if constexpr (H > 32) {  // one m16 tile per warp (register budget of the H = 64 accumulators)
    return go<H, 1, Mode, STAB>(a, frag, n_chunks, ctrls, stream);
  } else {
    return mt == 1 ? go<H, 1, Mode, STAB>(a, frag, n_chunks, ctrls, stream)
                   : go<H, 2, Mode, STAB>(a, frag, n_chunks, ctrls, stream);
  }
}
template <int H, int Mode>
cudaError_t by_stab(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, int mt, int n_chunks, int ctrls,
                    cudaStream_t stream) {
  // the side-slip term (atan) is compiled in only when its weight is nonzero
  return a.sys.cost.alpha_stab != 0.f ? by_mt<H, Mode, true>(a, frag, mt, n_chunks, ctrls, stream)
                                      : by_mt<H, Mode, false>(a, frag, mt, n_chunks, ctrls, stream);
}
}  // namespace tc_detail

template <int H>
cudaError_t launch_tail_tc(const mppi_dev::Acc* rows, int n, int stride, long long ctrl_stride, double lambda,
                           const mppi_dev::TailArgs& ta, int ctrls, bool pdl, cudaStream_t stream) {
  const size_t smem = mppi_dev::tail_smem_bytes<H>(n, ta.e.T);
  auto kern = mppi_dev::tail_kernel<H>;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  // one CTA per controller; a programmatic dependent launch (pdl) of the group
  // merge, so its prefetch of the plan, state and weights overlaps that kernel
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1, ctrls);
  cfg.blockDim = dim3(mppi_dev::kTailBlock);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, rows, n, stride, ctrl_stride, lambda, ta);
}

#ifdef TC_MODE
template cudaError_t tc_detail::by_stab<TC_H, TC_MODE>(const mppi_dev::RolloutArgs<float>&, const uint32_t*, int,
                                                        int, int, cudaStream_t);
#endif
#ifdef TC_TAIL
template cudaError_t launch_tail_tc<TC_H>(const mppi_dev::Acc*, int, int, long long, double, const mppi_dev::TailArgs&,
                                          int, bool, cudaStream_t);
#endif

}  // namespace mppi_host
