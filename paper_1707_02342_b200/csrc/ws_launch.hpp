// ws_launch.hpp — launchers of the warp-specialised fp32 rollout kernel
// (rollout_ws.cuh), compiled in their own translation units (ws_h32.cu,
// ws_h64.cu, tc_h32.cu) so the per-(H, L, noise) instantiations build in
// parallel.
#pragma once

#include <cuda_runtime.h>

#include "model.cuh"
#include "rollout.cuh"
#include "tail.cuh"

namespace mppi_host {

cudaError_t launch_rollout_ws_h32(const mppi_dev::RolloutArgs<float>& a, const mppi_dev::WeightHolder<float, 32>& w,
                                  int mode, int L, bool smem_weights, dim3 grid, size_t smem, cudaStream_t stream);
cudaError_t launch_rollout_ws_h64(const mppi_dev::RolloutArgs<float>& a, const mppi_dev::WeightHolder<float, 64>& w,
                                  int mode, int L, bool smem_weights, dim3 grid, size_t smem, cudaStream_t stream);

namespace tc_detail {
// whether the last tensor-core K1 enqueued was the warp-pair kernel (reporting)
extern int g_tc_last_pair;
// the per-(H, noise mode) launchers, one translation unit each (tc_h*_*.cu)
template <int H, int Mode>
cudaError_t by_stab(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, const mppi_dev::TailArgs& tail,
                    int mt, int n_chunks, int ctrls, cudaStream_t stream);
}  // namespace tc_detail

// Tensor-core rollout (rollout_tc.cuh) for hidden width H (32, 64): `frag` is
// the per-lane fragment table built by tc_build_fragments; n_chunks chunks of
// 16*mt samples from a.chunk0 (mt is 1 at H = 64).
template <int H>
cudaError_t launch_rollout_tc(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag,
                              const mppi_dev::TailArgs& tail, int mode, int mt, int n_chunks, int ctrls,
                              cudaStream_t stream);
// The tensor-core tail in one launch: element-parallel merge, then the epilogue
// by the last CTA (tail.cuh).  counters: one zero-initialised unsigned per controller.
template <int H>
cudaError_t launch_tail_tc(const mppi_dev::Acc* partials, int n, int stride, long long ctrl_stride, double lambda,
                           mppi_dev::Acc* merged, unsigned* counters, const mppi_dev::TailArgs& ta, int ctrls,
                           cudaStream_t stream);
// Whether the cooperative tensor-core K1 (merge + epilogue inside, tail mode 1)
// can run: the whole grid co-resident and the tail's scratch within the CTA's buffers.
template <int H>
bool tc_coop_fits(int T, int mt, int n_chunks, size_t epilogue_smem);
extern template cudaError_t launch_tail_tc<32>(const mppi_dev::Acc*, int, int, long long, double, mppi_dev::Acc*,
                                               unsigned*, const mppi_dev::TailArgs&, int, cudaStream_t);
extern template cudaError_t launch_tail_tc<64>(const mppi_dev::Acc*, int, int, long long, double, mppi_dev::Acc*,
                                               unsigned*, const mppi_dev::TailArgs&, int, cudaStream_t);
extern template bool tc_coop_fits<32>(int, int, int, size_t);
extern template bool tc_coop_fits<64>(int, int, int, size_t);
// Element-parallel merge of n chunk partial rows into one row per controller (tail.cuh).
cudaError_t launch_merge_elements(const mppi_dev::Acc* partials, int n, int stride, long long ctrl_stride,
                                  double lambda, mppi_dev::Acc* merged, int ctrls, cudaStream_t stream);

}  // namespace mppi_host
