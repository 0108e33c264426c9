// ws_launch.hpp — launchers of the warp-specialised fp32 rollout kernel
// (rollout_ws.cuh), compiled in their own translation units (ws_h32.cu,
// ws_h64.cu, tc_h32.cu) so the per-(H, L, noise) instantiations build in
// parallel.
#pragma once

#include <cuda_runtime.h>

#include "model.cuh"
#include "rollout.cuh"
#include "tail.cuh"
#include "group.cuh"

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
cudaError_t by_stab(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, int mt, int n_chunks, int ctrls,
                    cudaStream_t stream);
}  // namespace tc_detail

// Tensor-core rollout (rollout_tc.cuh) for hidden width H (32, 64): `frag` is
// the per-lane fragment table built by tc_build_fragments; n_chunks chunks of
// 16*mt samples from a.chunk0 (mt is 1 at H = 64).
template <int H>
cudaError_t launch_rollout_tc(const mppi_dev::RolloutArgs<float>& a, const uint32_t* frag, int mode, int mt,
                              int n_chunks, int ctrls, cudaStream_t stream);
// The tensor-core tail: merge of the n group rows and the epilogue, one CTA
// per controller (tail.cuh).
template <int H>
cudaError_t launch_tail_tc(const mppi_dev::Acc* rows, int n, int stride, long long ctrl_stride, double lambda,
                           const mppi_dev::TailArgs& ta, int ctrls, bool pdl, cudaStream_t stream);
extern template cudaError_t launch_tail_tc<32>(const mppi_dev::Acc*, int, int, long long, double,
                                               const mppi_dev::TailArgs&, int, bool, cudaStream_t);
extern template cudaError_t launch_tail_tc<64>(const mppi_dev::Acc*, int, int, long long, double,
                                               const mppi_dev::TailArgs&, int, bool, cudaStream_t);
// The tcgen05 / TMEM rollout (rollout_umma.cuh), H = 32 or 64: chunks of 128
// samples from a.chunk0; wimg is the weight image (umma_build_image).
template <int H>
cudaError_t launch_rollout_umma(const mppi_dev::RolloutArgs<float>& a, const unsigned char* wimg, int mode,
                                int n_chunks, int ctrls, cudaStream_t stream);
template <>
cudaError_t launch_rollout_umma<32>(const mppi_dev::RolloutArgs<float>&, const unsigned char*, int, int, int,
                                    cudaStream_t);
template <>
cudaError_t launch_rollout_umma<64>(const mppi_dev::RolloutArgs<float>&, const unsigned char*, int, int, int,
                                    cudaStream_t);
// Fixed-group merge of the chunk partials (group.cuh): groups [g0, g0 + n_local)
// of n_groups; programmatic dependent of the previous kernel when pdl.
cudaError_t launch_group_merge(const mppi_dev::Acc* partials, long long partials_ctrl_stride, int n_chunks,
                               int n_groups, int g0, int n_local, int stride, double lambda, mppi_dev::Acc* groups,
                               long long groups_ctrl_stride, int ctrls, bool pdl, cudaStream_t stream);

}  // namespace mppi_host
