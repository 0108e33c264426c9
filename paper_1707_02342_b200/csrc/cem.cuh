// cem.cuh — the cross-entropy weight rule on the device (cem_weights,
// proj/src/weights.cpp:27-53): the elite = lround(K (1 - delta)) lowest costs,
// ties broken by ascending sample index, each weighted 1 / elite.
//
// One CTA: a radix select over order-preserving 64-bit keys of the double
// costs (8 passes of 8 bits, shared-memory histograms) finds the elite-th
// smallest cost T and how many of the samples equal to T belong to the elite;
// a pass in ascending index order (block scan of the "== T" flags) then
// admits the first of them, exactly as the reference's stable
// (cost, index) sort.  The weighted update that follows is update_plan with
// these caller weights (weighted_agg_kernel, rollout.cuh), the plan update the
// epilogue (epilogue.cuh).
#pragma once

#include "epilogue.cuh"

namespace mppi_dev {

__device__ __forceinline__ unsigned long long cost_key(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// w[K] (1/elite or 0), rho_eta = (min cost, elite).  Non-finite costs: *bad_out
// = 1 and, if `status` is given, status->code = MPPI_ERR_NONFINITE (sticky).
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) cem_weights_kernel(const double* __restrict__ costs, int K, int elite,
                                                            double* w, double* rho_eta, int* bad_out,
                                                            StepStatus* status) {
  __shared__ unsigned hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ int s_kth;
  __shared__ double s_red[BLOCK / 32];
  __shared__ unsigned s_warp[BLOCK / 32];
  if (status && status->code != 0) return;  // a previous stage failed
  int bad = 0;
  double m = INFINITY;
  for (int k = threadIdx.x; k < K; k += BLOCK) {
    const double c = costs[k];
    bad |= !isfinite(c);
    m = (c < m) ? c : m;
  }
  bad = __syncthreads_or(bad);
  if (bad) {
    if (threadIdx.x == 0) {
      if (bad_out) *bad_out = 1;
      if (status) status->code = 2;  // cem_weights: non-finite cost (weights.cpp:33)
    }
    return;
  }
  const double rho = block_min<double, BLOCK>(m, s_red);
  if (threadIdx.x == 0) {
    s_prefix = 0ull;
    s_kth = elite - 1;
  }
  unsigned long long mask = 0ull;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += BLOCK) hist[i] = 0u;
    __syncthreads();
    const unsigned long long prefix = s_prefix;
    for (int k = threadIdx.x; k < K; k += BLOCK) {
      const unsigned long long key = cost_key(costs[k]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xFFull], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int kth = s_kth, d = 0;
      unsigned cum = 0;
      for (; d < 256; ++d) {
        if (cum + hist[d] > static_cast<unsigned>(kth)) break;
        cum += hist[d];
      }
      s_kth = kth - static_cast<int>(cum);
      s_prefix = prefix | (static_cast<unsigned long long>(d) << shift);
    }
    mask |= 0xFFull << shift;
    __syncthreads();
  }
  const unsigned long long thr = s_prefix;
  const int need_eq = s_kth + 1;  // samples equal to the threshold that are elite
  const double inv = 1.0 / static_cast<double>(elite);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int running = 0;  // "== thr" samples at lower indices seen so far
  for (int base = 0; base < K; base += BLOCK) {
    const int k = base + threadIdx.x;
    const unsigned long long key = (k < K) ? cost_key(costs[k]) : ~0ull;
    const bool eq = k < K && key == thr;
    const bool lt = k < K && key < thr;
    const unsigned ball = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) s_warp[wid] = __popc(ball);
    __syncthreads();
    int before = running;
    for (int i = 0; i < wid; ++i) before += static_cast<int>(s_warp[i]);
    before += __popc(ball & ((1u << lane) - 1u));
    if (k < K) w[k] = (lt || (eq && before < need_eq)) ? inv : 0.0;
    int tile = 0;
    for (int i = 0; i < BLOCK / 32; ++i) tile += static_cast<int>(s_warp[i]);
    running += tile;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    rho_eta[0] = rho;
    rho_eta[1] = static_cast<double>(elite);
    if (bad_out) *bad_out = 0;
  }
}

}  // namespace mppi_dev
