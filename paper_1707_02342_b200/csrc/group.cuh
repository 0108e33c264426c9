// group.cuh — the fixed-group merge of the chunk softmin partials: the unit
// the ranks exchange when the samples of one controller are sharded.
//
// K1 reduces every chunk of samples to a row (rho_c, eta_c, bad_c, 0,
// num_c[T][2]) relative to the chunk minimum.  The chunks of a controller are
// cut into n_groups CONTIGUOUS groups whose boundaries depend only on the
// global chunk count (group g = chunks [floor(g n / G), floor((g+1) n / G)),
// G = 8 * 2^j, the smallest such that no group holds more than
// kGroupRowsMax chunks).  Each group is merged into one row of the same format:
//   rho_g = min_c rho_c,  x_g[e] = sum_c exp(-(rho_c - rho_g) / lambda) P[c][e]
// (e = eta and the 2T numerators) in a FIXED order: stripe q of the CTA sums
// the rows c = q, q + 8, ... of the group sequentially, then the eight stripe
// sums are added as a balanced tree.  The order is a function of the group's
// rows only, so a rank that owns groups [g_lo, g_hi) produces exactly the rows
// the single-GPU run produces for them.
//
// Rank r of N owns groups [r G / N, (r+1) G / N) — a contiguous range of
// chunks — and the exchange is one all-gather of its G / N group rows
// (G x (4 + 2T) x 8 B for the whole job: 13 KB at T = 100), after which every
// rank merges the G rows in group order (tail.cuh / epilogue.cuh).  The plan
// is therefore bit-identical for every N that divides G, and on every rank.
// Reference: parallel_for_chunks makes results independent of the thread
// count (parallel.hpp:11-29, pinned by test_controller.cpp:199-217).
#pragma once

#include "rollout.cuh"
#include "shard.hpp"

namespace mppi_dev {

constexpr int kGroupStripes = 8;    // warps per CTA; stripe q sums rows q, q + 8, ...
constexpr int kGroupElems = 32;     // elements per CTA (one per lane)
constexpr int kGroupBlock = 32 * kGroupStripes;
static_assert(kGroupRowsMax % kGroupStripes == 0 && kGroupRowsMax <= kGroupBlock, "group shape");

// grid = (groups of this rank, ceil(stride / kGroupElems), controllers),
// block = kGroupBlock.  partials: [C][n_chunks][stride] (global chunk index);
// groups: [C][n_groups][stride] (global group index).  May be launched as a
// programmatic dependent of K1: nothing is read before the grid dependency.
// (A template only so that every translation unit may include it.)
template <int kUnused = 0>
__global__ void __launch_bounds__(kGroupBlock) group_merge_kernel(const Acc* __restrict__ partials,
                                                                  long long partials_ctrl_stride, int n_chunks,
                                                                  int n_groups, int g0, int stride, double lambda,
                                                                  Acc* __restrict__ groups,
                                                                  long long groups_ctrl_stride) {
  __shared__ Acc s_scale[kGroupRowsMax];
  __shared__ Acc s_part[kGroupStripes][kGroupElems];
  __shared__ Acc s_min[kGroupStripes];
  // the tail (a programmatic dependent) may launch now and stage its inputs
  // while K1 and this grid run; its own grid-dependency wait still covers
  // this grid's completion
  cudaTriggerProgrammaticLaunchCompletion();
  cudaGridDependencySynchronize();
  const int g = g0 + blockIdx.x, ctrl = blockIdx.z;
  const int r0 = group_first_chunk(g, n_chunks, n_groups), r1 = group_first_chunk(g + 1, n_chunks, n_groups);
  const int n = r1 - r0;  // <= kGroupRowsMax (0: an empty group, K < 8 chunks)
  MPPI_DCHECK(g < n_groups && n >= 0 && n <= kGroupRowsMax && r1 <= n_chunks);
  MPPI_DCHECK(static_cast<long long>(r1) * stride <= partials_ctrl_stride);
  const Acc* P = partials + static_cast<size_t>(ctrl) * partials_ctrl_stride + static_cast<size_t>(r0) * stride;
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int e = blockIdx.y * kGroupElems + lane;
  // this lane's element of its stripe's rows (q, q + 8, ...), all loads in
  // flight at once, issued before the group minimum is known
  constexpr int kPer = kGroupRowsMax / kGroupStripes;
  Acc v[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int r = q + kGroupStripes * i;
    v[i] = (r < n && e < stride) ? __ldcg(P + static_cast<size_t>(r) * stride + e) : 0.0;
  }
  // rho_g = min over the group's chunk minima; bad_g = any chunk non-finite
  Acc m = INFINITY;
  int bad = 0;
  if (threadIdx.x < n) {
    const Acc rr = __ldcg(P + static_cast<size_t>(threadIdx.x) * stride);
    bad = __ldcg(P + static_cast<size_t>(threadIdx.x) * stride + 2) != 0.0;
    m = rr;
    s_scale[threadIdx.x] = rr;
  }
  m = warp_min(m);
  if (lane == 0) s_min[q] = m;
  bad = __syncthreads_or(bad);
  Acc rho = s_min[0];
#pragma unroll
  for (int w = 1; w < kGroupStripes; ++w) rho = (s_min[w] < rho) ? s_min[w] : rho;
  // chunk scale exp(-(rho_c - rho_g) / lambda) in double (it_weights,
  // weights.cpp:15-23, relative to the group minimum)
  const double inv_lambda = 1.0 / lambda;
  if (threadIdx.x < n) s_scale[threadIdx.x] = exp(-(s_scale[threadIdx.x] - rho) * inv_lambda);
  __syncthreads();
  Acc s = 0.0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int r = q + kGroupStripes * i;
    if (r < n) s = fma(s_scale[r], v[i], s);
  }
  s_part[q][lane] = s;
  __syncthreads();
  if (q == 0 && e < stride) {
    const Acc(&p)[kGroupStripes][kGroupElems] = s_part;
    Acc v = ((p[0][lane] + p[1][lane]) + (p[2][lane] + p[3][lane])) +
            ((p[4][lane] + p[5][lane]) + (p[6][lane] + p[7][lane]));
    if (e == 0) v = rho;
    else if (e == 2) v = bad ? 1.0 : 0.0;
    else if (e == 3) v = 0.0;
    groups[static_cast<size_t>(ctrl) * groups_ctrl_stride + static_cast<size_t>(g) * stride + e] = v;
  }

}

}  // namespace mppi_dev
