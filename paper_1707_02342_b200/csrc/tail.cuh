// tail.cuh — the iteration tail of the tensor-core path: merge of the chunk
// softmin partials, then the epilogue of mpc_step.
//
// K1 reduces every chunk of samples to (rho_c, eta_c, bad_c, num_c[T][2])
// relative to the chunk minimum.  The merge is ELEMENT-parallel: rho =
// min_c rho_c, and every other element e is
//   merged[e] = sum_c exp(-(rho_c - rho) / lambda) * P[c][e],
// computed by one CTA of kMergeBlock threads per element (thread j takes chunks
// j, j + kMergeBlock, ... in ascending order; the thread sums are then added
// by a fixed butterfly + warp-order tree).  The summation order depends only
// on the chunk count, never on which CTA handles which element, so
//   * the cooperative K1 (one wave: grid.sync, merge by all CTAs, grid.sync,
//     epilogue by CTA 0 — no extra kernel boundary), and
//   * merge_elements_kernel after a separate K1 (large K, or ranks > 1 after
//     the all-gather of chunk partials)
// produce bit-identical plans.  The epilogue then runs on the single merged
// row (scale exp(0) = 1: the row passes through unchanged).
#pragma once

#include <cooperative_groups.h>

#include <algorithm>

#include "epilogue.cuh"

namespace mppi_dev {

constexpr int kMergeBlock = 128;
constexpr int kMergeElems = 8;  // elements per pass of a CTA (independent loads in flight)
constexpr int kMergeRows = 8;   // rows per thread of merge_elements' single-pass path
constexpr int kMergeFastElems = 4;  // elements per CTA of that path (the tail's quarter-size grid)

struct TailArgs {
  int mode;                             // 0: chunk partials only; 1: cooperative merge + epilogue in K1
  Acc* merged;                          // [C][partial_stride]: the merged row
  const void* plant_w;                  // MlpParams<float, H> of the model (device plant)
  EpilogueArgs<float> e;                // epilogue over `merged` (n_chunks = 1)
};

// Deterministic CTA sum of kMergeElems values per thread (butterfly, then
// warps in order).  s_part: (BLOCK/32) x kMergeElems doubles.
template <int BLOCK>
__device__ __forceinline__ void block_sum_n(Acc (&v)[kMergeElems], Acc* s_part) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < kMergeElems; ++j) v[j] = warp_sum(v[j]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < kMergeElems; ++j) s_part[wid * kMergeElems + j] = v[j];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kMergeElems; ++j) {
    Acc s = s_part[j];
    for (int w = 1; w < BLOCK / 32; ++w) s = s + s_part[w * kMergeElems + j];
    v[j] = s;
  }
}

// One CTA (BLOCK threads): merged elements e0, e0 + estep, ... of the rows
// P[0..n) (stride doubles each).  smem: merge_smem_bytes(n).  The CTA with
// e0 == 0 also writes rho, bad and the reserved slot.
template <int BLOCK, bool FAST = true>
__device__ void merge_elements(const Acc* P, int n, int stride, double lambda, Acc* merged, int e0, int estep,
                               double* smem) {
  double* s_scale = smem;
  double* s_part = smem + n;
  // one pass over the rows when every thread holds at most kMergeRows of them
  // and the CTA has at most kMergeFastElems elements: the element values
  // are loaded together with rho (one round trip less) and the scales stay in
  // registers.  Same per-thread row order and the same scale values as the
  // general path below, so the sums are bit-identical.
  // (FAST = false inside K1's cooperative tail: its registers would spill K1)
  if (FAST && n <= kMergeRows * BLOCK && e0 + kMergeFastElems * estep >= stride) {
    Acc rr[kMergeRows], x[kMergeRows][kMergeFastElems];
    Acc m = INFINITY;
    int bad = 0;
#pragma unroll
    for (int i = 0; i < kMergeRows; ++i) {
      const int r = threadIdx.x + i * BLOCK;
      rr[i] = INFINITY;
#pragma unroll
      for (int j = 0; j < kMergeFastElems; ++j) x[i][j] = 0.0;
      if (r < n) {
        const Acc* pr = P + static_cast<size_t>(r) * stride;
        rr[i] = __ldcg(pr);
        bad |= (__ldcg(pr + 2) != 0.0);
#pragma unroll
        for (int j = 0; j < kMergeFastElems; ++j) {
          const int e = e0 + j * estep;
          if (e < stride) x[i][j] = __ldcg(pr + e);
        }
        m = (rr[i] < m) ? rr[i] : m;
      }
    }
    m = warp_min(m);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = m;
    bad = __syncthreads_or(bad);
    Acc rho = s_part[0];
    for (int w = 1; w < BLOCK / 32; ++w) rho = (s_part[w] < rho) ? s_part[w] : rho;
    if (e0 == 0 && threadIdx.x == 0) {
      merged[0] = rho;
      merged[2] = bad ? 1.0 : 0.0;
      merged[3] = 0.0;
    }
    const double inv_lambda = 1.0 / lambda;
    Acc acc[kMergeElems];  // (block_sum_n reduces kMergeElems; the rest stay 0)
#pragma unroll
    for (int j = 0; j < kMergeElems; ++j) acc[j] = 0.0;
#pragma unroll
    for (int i = 0; i < kMergeRows; ++i) {
      if (threadIdx.x + i * BLOCK < n) {
        const Acc sc = static_cast<double>(__expf(static_cast<float>(-(rr[i] - rho) * inv_lambda)));
#pragma unroll
        for (int j = 0; j < kMergeFastElems; ++j) acc[j] = fma(sc, x[i][j], acc[j]);
      }
    }
    block_sum_n<BLOCK>(acc, s_part + BLOCK / 32);
    if (threadIdx.x == 0)
#pragma unroll
      for (int j = 0; j < kMergeFastElems; ++j) {
        const int e = e0 + j * estep;
        if (e < stride && (e == 1 || e >= kPartialHeader)) merged[e] = acc[j];
      }
    return;
  }
  Acc m = INFINITY;
  int bad = 0;
#pragma unroll 8
  for (int r = threadIdx.x; r < n; r += BLOCK) {
    const Acc rho_r = __ldcg(P + static_cast<size_t>(r) * stride);
    bad |= (__ldcg(P + static_cast<size_t>(r) * stride + 2) != 0.0);
    m = (rho_r < m) ? rho_r : m;
    s_scale[r] = rho_r;
  }
  m = warp_min(m);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = m;
  bad = __syncthreads_or(bad);
  Acc rho = s_part[0];
  for (int w = 1; w < BLOCK / 32; ++w) rho = (s_part[w] < rho) ? s_part[w] : rho;
  // scale of row r, e^{-(rho_r - rho)/lambda} (fp32 SFU exp of the double
  // argument: ~1e-7 relative, deterministic, against ~1e-5 update tolerances)
  const double inv_lambda = 1.0 / lambda;
  for (int r = threadIdx.x; r < n; r += BLOCK)
    s_scale[r] = static_cast<double>(__expf(static_cast<float>(-(s_scale[r] - rho) * inv_lambda)));
  __syncthreads();
  if (e0 == 0 && threadIdx.x == 0) {
    merged[0] = rho;
    merged[2] = bad ? 1.0 : 0.0;
    merged[3] = 0.0;
  }
  for (int eb = e0; eb < stride; eb += kMergeElems * estep) {
    Acc acc[kMergeElems];
#pragma unroll
    for (int j = 0; j < kMergeElems; ++j) acc[j] = 0.0;
#pragma unroll 4
    for (int r = threadIdx.x; r < n; r += BLOCK) {
      const Acc sc = s_scale[r];
      const Acc* pr = P + static_cast<size_t>(r) * stride;
      Acc x[kMergeElems];
#pragma unroll
      for (int j = 0; j < kMergeElems; ++j) {
        const int e = eb + j * estep;
        x[j] = (e < stride) ? __ldcg(pr + e) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < kMergeElems; ++j) acc[j] = fma(sc, x[j], acc[j]);
    }
    block_sum_n<BLOCK>(acc, s_part + BLOCK / 32);
    if (threadIdx.x == 0)
#pragma unroll
      for (int j = 0; j < kMergeElems; ++j) {
        const int e = eb + j * estep;
        if (e < stride && (e == 1 || e >= kPartialHeader)) merged[e] = acc[j];
      }
  }
}

template <int kUnused = 0>
__global__ void __launch_bounds__(kMergeBlock) merge_elements_kernel(const Acc* __restrict__ partials, int n,
                                                                     int stride, long long ctrl_stride,
                                                                     double lambda, Acc* merged) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ctrl = blockIdx.y;
  merge_elements<kMergeBlock>(partials + static_cast<size_t>(ctrl) * ctrl_stride, n, stride, lambda,
                              merged + static_cast<size_t>(ctrl) * stride, blockIdx.x, gridDim.x,
                              reinterpret_cast<double*>(smem_raw));
}

__host__ __device__ constexpr size_t merge_smem_bytes(int n) {
  return sizeof(double) * (n + (kMergeBlock / 32) * (kMergeElems + 1));
}

// The epilogue of mpc_step on the merged row, for one CTA of kMergeBlock
// threads (fp32 vehicle model, H = 32 or 64): every global input (status,
// merged row, plan, plant state, weights) is fetched in one phase, then
// agg = num / eta, Savitzky-Golay (smoothing.cpp:48-65, mirror padding),
// U' = U + agg (double, rounded once; ControlPlan finiteness check,
// types.hpp:79-83), u0 = clamp(U'[0]), slide, ++iteration, and the device
// plant step run with three block barriers and one warp for the plant MLP
// (lane j owns hidden units j, j + 32, ...; the operation order of each unit
// is that of epilogue_kernel).  smem: fast_epilogue_smem_bytes<H>(T).
template <int H>
__host__ __device__ constexpr size_t fast_epilogue_smem_bytes(int T) {
  return sizeof(double) * 2 * T + sizeof(float) * 2 * T;  // agg + U' (reuses the merge scratch)
}
// What every tail CTA fetches before waiting for K1 (none of it is written by
// K1): the plan, the plant state and the model weights.  smem: tail_pre_bytes.
template <int H>
__host__ __device__ constexpr size_t tail_pre_bytes(int T) {
  return ((sizeof(float) * (2 * T + 8) + 15) & ~size_t(15)) + sizeof(MlpParams<float, H>);
}
template <int H>
__device__ __forceinline__ void tail_prefetch(const EpilogueArgs<float>& a, const MlpParams<float, H>* w_src, int ctrl,
                                              unsigned char* pre) {
  const int T = a.T;
  float* s_plan = reinterpret_cast<float*>(pre);
  float* s_x = s_plan + 2 * T;
  MlpParams<float, H>* s_w =
      reinterpret_cast<MlpParams<float, H>*>(pre + ((sizeof(float) * (2 * T + 8) + 15) & ~size_t(15)));
  const float* plan = a.plan + static_cast<size_t>(ctrl) * 2 * T;
  for (int i = threadIdx.x; i < 2 * T; i += kMergeBlock) s_plan[i] = plan[i];
  if (threadIdx.x < 8) s_x[threadIdx.x] = a.x0[static_cast<size_t>(ctrl) * 8 + threadIdx.x];
  if (a.plant) {
    const float4* src = reinterpret_cast<const float4*>(w_src);
    float4* dst = reinterpret_cast<float4*>(s_w);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(MlpParams<float, H>) / 16); i += kMergeBlock)
      dst[i] = src[i];
  }
}
// The finished status of controller ctrl into the mapped host mirror (one
// thread; its own earlier writes to *st are ordered before these reads): the
// step graph then needs no device-to-host copy node.
__device__ __forceinline__ void publish_status(const EpilogueArgs<float>& a, int ctrl) {
  if (!a.status_host) return;
  const StepStatus* st = a.status + ctrl;
  StepStatus* sh = a.status_host + ctrl;
  sh->code = st->code;
  sh->u0[0] = st->u0[0];
  sh->u0[1] = st->u0[1];
#pragma unroll
  for (int i = 0; i < 8; ++i) sh->x[i] = st->x[i];
  sh->iteration = st->iteration;
}

template <int H>
__device__ __forceinline__ void epilogue_fast(const EpilogueArgs<float>& a, const Acc* row, int ctrl,
                                              unsigned char* smem, const unsigned char* pre) {
  constexpr int U = H / 32;  // hidden units per lane
  const int T = a.T;
  double* s_agg = reinterpret_cast<double*>(smem);
  float* s_new = reinterpret_cast<float*>(s_agg + 2 * T);
  const float* s_plan = reinterpret_cast<const float*>(pre);
  const float* s_x = s_plan + 2 * T;
  const MlpParams<float, H>* s_w =
      reinterpret_cast<const MlpParams<float, H>*>(pre + ((sizeof(float) * (2 * T + 8) + 15) & ~size_t(15)));
  __shared__ int s_code;
  __shared__ double s_sg[kMaxSgWindow];
  for (int j = threadIdx.x; j < a.sg_window; j += kMergeBlock) s_sg[j] = a.sg[j];
  StepStatus* st = a.status + ctrl;
  float* plan = a.plan + static_cast<size_t>(ctrl) * 2 * T;
  // ---- phase 1: the merged row and the status (the rest was prefetched)
  if (threadIdx.x == 0) {
    int code = __ldcg(&st->code);
    if (code == 0 && __ldcg(row + 2) != 0.0) code = 2;  // it_weights: non-finite cost (weights.cpp:12)
    s_code = code;
  }
  const double eta_l = __ldcg(row + 1);
  for (int i = threadIdx.x; i < 2 * T; i += kMergeBlock)
    s_agg[i] = __ldcg(row + kPartialHeader + i) / eta_l;  // agg = num / eta, once per element
  __syncthreads();
  if (s_code != 0) {
    if (threadIdx.x == 0) {
      if (__ldcg(&st->code) == 0) st->code = s_code;
      publish_status(a, ctrl);
    }
    return;
  }
  // ---- SG smoothing of agg, U' = U + SG(agg)
  const int half = a.sg_window / 2;
  int nonfinite = 0;
  for (int i = threadIdx.x; i < 2 * T; i += kMergeBlock) {
    const int t = i >> 1, c = i & 1;
    Acc v;
    if (a.sg_window > 0) {
      Acc acc = 0.0;
      for (int j = -half; j <= half; ++j) {
        // reflect_index (smoothing.cpp:37-44); one mirror suffices inside the
        // interior, the loop form only when the window exceeds the horizon
        int idx = t + j;
        if (idx < 0 || idx >= T) idx = reflect_index(idx, T);
        acc = __dadd_rn(acc, __dmul_rn(s_sg[j + half], s_agg[idx * 2 + c]));
      }
      v = acc;
    } else {
      v = s_agg[i];
    }
    const float nv = static_cast<float>(__dadd_rn(static_cast<Acc>(s_plan[i]), v));
    nonfinite |= !isfinite(nv);
    s_new[i] = nv;
  }
  if (__syncthreads_or(nonfinite)) {  // ControlPlan rejects non-finite plans
    if (threadIdx.x == 0) {
      st->code = 1;
      publish_status(a, ctrl);
    }
    return;
  }
  const float u0 = clamp_r(s_new[0], a.lo0, a.hi0), u1 = clamp_r(s_new[1], a.lo1, a.hi1);
  for (int i = threadIdx.x; i < 2 * T; i += kMergeBlock)
    plan[i] = a.slide ? ((i + 2 < 2 * T) ? s_new[i + 2] : 0.f) : s_new[i];
  uint64_t it = a.iters[ctrl];
  if (a.increment) it += 1;
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  if (lane == 0) {
    st->u0[0] = static_cast<double>(u0);
    st->u0[1] = static_cast<double>(u1);
    if (a.u_trace) {
      const uint64_t idx = it - 1 - a.trace_base[ctrl];
      a.u_trace[(idx * a.n_ctrl + ctrl) * 2] = u0;
      a.u_trace[(idx * a.n_ctrl + ctrl) * 2 + 1] = u1;
    }
  }
  if (a.plant) {
    const MlpParams<float, H>& w = *s_w;
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = s_x[i];
    const float in[6] = {x[3], x[4], x[5], x[6], u0, u1};
    float h1[U], h2[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = lane + 32 * u;
      float acc = w.b1[j];
#pragma unroll
      for (int i = 0; i < 6; ++i) acc = fma_r(w.w1t[i][j], in[i], acc);
      h1[u] = tanh_r(acc);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = lane + 32 * u;
      float acc = w.b2[j];
#pragma unroll
      for (int uu = 0; uu < U; ++uu)
#pragma unroll 8
        for (int i = 0; i < 32; ++i) acc = fma_r(w.w2t[32 * uu + i][j], __shfl_sync(0xffffffffu, h1[uu], i), acc);
      h2[u] = tanh_r(acc);
    }
    float d = (lane < 4) ? w.b3[lane] : 0.f;
#pragma unroll
    for (int uu = 0; uu < U; ++uu)
#pragma unroll 8
      for (int i = 0; i < 32; ++i) {
        const float hi = __shfl_sync(0xffffffffu, h2[uu], i);
        if (lane < 4) d = fma_r(w.w3t[32 * uu + i][lane], hi, d);
      }
    float dd[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) dd[o] = __shfl_sync(0xffffffffu, d, o);
    if (lane == 0) {
      advance_split<float>(x, dd, a.sys.dt);
      float* xo = a.x0 + static_cast<size_t>(ctrl) * 8;
      for (int i = 0; i < 7; ++i) xo[i] = x[i];
      for (int i = 0; i < 8; ++i) st->x[i] = static_cast<double>(x[i]);
      if (a.x_trace) {
        const uint64_t idx = it - a.trace_base[ctrl];
        for (int i = 0; i < 8; ++i) a.x_trace[(idx * a.n_ctrl + ctrl) * 8 + i] = x[i];
      }
    }
  }
  if (lane == 0) {
    a.iters[ctrl] = it;
    st->iteration = it;
    publish_status(a, ctrl);
  }
}

// The tensor-core path's tail in one launch: the element-parallel merge by
// every CTA, then the epilogue by the CTA that finishes last (threadfence +
// ticket; the counter resets itself).  grid = (elements CTAs, controllers).
template <int H>
__global__ void __launch_bounds__(kMergeBlock) tail_kernel(const Acc* __restrict__ partials, int n, int stride,
                                                           long long ctrl_stride, double lambda, Acc* merged,
                                                           unsigned* counters, const __grid_constant__ TailArgs ta) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned s_ticket;
  const size_t m0 = merge_smem_bytes(n), m1 = fast_epilogue_smem_bytes<H>(ta.e.T);
  const size_t scratch = ((m0 > m1 ? m0 : m1) + 15) & ~size_t(15);
  unsigned char* pre = smem_raw + scratch;
  // plan, plant state and weights are not written by K1: fetch them while K1
  // may still be running (this kernel is its programmatic dependent)
  tail_prefetch<H>(ta.e, static_cast<const MlpParams<float, H>*>(ta.plant_w), blockIdx.y, pre);
  // everything below reads K1's output
  cudaGridDependencySynchronize();
  const int ctrl = blockIdx.y;
  Acc* row = merged + static_cast<size_t>(ctrl) * stride;
  merge_elements<kMergeBlock>(partials + static_cast<size_t>(ctrl) * ctrl_stride, n, stride, lambda, row, blockIdx.x,
                              gridDim.x, reinterpret_cast<double*>(smem_raw));
  // merge_elements' writes are thread 0's: its fence orders them before the ticket
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_ticket = atomicAdd(counters + ctrl, 1u);
  }
  __syncthreads();
  if (s_ticket != gridDim.x - 1) return;
  __threadfence();
  if (threadIdx.x == 0) counters[ctrl] = 0;
  epilogue_fast<H>(ta.e, row, ctrl, smem_raw, pre);
}

}  // namespace mppi_dev
