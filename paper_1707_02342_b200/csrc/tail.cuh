// tail.cuh — the iteration tail of the tensor-core path: merge of the group
// softmin partials, then the epilogue of mpc_step, in ONE CTA per controller.
//
// The chunk partials of K1 are first merged into a fixed set of group rows
// (group.cuh); on N > 1 ranks the group rows are all-gathered.  This tail
// merges the G group rows (G = 8 at c0/c1, at most a few hundred at K = 2^20):
//   rho = min_g rho_g,  merged[e] = sum_g exp(-(rho_g - rho) / lambda) P[g][e]
// with one thread per element summing the rows in group order — an order that
// depends only on G, never on the rank count — into shared memory, and then
// runs the epilogue on the merged row in the same CTA: no second launch, no
// ticket, no global round trip for the merged row.
#pragma once

#include <algorithm>

#include "epilogue.cuh"

namespace mppi_dev {

constexpr int kTailBlock = 256;  // threads of the tail CTA (>= the 4 + 2T elements at T <= 126)

struct TailArgs {
  const void* plant_w;                  // MlpParams<float, H> of the model (device plant)
  EpilogueArgs<float> e;                // epilogue over the merged row (n_chunks = 1)
};

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
  for (int i = threadIdx.x; i < 2 * T; i += kTailBlock) s_plan[i] = plan[i];
  if (threadIdx.x < 8) s_x[threadIdx.x] = a.x0[static_cast<size_t>(ctrl) * 8 + threadIdx.x];
  if (a.plant) {
    const float4* src = reinterpret_cast<const float4*>(w_src);
    float4* dst = reinterpret_cast<float4*>(s_w);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(MlpParams<float, H>) / 16); i += kTailBlock)
      dst[i] = src[i];
  }
}
// The finished status of controller ctrl into the mapped host mirror (one
// thread; its own earlier writes to *st are ordered before these reads): the
// step graph then needs no device-to-host copy node.
// Then the sequence word: seq0 + 1, after a system-scope fence, so a host that
// sees the new sequence sees every field of this step.
__device__ __forceinline__ void publish_status(const EpilogueArgs<float>& a, int ctrl, unsigned long long seq0) {
  if (!a.status_host) return;
  const StepStatus* st = a.status + ctrl;
  StepStatus* sh = a.status_host + ctrl;
  sh->code = st->code;
  sh->u0[0] = st->u0[0];
  sh->u0[1] = st->u0[1];
#pragma unroll
  for (int i = 0; i < 8; ++i) sh->x[i] = st->x[i];
  sh->iteration = st->iteration;
  __threadfence_system();
  *reinterpret_cast<volatile unsigned long long*>(&sh->seq) = seq0 + 1;
}

template <int H>
__device__ __forceinline__ void epilogue_fast(const EpilogueArgs<float>& a, const Acc* s_row, int bad, int ctrl,
                                              unsigned char* smem, const unsigned char* pre, int code0, uint64_t it0,
                                              unsigned long long seq0) {
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
  for (int j = threadIdx.x; j < a.sg_window; j += kTailBlock) s_sg[j] = a.sg[j];
  StepStatus* st = a.status + ctrl;
  float* plan = a.plan + static_cast<size_t>(ctrl) * 2 * T;
  // ---- phase 1: the merged row (shared memory) and the status (prefetched
  // before the grid dependency with the plan, the plant state and the weights)
  if (threadIdx.x == 0) {
    int code = code0;
    if (code == 0 && bad) code = 2;  // it_weights: non-finite cost (weights.cpp:12)
    s_code = code;
  }
  const double inv_eta = 1.0 / s_row[1];
  for (int i = threadIdx.x; i < 2 * T; i += kTailBlock)
    s_agg[i] = s_row[kPartialHeader + i] * inv_eta;  // agg = num / eta
  __syncthreads();
  if (s_code != 0) {
    if (threadIdx.x == 0) {
      if (__ldcg(&st->code) == 0) st->code = s_code;
      publish_status(a, ctrl, seq0);
    }
    return;
  }
  // ---- SG smoothing of agg, U' = U + SG(agg)
  const int half = a.sg_window / 2;
  int nonfinite = 0;
  for (int i = threadIdx.x; i < 2 * T; i += kTailBlock) {
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
      publish_status(a, ctrl, seq0);
    }
    return;
  }
  const float u0 = clamp_r(s_new[0], a.lo0, a.hi0), u1 = clamp_r(s_new[1], a.lo1, a.hi1);
  for (int i = threadIdx.x; i < 2 * T; i += kTailBlock)
    plan[i] = a.slide ? ((i + 2 < 2 * T) ? s_new[i + 2] : 0.f) : s_new[i];
  uint64_t it = it0;
  if (a.increment) it += 1;
  if (threadIdx.x == 0) MPPI_STAMP_MIN(5);  // SG + U' + plan written (thread 0)
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
    // the plant step of the same MLP by warp 0: lane j owns hidden units
    // j, j + 32, ...; activations go through shared memory (broadcast reads,
    // so every FMA chain has its operands without a shuffle round trip);
    // per unit the operation order is that of epilogue_kernel
    __shared__ float s_h[2 * H];
    __shared__ float s_d[4];
    const MlpParams<float, H>& w = *s_w;
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = s_x[i];
    const float in[6] = {x[3], x[4], x[5], x[6], u0, u1};
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = lane + 32 * u;
      float acc = w.b1[j];
#pragma unroll
      for (int i = 0; i < 6; ++i) acc = fma_r(w.w1t[i][j], in[i], acc);
      s_h[j] = tanh_r(acc);
    }
    __syncwarp();
    // (every operand of a unit's FMA chain is loaded before the chain starts:
    // one shared-memory round trip instead of one per unrolled batch; the
    // chain itself keeps the per-unit order)
    float hv[H];
#pragma unroll
    for (int i = 0; i < H; ++i) hv[i] = s_h[i];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = lane + 32 * u;
      float wv[H];
#pragma unroll
      for (int i = 0; i < H; ++i) wv[i] = w.w2t[i][j];
      float acc = w.b2[j];
#pragma unroll
      for (int i = 0; i < H; ++i) acc = fma_r(wv[i], hv[i], acc);
      s_h[H + j] = tanh_r(acc);
    }
    __syncwarp();
    if (lane < 4) {
      float wv[H], h2[H];
#pragma unroll
      for (int i = 0; i < H; ++i) {
        wv[i] = w.w3t[i][lane];
        h2[i] = s_h[H + i];
      }
      float d = w.b3[lane];
#pragma unroll
      for (int i = 0; i < H; ++i) d = fma_r(wv[i], h2[i], d);
      s_d[lane] = d;
    }
    __syncwarp();
    if (lane == 0) {
      float dd[4] = {s_d[0], s_d[1], s_d[2], s_d[3]};
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
  if (lane == 0) MPPI_STAMP_MIN(6);  // plant done
  if (lane == 0) {
    a.iters[ctrl] = it;
    st->iteration = it;
    publish_status(a, ctrl, seq0);
  }
}

// The tensor-core path's tail: grid = (1, controllers), block = kTailBlock.
// rows: [C][n][stride] group rows.  smem: tail_smem_bytes<H>(n, T).
template <int H>
__host__ __device__ constexpr size_t tail_smem_bytes(int n, int T) {
  const size_t merge = sizeof(double) * (n + kPartialHeader + 2 * T);  // scales + the merged row
  const size_t epi = fast_epilogue_smem_bytes<H>(T);
  return ((merge + epi + 15) & ~size_t(15)) + tail_pre_bytes<H>(T);
}
template <int H>
__global__ void __launch_bounds__(kTailBlock) tail_kernel(const Acc* __restrict__ rows, int n, int stride,
                                                          long long ctrl_stride, double lambda,
                                                          const __grid_constant__ TailArgs ta) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Acc s_min[kTailBlock / 32];
  const int T = ta.e.T;
  Acc* s_scale = reinterpret_cast<Acc*>(smem_raw);
  Acc* s_row = s_scale + n;
  unsigned char* epi = reinterpret_cast<unsigned char*>(s_row + stride);
  unsigned char* pre = smem_raw + ((sizeof(double) * (n + stride) + fast_epilogue_smem_bytes<H>(T) + 15) & ~size_t(15));
  const int ctrl = blockIdx.y;
  // plan, plant state and weights are not written by the group merge: fetch
  // them while it may still be running (this kernel is its programmatic dependent)
  tail_prefetch<H>(ta.e, static_cast<const MlpParams<float, H>*>(ta.plant_w), ctrl, pre);
  // the sticky status and the iteration counter are not written by K1 or the
  // group merge either (a failed step clears the status before the next one)
  const int code0 = (threadIdx.x == 0) ? __ldcg(&ta.e.status[ctrl].code) : 0;
  const uint64_t it0 = ta.e.iters[ctrl];
  // the host mirror's sequence word (a PCIe read, hidden behind the wait)
  const unsigned long long seq0 =
      (threadIdx.x == 0 && ta.e.status_host)
          ? *reinterpret_cast<const volatile unsigned long long*>(&ta.e.status_host[ctrl].seq)
          : 0ull;
  cudaGridDependencySynchronize();  // everything below reads the group rows
  if (threadIdx.x == 0) MPPI_STAMP_MIN(3);
  const Acc* P = rows + static_cast<size_t>(ctrl) * ctrl_stride;
  MPPI_DCHECK(static_cast<long long>(n) * stride <= ctrl_stride && stride == kPartialHeader + 2 * T);
  // rho = min over the group rows, bad = any group non-finite
  Acc m = INFINITY;
  int bad = 0;
  for (int r = threadIdx.x; r < n; r += kTailBlock) {
    const Acc rr = __ldcg(P + static_cast<size_t>(r) * stride);
    bad |= __ldcg(P + static_cast<size_t>(r) * stride + 2) != 0.0;
    m = (rr < m) ? rr : m;
    s_scale[r] = rr;
  }
  m = warp_min(m);
  if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = m;
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) MPPI_STAMP_MIN(7);  // group minima loaded
  Acc rho = s_min[0];
#pragma unroll
  for (int w = 1; w < kTailBlock / 32; ++w) rho = (s_min[w] < rho) ? s_min[w] : rho;
  const double inv_lambda = 1.0 / lambda;
  for (int r = threadIdx.x; r < n; r += kTailBlock) s_scale[r] = exp(-(s_scale[r] - rho) * inv_lambda);
  __syncthreads();
  if (threadIdx.x == 0) MPPI_STAMP_MIN(8);  // scales
  // merged element e (eta and the numerators): the rows in group order
  for (int e = threadIdx.x; e < stride; e += kTailBlock) {
    if (e == 1 || e >= kPartialHeader) {
      Acc acc = 0.0;
      const Acc* pe = P + e;
#pragma unroll 8
      for (int r = 0; r < n; ++r) acc = fma(s_scale[r], __ldcg(pe + static_cast<size_t>(r) * stride), acc);
      s_row[e] = acc;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) MPPI_STAMP_MIN(4);  // merged row in shared memory
  epilogue_fast<H>(ta.e, s_row, bad, ctrl, epi, pre, code0, it0, seq0);
#ifdef MPPI_STAMPS
  if (threadIdx.x == 0) {
    volatile unsigned long long* s = g_stamps;
    const unsigned long long e = gtimer();
    printf("STAMPS k1_end->tail_start %lld rho_loads %lld scales %lld elements %lld sg_plan %lld plant %lld status %lld ns\n",
           static_cast<long long>(s[3] - s[0]), static_cast<long long>(s[7] - s[3]),
           static_cast<long long>(s[8] - s[7]), static_cast<long long>(s[4] - s[8]),
           static_cast<long long>(s[5] - s[4]), static_cast<long long>(s[6] - s[5]), static_cast<long long>(e - s[6]));
    s[0] = 0;
    s[3] = ~0ull; s[4] = ~0ull; s[5] = ~0ull; s[6] = ~0ull; s[7] = ~0ull; s[8] = ~0ull;
  }
#endif
}

}  // namespace mppi_dev
