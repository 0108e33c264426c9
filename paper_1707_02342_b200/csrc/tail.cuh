// tail.cuh — the iteration tail fused into K1 (tensor-core path).
//
// K1 reduces each chunk of samples to softmin partials (rho_c, eta_c, bad_c,
// num_c[T][2]) relative to the chunk minimum.  Instead of two more kernels
// (pre-merge, epilogue) after K1, the warp that finishes LAST in each group of
// G chunks merges that group (in chunk order), and the warp that finishes the
// last group runs the whole epilogue of mpc_step for its controller
// (controller.cpp:137-146): merge of the group partials in group order,
// agg = num / eta, Savitzky-Golay (smoothing.cpp:48-65, mirror padding),
// U' = U + agg with the ControlPlan finiteness check (types.hpp:79-83),
// u0 = clamp(U'[0]), slide, ++iteration, and the device plant step of the
// closed loop.  "Last" is decided by a per-group / per-controller atomic
// ticket after a __threadfence, the classic threadfence-reduction pattern;
// every merge runs in a fixed order, so the result does not depend on which
// warp happens to finish last.  Counters reset themselves for the next launch.
//
// With samples sharded over ranks, K1 stops after the group merge (mode 1),
// the group partials are all-gathered, and tail_final_kernel runs the same
// final-merge + epilogue code on every rank: the arithmetic is identical to
// the single-GPU fused path, so the plan is bit-identical for any rank count
// whose chunk ranges are whole groups.
#pragma once

#include "epilogue.cuh"

namespace mppi_dev {

struct TailArgs {
  int mode;                       // 0: chunk partials only; 1: + group merge; 2: + final epilogue
  int G;                          // chunks per group
  int n_chunks;                   // chunks of the controller (all ranks)
  int n_groups;                   // groups of the controller (all ranks)
  long long groups_ctrl_stride;   // doubles per controller in `groups`
  unsigned* counters;             // [C][n_groups + 1]
  Acc* groups;                    // [C][n_groups][partial_stride]
  Acc* final_rows;                // [C][partial_stride]: the merged partial of the controller
  const MlpParams<float, 32>* plant_w;  // device plant weights (closed loop)
  EpilogueArgs<float> e;          // epilogue flags / state pointers (e.partials unused)
};

// Merge partial rows [r0, r1) of `P` (stride doubles each, r1 - r0 <= 256)
// into `out` (same row format), one warp: rho = min rho_r, then every element
// e >= 1 is sum_r exp(-(rho_r - rho)/lambda) * P[r][e] in ascending row
// order.  Lane l owns rows r0 + l + 32j (its own rows summed in order, then
// the 32 lane sums added in lane order through a transposed shared-memory
// block), so the row reads are contiguous per lane and many loads are in
// flight at once.  red: 32 x kRedStride doubles of scratch.
constexpr int kRedStride = 33;
__device__ __forceinline__ void warp_merge_rows(const Acc* P, int r0, int r1, int stride, double lambda, Acc* out,
                                                double* red, int lane) {
  constexpr int kMaxJ = 8;
  Acc m = INFINITY;
  bool bad = false;
  for (int r = r0 + lane; r < r1; r += 32) {
    const Acc* pr = P + static_cast<size_t>(r) * stride;
    const Acc rho = __ldcg(pr);
    m = (rho < m) ? rho : m;
    bad = bad || (__ldcg(pr + 2) != 0.0);
  }
  const Acc rho = warp_min(m);
  const bool any_bad = __any_sync(0xffffffffu, bad);
  double scale[kMaxJ];
#pragma unroll
  for (int j = 0; j < kMaxJ; ++j) {
    const int r = r0 + lane + 32 * j;
    scale[j] = (r < r1) ? exp(-(__ldcg(P + static_cast<size_t>(r) * stride) - rho) / lambda) : 0.0;
  }
  for (int eb = 0; eb < stride; eb += 32) {
    double v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = 0.0;
#pragma unroll
    for (int j = 0; j < kMaxJ; ++j) {
      const int r = r0 + lane + 32 * j;
      if (r < r1) {  // r >= r1 for every lane once j passes the last row: uniform exit
        const Acc* pr = P + static_cast<size_t>(r) * stride + eb;
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = fma(scale[j], (eb + e < stride) ? __ldcg(pr + e) : 0.0, v[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) red[e * kRedStride + lane] = v[e];
    __syncwarp();
    Acc sum = 0.0;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) sum = sum + red[lane * kRedStride + l];
    if (eb + lane < stride) out[eb + lane] = sum;
    __syncwarp();
  }
  if (lane == 0) {
    out[0] = rho;
    out[2] = any_bad ? 1.0 : 0.0;
    out[3] = 0.0;
  }
  __syncwarp();
}

// Final merge over the group partials + the epilogue of mpc_step, one warp.
// `fin` is a global row (stride doubles) for the merged partial; red: the
// warp's 32 x kRedStride scratch.
template <int kUnused = 0>
__device__ __noinline__ void tail_final_warp(const TailArgs& ta, int ctrl, int T, int partial_stride,
                                             double lambda, double* red, int lane) {
  const EpilogueArgs<float>& e = ta.e;
  StepStatus* st = e.status + ctrl;
  if (__ldcg(&st->code) != 0) return;
  const Acc* Gp = ta.groups + static_cast<size_t>(ctrl) * ta.groups_ctrl_stride;
  Acc* fin = ta.final_rows + static_cast<size_t>(ctrl) * partial_stride;
  warp_merge_rows(Gp, 0, ta.n_groups, partial_stride, lambda, fin, red, lane);
  if (fin[2] != 0.0) {
    if (lane == 0) st->code = 2;  // it_weights: non-finite cost (weights.cpp:12)
    return;
  }
  const Acc eta = fin[1];
  double* agg = red;                                        // 2T doubles
  float* s_new = reinterpret_cast<float*>(red + 2 * T);     // 2T floats (T <= 256)
  for (int i = lane; i < 2 * T; i += 32) agg[i] = fin[kPartialHeader + i] / eta;
  __syncwarp();
  // SG smoothing of agg = num / eta, then U' = U + SG(agg) in double, rounded once
  float* plan = e.plan + static_cast<size_t>(ctrl) * 2 * T;
  const int half = e.sg_window / 2;
  bool nonfinite = false;
  for (int i = lane; i < 2 * T; i += 32) {
    const int t = i >> 1, c = i & 1;
    Acc v;
    if (e.sg_window > 0) {
      Acc acc = 0.0;
      for (int j = -half; j <= half; ++j)
        acc = __dadd_rn(acc, __dmul_rn(e.sg[j + half], agg[reflect_index(t + j, T) * 2 + c]));
      v = acc;
    } else {
      v = agg[i];
    }
    const float nv = static_cast<float>(__dadd_rn(static_cast<Acc>(plan[i]), v));
    nonfinite = nonfinite || !isfinite(nv);
    s_new[i] = nv;
  }
  if (__any_sync(0xffffffffu, nonfinite)) {
    if (lane == 0) st->code = 1;  // ControlPlan rejects non-finite plans
    return;
  }
  __syncwarp();
  const float u0 = clamp_r(s_new[0], e.lo0, e.hi0), u1 = clamp_r(s_new[1], e.lo1, e.hi1);
  for (int i = lane; i < 2 * T; i += 32) plan[i] = e.slide ? ((i + 2 < 2 * T) ? s_new[i + 2] : 0.f) : s_new[i];
  uint64_t it = e.iters[ctrl];
  if (e.increment) it += 1;
  if (lane == 0) {
    st->u0[0] = static_cast<double>(u0);
    st->u0[1] = static_cast<double>(u1);
    if (e.u_trace) {
      const uint64_t idx = it - 1 - e.trace_base[ctrl];
      e.u_trace[(idx * e.n_ctrl + ctrl) * 2] = u0;
      e.u_trace[(idx * e.n_ctrl + ctrl) * 2 + 1] = u1;
    }
  }
  if (e.plant) {
    // the device plant: the same MLP model stepped with the executed input
    // (operation order of epilogue_kernel: lane j = hidden unit j)
    float* x = e.x0 + static_cast<size_t>(ctrl) * 8;
    const MlpParams<float, 32>& w = *ta.plant_w;
    const float in[6] = {x[3], x[4], x[5], x[6], u0, u1};
    float acc = w.b1[lane];
#pragma unroll
    for (int i = 0; i < 6; ++i) acc = fma_r(w.w1t[i][lane], in[i], acc);
    const float h1 = tanh_r(acc);
    acc = w.b2[lane];
#pragma unroll 8
    for (int i = 0; i < 32; ++i) acc = fma_r(w.w2t[i][lane], __shfl_sync(0xffffffffu, h1, i), acc);
    const float h2 = tanh_r(acc);
    float d = (lane < 4) ? w.b3[lane] : 0.f;
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
      const float hi = __shfl_sync(0xffffffffu, h2, i);
      if (lane < 4) d = fma_r(w.w3t[i][lane], hi, d);
    }
    float dd[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) dd[o] = __shfl_sync(0xffffffffu, d, o);
    if (lane == 0) {
      float xs[7];
      for (int i = 0; i < 7; ++i) xs[i] = x[i];
      advance_split<float>(xs, dd, e.sys.dt);
      for (int i = 0; i < 7; ++i) x[i] = xs[i];
      for (int i = 0; i < 8; ++i) st->x[i] = static_cast<double>(x[i]);
      if (e.x_trace) {
        const uint64_t idx = it - e.trace_base[ctrl];
        for (int i = 0; i < 8; ++i) e.x_trace[(idx * e.n_ctrl + ctrl) * 8 + i] = x[i];
      }
    }
  }
  if (lane == 0) {
    e.iters[ctrl] = it;
    st->iteration = it;
  }
}

// Called by every warp of K1 after it wrote its chunk partial `chunk` (all
// lanes).  scratch: per-warp shared memory (see tail_final_warp).
__device__ __forceinline__ void tail_after_chunk(const TailArgs& ta, int ctrl, int chunk, int T, int partial_stride,
                                                 long long partials_ctrl_stride, const Acc* partials, double lambda,
                                                 double* scratch, int lane) {
  if (ta.mode == 0) return;
  __threadfence();
  __syncwarp();
  unsigned* cnt = ta.counters + static_cast<size_t>(ctrl) * (ta.n_groups + 1);
  const int grp = chunk / ta.G;
  const int c0 = grp * ta.G, c1 = min(ta.n_chunks, c0 + ta.G);
  unsigned ticket = 0;
  if (lane == 0) ticket = atomicAdd(cnt + grp, 1u);
  ticket = __shfl_sync(0xffffffffu, ticket, 0);
  if (ticket != static_cast<unsigned>(c1 - c0 - 1)) return;  // not the last chunk of the group
  __threadfence();
  Acc* gout = ta.groups + static_cast<size_t>(ctrl) * ta.groups_ctrl_stride + static_cast<size_t>(grp) * partial_stride;
  warp_merge_rows(partials + static_cast<size_t>(ctrl) * partials_ctrl_stride, c0, c1, partial_stride, lambda, gout,
                  scratch, lane);
  if (lane == 0) cnt[grp] = 0;  // reset for the next launch
  if (ta.mode < 2) return;
  __threadfence();
  __syncwarp();
  if (lane == 0) ticket = atomicAdd(cnt + ta.n_groups, 1u);
  ticket = __shfl_sync(0xffffffffu, ticket, 0);
  if (ticket != static_cast<unsigned>(ta.n_groups - 1)) return;
  __threadfence();
  tail_final_warp<>(ta, ctrl, T, partial_stride, lambda, scratch, lane);
  if (lane == 0) cnt[ta.n_groups] = 0;
}

// Ranks > 1: the final merge + epilogue after the all-gather of group
// partials (one warp per controller; same code as the fused path).
template <int kUnused = 0>
__global__ void __launch_bounds__(32) tail_final_kernel(const __grid_constant__ TailArgs ta, int T,
                                                        int partial_stride, double lambda) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  tail_final_warp<>(ta, blockIdx.x, T, partial_stride, lambda, reinterpret_cast<double*>(smem_raw), threadIdx.x);
}

}  // namespace mppi_dev
