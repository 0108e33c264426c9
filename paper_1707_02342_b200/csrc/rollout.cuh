// rollout.cuh — K1: fused rollout + chunk-level softmin partials.
//
// One CTA owns one chunk of BLOCK consecutive global sample indices; one thread
// owns one sample.  Per thread: T steps of {eps from the counter stream (or the
// injected batch), zero-mean rewrite, v = u + eps, coupling, clamp, MLP
// dynamics, Euler split, costmap lookup, state cost} — rollout_batch,
// controller.cpp:55-109 — then the terminal cost.  The CTA then reduces its
// chunk to (rho_c = min S, eta_c = sum exp(-(S - rho_c)/lambda),
// num_c[t][c] = sum exp(-(S - rho_c)/lambda) eps'[t][c]) where eps' is the batch
// as rollout_batch leaves it (eps - U for zero-mean samples,
// controller.cpp:70-72).  eps' is REGENERATED from the counters for the
// numerator, so the K x T x 2 batch never touches HBM.  The per-chunk
// partials are merged into fixed groups (group.cuh) and the group rows in
// group order by K2 (epilogue.cuh), which makes the result independent of the
// GPU count and of scheduling.
#pragma once

#include "model.cuh"
#include "noise.cuh"

namespace mppi_dev {

constexpr int kPartialHeader = 4;  // rho, eta, bad, reserved

// Mixed precision: the per-step dynamics and cost terms run in R (fp32 in
// production); the T-term cost sum, the softmin (rho, eta, w) and the
// weighted-noise numerators are accumulated in double.  With costs ~1e5 an
// fp32 running sum carries ~0.1 absolute error, which lambda = 6.66 turns into
// ~1% weight error; the double accumulators cost O(K T) adds against the
// O(K T H^2) FMAs of the MLP.
using Acc = double;

template <class R>
struct RolloutArgs {
  int K, T;
  int zero_start;         // samples k >= zero_start are zero-mean (sampler.cpp:36-37)
  int chunk0;             // global chunk index of blockIdx.x == 0 (rank offset)
  int chunk_end;          // one past the last chunk of this rank (tensor-core kernel)
  int partial_stride;     // kPartialHeader + 2T
  long long partials_ctrl_stride;
  R lambda, gamma, sigma0, sigma1, scale0, scale1;
  double dscale0, dscale1, dlambda;
  SystemArgs<R> sys;
  const R* plan;          // [C][T][2]
  const R* x0;            // [C][8]
  const R* const* maps;   // [C] value pointers (nullptr for map-less systems)
  int map_w, map_h;
  R map_x0, map_y0, map_res, map_inv_res;
  const R* inj;           // injected batch, device layout [T][K][2]
  const uint64_t* seeds;  // [C]
  const uint64_t* iters;  // [C]
  const int* abort_flag;  // sticky status code of controller c at abort_flag[c * abort_stride]: nonzero -> skip
  int abort_stride;       // ints between consecutive controllers' codes (sizeof(StepStatus) / 4)
  Acc* costs;             // [C][K]
  Acc* partials;          // [C][chunks][partial_stride]
  R* trace_states;        // (T+1) x 7 trajectory of sample trace_k (or nullptr)
  int trace_k;
  int pdl;                // host: launch K1 as a programmatic dependent (tensor-core path)
};

// The step graph's first node on the tensor-core path: the controllers'
// states from the mapped pinned host buffer into device memory, one float4
// (half a controller's 8-float row) per thread, every PCIe read in flight at
// once, with K1 launched as its programmatic dependent.  (A one-warp loop
// over C x 8 floats serialised C / 4 PCIe round trips per thread: ~0.2 ms
// for the 512-controller c3 fleet.)
template <int kUnused = 0>
__global__ void fetch_x0_kernel(const float4* __restrict__ host_x0, float4* __restrict__ x0, int n4) {
  cudaTriggerProgrammaticLaunchCompletion();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n4) x0[i] = host_x0[i];
}
constexpr int kFetchX0Block = 256;

template <class R, int Mode>
__device__ __forceinline__ NoiseStream<R, Mode> make_noise(const RolloutArgs<R>& a, int ctrl, int k) {
  NoiseStream<R, Mode> ns;
  ns.scale0 = a.scale0;
  ns.scale1 = a.scale1;
  ns.dscale0 = a.dscale0;
  ns.dscale1 = a.dscale1;
  ns.inj = a.inj;
  ns.K = a.K;
  ns.k = static_cast<uint32_t>(k);
  const uint64_t it = a.iters[ctrl];
  const uint64_t seed = a.seeds[ctrl];
  ns.seed = seed;
  ns.iteration = it;
  if constexpr (Mode == kRefSplitmix) ns.prefix = ref_hash_prefix(seed, it);
  ns.z2 = R(0);
  ns.z3 = R(0);
  return ns;
}

// Rollout of one sample (the body of the rollout_batch k-loop).  If
// `states_out` is non-null, the (T+1) x state_dim trajectory is written.
template <class R, int H, class Sys, int Mode>
__device__ __forceinline__ Acc rollout_one(const RolloutArgs<R>& a, const MlpParams<R, H>& w,
                                         const R* __restrict__ plan, int ctrl, int k,
                                         R* states_out) {
  NoiseStream<R, Mode> ns = make_noise<R, Mode>(a, ctrl, k);
  const bool zm = k >= a.zero_start;
  R x[7];
#pragma unroll
  for (int i = 0; i < 7; ++i) x[i] = (i < Sys::kStateDim) ? a.x0[ctrl * 8 + i] : R(0);
  if (states_out)
    for (int i = 0; i < Sys::kStateDim; ++i) states_out[i] = x[i];
  MapDev<R> map;
  if constexpr (Sys::kHasMap) {
    map.values = a.maps[ctrl];
    map.width = a.map_w;
    map.height = a.map_h;
    map.x0 = a.map_x0;
    map.y0 = a.map_y0;
    map.res = a.map_res;
    map.inv_res = a.map_inv_res;
  }
  const R half_lambda = mul_rn(R(0.5), a.lambda);
  const R gml = sub_rn(a.gamma, a.lambda);
  Acc cost = 0.0;
  // The running cost of step t needs the costmap at x_{t+1}; its four taps are
  // fetched right after the step and consumed one MLP later, hiding the L2
  // latency behind the next step's FMAs.
  MapTaps<R> q{};
  R p_roll = R(0), p_vx = R(0), p_vy = R(0), p_coup = R(0);
  for (int t = 0; t < a.T; ++t) {
    const R u0 = plan[2 * t], u1 = plan[2 * t + 1];
    R e0, e1;
    ns.eps(t, e0, e1);
    if (zm) {
      e0 = sub_rn(e0, u0);
      e1 = sub_rn(e1, u1);
    }
    const R v0 = add_rn(u0, e0), v1 = add_rn(u1, e1);
    R uv = div_r(mul_rn(u0, v0), a.sigma0);
    uv = add_rn(uv, div_r(mul_rn(u1, v1), a.sigma1));
    R coupling;
    if (zm) {
      R uu = div_r(mul_rn(u0, u0), a.sigma0);
      uu = add_rn(uu, div_r(mul_rn(u1, u1), a.sigma1));
      coupling = add_rn(mul_rn(gml, uv), mul_rn(half_lambda, uu));
    } else {
      coupling = mul_rn(a.gamma, uv);
    }
    Sys::step(x, v0, v1, w, a.sys);
    if (states_out)
      for (int i = 0; i < Sys::kStateDim; ++i) states_out[(t + 1) * Sys::kStateDim + i] = x[i];
    if constexpr (Sys::kHasMap) {
      if (t > 0) {
        const R h = map_interp(q);
        const R rc = state_cost_h(h, p_roll, p_vx, p_vy, a.sys.decay_pow[t - 1], a.sys.cost);
        cost += static_cast<Acc>(add_rn(rc, p_coup));
      }
      q = map_fetch(map, x[0], x[1]);
      p_roll = x[3];
      p_vx = x[4];
      p_vy = x[5];
      p_coup = coupling;
    } else {
      cost += static_cast<Acc>(add_rn(Sys::cost(x, a.sys), coupling));
    }
  }
  if constexpr (Sys::kHasMap) {
    const R h = map_interp(q);
    const R rc = state_cost_h(h, p_roll, p_vx, p_vy, a.sys.decay_pow[a.T - 1], a.sys.cost);
    cost += static_cast<Acc>(add_rn(rc, p_coup));
    // terminal cost = state_cost(x_T, T) (controller.cpp:27-30): same taps.
    if (a.sys.with_terminal)
      cost += static_cast<Acc>(state_cost_h(h, p_roll, p_vx, p_vy, a.sys.decay_pow[a.T], a.sys.cost));
  }
  return cost;
}

template <class R, int BLOCK>
__device__ __forceinline__ R block_min(R v, R* s_red) {
  v = warp_min(v);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) s_red[wid] = v;
  __syncthreads();
  R r = s_red[0];
#pragma unroll
  for (int i = 1; i < BLOCK / 32; ++i) r = (s_red[i] < r) ? s_red[i] : r;
  return r;
}
// Deterministic block sum: xor-butterfly within warps, then warps in order.
template <class R, int BLOCK>
__device__ __forceinline__ R block_sum(R v, R* s_red) {
  v = warp_sum(v);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) s_red[wid] = v;
  __syncthreads();
  R r = s_red[0];
#pragma unroll
  for (int i = 1; i < BLOCK / 32; ++i) r = r + s_red[i];
  return r;
}

// K1.  grid = (chunks of this rank, controllers), block = BLOCK samples.
// Dynamic smem: per-warp numerators (BLOCK/32 x 2T, double) + plan (2T, R).
template <class R, int H, class Sys, int Mode, int BLOCK>
__global__ void __launch_bounds__(BLOCK) rollout_kernel(const __grid_constant__ RolloutArgs<R> a,
                                                        const __grid_constant__ WeightHolder<R, H> wh) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Acc* s_num = reinterpret_cast<Acc*>(smem_raw);
  R* s_plan = reinterpret_cast<R*>(s_num + (BLOCK / 32) * 2 * a.T);
  __shared__ Acc s_red[BLOCK / 32];
  const int ctrl = blockIdx.y;
  if (a.abort_flag[static_cast<size_t>(ctrl) * a.abort_stride] != 0) return;
  const int chunk = a.chunk0 + blockIdx.x;
  const int k = chunk * BLOCK + threadIdx.x;
  const bool valid = k < a.K;
  const int T = a.T;
  for (int i = threadIdx.x; i < 2 * T; i += BLOCK) s_plan[i] = a.plan[static_cast<size_t>(ctrl) * 2 * T + i];
  __syncthreads();

  Acc cost = 0.0;
  if (valid) {
    cost = rollout_one<R, H, Sys, Mode>(a, wh.get(), s_plan, ctrl, k, nullptr);
    a.costs[static_cast<size_t>(ctrl) * a.K + k] = cost;
  }
  const bool bad = valid && !isfinite(cost);
  const int any_bad = __syncthreads_or(bad);
  const Acc rho = block_min<Acc, BLOCK>(valid ? cost : Acc(INFINITY), s_red);
  // it_weights (weights.cpp:15-23) relative to the chunk minimum.
  const Acc wk = valid ? exp(-(cost - rho) / a.dlambda) : 0.0;
  const Acc eta = block_sum<Acc, BLOCK>(wk, s_red);

  // Weighted numerator over the regenerated batch.
  NoiseStream<R, Mode> ns = make_noise<R, Mode>(a, ctrl, valid ? k : 0);
  const bool zm = k >= a.zero_start;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = 0; t < T; ++t) {
    R e0 = R(0), e1 = R(0);
    if (valid) {
      ns.eps(t, e0, e1);
      if (zm) {
        e0 = sub_rn(e0, s_plan[2 * t]);
        e1 = sub_rn(e1, s_plan[2 * t + 1]);
      }
    }
    const Acc n0 = warp_sum(wk * static_cast<Acc>(e0));
    const Acc n1 = warp_sum(wk * static_cast<Acc>(e1));
    if (lane == 0) {
      s_num[(wid * T + t) * 2] = n0;
      s_num[(wid * T + t) * 2 + 1] = n1;
    }
  }
  __syncthreads();
  Acc* out = a.partials + static_cast<size_t>(ctrl) * a.partials_ctrl_stride +
             static_cast<size_t>(chunk) * a.partial_stride;
  MPPI_DCHECK(static_cast<long long>(chunk + 1) * a.partial_stride <= a.partials_ctrl_stride);
  for (int i = threadIdx.x; i < 2 * T; i += BLOCK) {
    Acc s = s_num[i];
#pragma unroll
    for (int w2 = 1; w2 < BLOCK / 32; ++w2) s = s + s_num[w2 * 2 * T + i];
    out[kPartialHeader + i] = s;
  }
  if (threadIdx.x == 0) {
    out[0] = rho;
    out[1] = eta;
    out[2] = any_bad ? 1.0 : 0.0;
    out[3] = 0.0;
  }
}

// Single-sample trajectory (parity: state trajectories step by step).
template <class R, int H, class Sys, int Mode>
__global__ void rollout_states_kernel(const __grid_constant__ RolloutArgs<R> a,
                                      const __grid_constant__ WeightHolder<R, H> wh, int k,
                                      R* states_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  rollout_one<R, H, Sys, Mode>(a, wh.get(), a.plan, 0, k, states_out);
}

// The batch as rollout_batch leaves it, in the reference layout (double):
// eps[k][c][t], zero-mean samples rewritten to eps - U.
template <class R, int Mode>
__global__ void materialize_batch_kernel(const __grid_constant__ RolloutArgs<R> a, int rewrite,
                                         double* eps_out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.K) return;
  NoiseStream<R, Mode> ns = make_noise<R, Mode>(a, 0, k);
  const bool zm = rewrite && k >= a.zero_start;
  for (int t = 0; t < a.T; ++t) {
    R e0, e1;
    ns.eps(t, e0, e1);
    if (zm) {
      e0 = sub_rn(e0, a.plan[2 * t]);
      e1 = sub_rn(e1, a.plan[2 * t + 1]);
    }
    eps_out[(static_cast<size_t>(k) * 2 + 0) * a.T + t] = static_cast<double>(e0);
    eps_out[(static_cast<size_t>(k) * 2 + 1) * a.T + t] = static_cast<double>(e1);
  }
}

// update_plan aggregation (controller.cpp:124-128) with caller weights:
// agg[t][c] = sum_k w_k eps'_k[t][c], ascending k, zero weights skipped,
// unfused multiply then add (bit-identical to the sequential reference loop).
// One thread per timestep; eps' regenerated per (k, t).
template <class R, int Mode>
__global__ void weighted_agg_kernel(const __grid_constant__ RolloutArgs<R> a,
                                    const Acc* __restrict__ w, Acc* agg) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.T) return;
  const uint64_t it = a.iters[0], seed = a.seeds[0];
  Acc s0 = 0.0, s1 = 0.0;
  const R u0 = a.plan[2 * t], u1 = a.plan[2 * t + 1];
  const uint64_t prefix = ref_hash_prefix(seed, it);
  for (int k = 0; k < a.K; ++k) {
    const Acc wk = w[k];
    if (wk == 0.0) continue;
    R e0, e1;
    if constexpr (Mode == kInjected) {
      e0 = a.inj[(static_cast<size_t>(t) * a.K + k) * 2];
      e1 = a.inj[(static_cast<size_t>(t) * a.K + k) * 2 + 1];
    } else if constexpr (Mode == kRefSplitmix) {
      double z0, z1;
      ref_normal_pair(prefix, static_cast<uint64_t>(k), static_cast<uint64_t>(t), z0, z1);
      e0 = static_cast<R>(a.dscale0 * z0);
      e1 = static_cast<R>(a.dscale1 * z1);
    } else {
      const uint4 d = philox_draw(seed, it, static_cast<uint32_t>(k), static_cast<uint32_t>(t) >> 1);
      R z0, z1;
      if (t & 1) philox_box_muller(d.z, d.w, z0, z1);
      else philox_box_muller(d.x, d.y, z0, z1);
      e0 = a.scale0 * z0;
      e1 = a.scale1 * z1;
    }
    if (k >= a.zero_start) {
      e0 = sub_rn(e0, u0);
      e1 = sub_rn(e1, u1);
    }
    s0 = __dadd_rn(s0, __dmul_rn(wk, static_cast<Acc>(e0)));
    s1 = __dadd_rn(s1, __dmul_rn(wk, static_cast<Acc>(e1)));
  }
  agg[2 * t] = s0;
  agg[2 * t + 1] = s1;
}

// Reference layout (double, [k][c][t]) -> device layout (R, [T][K][2]).
template <class R>
__global__ void inject_transpose_kernel(const double* __restrict__ ref, int K, int T, R* dev) {
  const size_t n = static_cast<size_t>(K) * T;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % K);
    const int t = static_cast<int>(i / K);
    dev[i * 2] = static_cast<R>(ref[(static_cast<size_t>(k) * 2) * T + t]);
    dev[i * 2 + 1] = static_cast<R>(ref[(static_cast<size_t>(k) * 2 + 1) * T + t]);
  }
}

}  // namespace mppi_dev
