// rollout_ws.cuh — K1 production variant: warp-specialised fp32 rollout.
//
// The generic K1 (rollout.cuh) gives each thread one whole sample, which at
// the BASELINE sizes leaves < 1 warp per SM sub-partition (K = 16384 -> 512
// warps for 592 SMSPs) and runs latency-bound.  Here a CTA of L warps owns one
// group of 32 samples (lane = sample) and the MLP is split by hidden unit:
// warp r computes units [r H/L, (r+1) H/L) for all 32 samples, so every
// weight an instruction reads is warp-uniform and comes through the uniform
// datapath (LDCU -> FFMA2 uniform-register operand), while L x more warps hide
// each other's latency.  Per step:
//
//   A  inputs (dynamic state, clamped v_t from shared memory)
//   B  layer 1 for own units, tanh, h1 -> smem                 | barrier 1
//   D  layer 2 for own units over all H h1 (LDS.128), tanh,
//      layer-3 partial sums of own units -> smem               | barrier 2
//   F  d = b3 + sum_r partial_r (fixed order: identical in every warp),
//      Euler update of the dynamic block (all warps, registers)
//   G  role 0: kinematic update, costmap taps, running cost of step t-1;
//      role 1: noise, zero-mean rewrite, v_{t+1}, clamp, coupling (before
//      barrier 2 of step t, consumed after it).
//
// MLP arithmetic is fp32 with paired fma.rn.f32x2 (one FFMA2 = two outputs);
// tanh(x) = 1 - 2 / (1 + 2^(2x log2 e)) with ex2.approx / rcp.approx
// (|error| <= ~3e-7, checked against the oracle's std::tanh in the parity
// tests).  The cost sum, softmin and numerators are double (Acc).
#pragma once

#include "rollout.cuh"

namespace mppi_dev {

// d = a * b + c on a pair of fp32 lanes (sm_100 FFMA2), round-to-nearest.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// tanh on a pair: 1 - 2 / (1 + 2^(2 x log2 e)); saturates correctly at
// +-inf (ex2 -> inf -> rcp -> 0, ex2 -> 0 -> 1 - 2), NaN propagates.
__device__ __forceinline__ float2 tanh2(float2 x) {
  const float k = 2.8853900817779268f;  // 2 / ln 2
  const float2 y = ffma2(x, make_float2(k, k), make_float2(0.f, 0.f));
  const float2 e = make_float2(ex2_approx(y.x), ex2_approx(y.y));
  const float2 d = ffma2(e, make_float2(1.f, 1.f), make_float2(1.f, 1.f));
  const float2 r = make_float2(rcp_approx(d.x), rcp_approx(d.y));
  return ffma2(r, make_float2(-2.f, -2.f), make_float2(1.f, 1.f));
}

// Shared memory of one group (CTA): h1 rows padded to H+4 floats so that the
// per-lane LDS.128 / STS.128 of 8 consecutive lanes hit distinct bank quads.
template <int H, int L>
struct WsSmem {
  static constexpr int kStride = H + 4;
  float h1[32 * kStride];
  float4 part[L][32];          // layer-3 partial sums per role
  float2 v[2][32];             // clamped v_t, double-buffered by t parity
  float coup[2][32];           // coupling of step t
  Acc w[32];                   // softmin weights of the group
};

// SW = true stages the weights in shared memory (LDS.128 into registers);
// SW = false reads them from the kernel-parameter constant bank (LDCU into
// uniform registers).
template <int H, int L, int Mode, bool SW>
__global__ void __launch_bounds__(32 * L, 1) rollout_ws_kernel(const __grid_constant__ RolloutArgs<float> a,
                                                            const __grid_constant__ WeightHolder<float, H> wh) {
  static_assert(H % (4 * L) == 0, "each role owns a multiple of 4 hidden units");
  constexpr int U = H / L;            // hidden units per role
  constexpr int kNoiseRole = (L > 1) ? 1 : 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* s_plan = reinterpret_cast<float*>(smem_raw);             // 2T floats
  __shared__ __align__(16) WsSmem<H, L> sm;

  const int ctrl = blockIdx.y;
  if (a.abort_flag[static_cast<size_t>(ctrl) * a.abort_stride] != 0) return;
  const int role = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int chunk = a.chunk0 + blockIdx.x;
  const int k = chunk * 32 + lane;
  const bool valid = k < a.K;
  const int T = a.T;
  for (int i = threadIdx.x; i < 2 * T; i += 32 * L) s_plan[i] = a.plan[static_cast<size_t>(ctrl) * 2 * T + i];
  __shared__ __align__(16) MlpParams<float, SW ? H : 2> s_w;
  if constexpr (SW) {
    const float4* src = reinterpret_cast<const float4*>(&wh.get());
    float4* dst = reinterpret_cast<float4*>(&s_w);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(MlpParams<float, H>) / 16); i += 32 * L) dst[i] = src[i];
  }
  __syncthreads();

  const MlpParams<float, H>& w = [&]() -> const MlpParams<float, H>& {
    if constexpr (SW) return s_w;
    else return wh.get();
  }();
  const bool zm = k >= a.zero_start;
  const float dt = a.sys.dt;

  // noise role state
  NoiseStream<float, Mode> ns = make_noise<float, Mode>(a, ctrl, valid ? k : 0);
  const float inv_s0 = 1.0f / a.sigma0, inv_s1 = 1.0f / a.sigma1;
  const float gml = a.gamma - a.lambda, half_lambda = 0.5f * a.lambda;
  auto produce_v = [&](int t, int buf) {
    float e0 = 0.f, e1 = 0.f;
    if (valid) ns.eps(t, e0, e1);
    const float u0 = s_plan[2 * t], u1 = s_plan[2 * t + 1];
    if (zm) {
      e0 = e0 - u0;
      e1 = e1 - u1;
    }
    const float v0 = u0 + e0, v1 = u1 + e1;
    const float uv = __fmul_rn(__fmul_rn(u0, v0), inv_s0) + __fmul_rn(__fmul_rn(u1, v1), inv_s1);
    float coup;
    if (zm) {
      const float uu = __fmul_rn(__fmul_rn(u0, u0), inv_s0) + __fmul_rn(__fmul_rn(u1, u1), inv_s1);
      coup = __fadd_rn(__fmul_rn(gml, uv), __fmul_rn(half_lambda, uu));
    } else {
      coup = __fmul_rn(a.gamma, uv);
    }
    sm.v[buf][lane] = make_float2(clamp_r(v0, a.sys.lo0, a.sys.hi0), clamp_r(v1, a.sys.lo1, a.sys.hi1));
    sm.coup[buf][lane] = coup;
  };
  if (role == kNoiseRole) produce_v(0, 0);

  // state (every role keeps the dynamic block; role 0 also the pose and cost)
  const float* x0 = a.x0 + ctrl * 8;
  float px = x0[0], py = x0[1], th = x0[2];
  float roll = x0[3], vx = x0[4], vy = x0[5], thd = x0[6];
  MapDev<float> map;
  map.values = a.maps[ctrl];
  map.width = a.map_w;
  map.height = a.map_h;
  map.x0 = a.map_x0;
  map.y0 = a.map_y0;
  map.res = a.map_res;
  map.inv_res = a.map_inv_res;
  Acc cost = 0.0;
  MapTaps<float> q{};
  float p_roll = 0.f, p_vx = 0.f, p_vy = 0.f, p_coup = 0.f;
  __syncthreads();

  for (int t = 0; t < T; ++t) {
    const int buf = t & 1;
    // ---- A: inputs
    const float2 vv = sm.v[buf][lane];
    const float coup_t = sm.coup[buf][lane];
    const float in[6] = {roll, vx, vy, thd, vv.x, vv.y};
    // ---- B: layer 1 (own units), tanh, publish
    float2 h1o[U / 2];
#pragma unroll
    for (int p = 0; p < U / 2; ++p)
      h1o[p] = *reinterpret_cast<const float2*>(&w.b1[role * U + 2 * p]);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
#pragma unroll
      for (int p = 0; p < U / 2; ++p)
        h1o[p] = ffma2(*reinterpret_cast<const float2*>(&w.w1t[i][role * U + 2 * p]), make_float2(in[i], in[i]),
                       h1o[p]);
    }
#pragma unroll
    for (int p = 0; p < U / 2; ++p) h1o[p] = tanh2(h1o[p]);
    float h1[H];
    if constexpr (L == 1) {
#pragma unroll
      for (int p = 0; p < U / 2; ++p) {
        h1[2 * p] = h1o[p].x;
        h1[2 * p + 1] = h1o[p].y;
      }
    } else {
      float* my_h1 = &sm.h1[lane * WsSmem<H, L>::kStride + role * U];
#pragma unroll
      for (int p = 0; p < U / 2; p += 2)
        *reinterpret_cast<float4*>(my_h1 + 2 * p) = make_float4(h1o[p].x, h1o[p].y, h1o[p + 1].x, h1o[p + 1].y);
      __syncthreads();  // barrier 1
      // ---- D: layer 2 over all H inputs, tanh, layer-3 partials
      const float* row = &sm.h1[lane * WsSmem<H, L>::kStride];
#pragma unroll
      for (int i = 0; i < H; i += 4) {
        const float4 f = *reinterpret_cast<const float4*>(row + i);
        h1[i] = f.x;
        h1[i + 1] = f.y;
        h1[i + 2] = f.z;
        h1[i + 3] = f.w;
      }
    }
    float2 acc[U / 2];
#pragma unroll
    for (int p = 0; p < U / 2; ++p) acc[p] = *reinterpret_cast<const float2*>(&w.b2[role * U + 2 * p]);
    {
      // weight rows of own units as float4 (LDS.128 broadcast), double
      // buffered one input ahead so the loads overlap the FFMA2s
      constexpr int Q = U / 4;
      const float4* W2 = reinterpret_cast<const float4*>(&w.w2t[0][role * U]);
      float4 wb[2][Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) wb[0][q] = W2[q];
#pragma unroll
      for (int i = 0; i < H; ++i) {
        if (i + 1 < H) {
#pragma unroll
          for (int q = 0; q < Q; ++q) wb[(i + 1) & 1][q] = W2[(i + 1) * (H / 4) + q];
        }
        const float2 hh = make_float2(h1[i], h1[i]);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const float4 wv = wb[i & 1][q];
          acc[2 * q] = ffma2(make_float2(wv.x, wv.y), hh, acc[2 * q]);
          acc[2 * q + 1] = ffma2(make_float2(wv.z, wv.w), hh, acc[2 * q + 1]);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < U / 2; ++p) acc[p] = tanh2(acc[p]);
    // partial out_o = sum over own units j of W3[o][j] h2_j, two chains
    float2 pa01 = make_float2(0.f, 0.f), pa23 = make_float2(0.f, 0.f);
    float2 pb01 = make_float2(0.f, 0.f), pb23 = make_float2(0.f, 0.f);
#pragma unroll
    for (int p = 0; p < U / 2; ++p) {
      const int j0 = role * U + 2 * p, j1 = j0 + 1;
      pa01 = ffma2(*reinterpret_cast<const float2*>(&w.w3t[j0][0]), make_float2(acc[p].x, acc[p].x), pa01);
      pa23 = ffma2(*reinterpret_cast<const float2*>(&w.w3t[j0][2]), make_float2(acc[p].x, acc[p].x), pa23);
      pb01 = ffma2(*reinterpret_cast<const float2*>(&w.w3t[j1][0]), make_float2(acc[p].y, acc[p].y), pb01);
      pb23 = ffma2(*reinterpret_cast<const float2*>(&w.w3t[j1][2]), make_float2(acc[p].y, acc[p].y), pb23);
    }
    const float4 mine = make_float4(pa01.x + pb01.x, pa01.y + pb01.y, pa23.x + pb23.x, pa23.y + pb23.y);
    if constexpr (L > 1) sm.part[role][lane] = mine;
    // noise role: v_{t+1} and its coupling, published before barrier 2
    if (role == kNoiseRole && t + 1 < T) produce_v(t + 1, buf ^ 1);
    __syncthreads();  // barrier 2
    // ---- F: layer-3 reduction (fixed role order) and the dynamic Euler update
    float4 d = make_float4(w.b3[0], w.b3[1], w.b3[2], w.b3[3]);
#pragma unroll
    for (int r = 0; r < L; ++r) {
      const float4 pr = (L == 1) ? mine : sm.part[r][lane];
      d.x += pr.x;
      d.y += pr.y;
      d.z += pr.z;
      d.w += pr.w;
    }
    const float vx_old = vx, vy_old = vy, thd_old = thd;
    roll = add_rn(roll, mul_rn(d.x, dt));
    vx = add_rn(vx, mul_rn(d.y, dt));
    vy = add_rn(vy, mul_rn(d.z, dt));
    thd = add_rn(thd, mul_rn(d.w, dt));
    // ---- G (role 0): pose, costmap taps, running cost of step t-1
    if (role == 0) {
      float s, c;
      sincosf(th, &s, &c);
      px = add_rn(px, mul_rn(sub_rn(mul_rn(c, vx_old), mul_rn(s, vy_old)), dt));
      py = add_rn(py, mul_rn(add_rn(mul_rn(s, vx_old), mul_rn(c, vy_old)), dt));
      th = add_rn(th, mul_rn(thd_old, dt));
      if (t > 0) {
        const float h = map_interp(q);
        const float rc = state_cost_h(h, p_roll, p_vx, p_vy, a.sys.decay_pow[t - 1], a.sys.cost);
        cost += static_cast<Acc>(add_rn(rc, p_coup));
      }
      q = map_fetch(map, px, py);
      p_roll = roll;
      p_vx = vx;
      p_vy = vy;
      p_coup = coup_t;
      if (a.trace_states && k == a.trace_k) {
        float* so = a.trace_states + (t + 1) * 7;
        so[0] = px; so[1] = py; so[2] = th; so[3] = roll; so[4] = vx; so[5] = vy; so[6] = thd;
      }
    }
  }

  // ---- terminal cost (role 0) and the chunk softmin partials
  if (role == 0) {
    const float h = map_interp(q);
    cost += static_cast<Acc>(add_rn(state_cost_h(h, p_roll, p_vx, p_vy, a.sys.decay_pow[T - 1], a.sys.cost),
                                    p_coup));
    if (a.sys.with_terminal)
      cost += static_cast<Acc>(state_cost_h(h, p_roll, p_vx, p_vy, a.sys.decay_pow[T], a.sys.cost));
    if (valid) a.costs[static_cast<size_t>(ctrl) * a.K + k] = cost;
    const bool bad = valid && !isfinite(cost);
    const Acc rho = warp_min(valid ? cost : Acc(INFINITY));
    const Acc wk = valid ? exp(-(cost - rho) / a.dlambda) : 0.0;
    const Acc eta = warp_sum(wk);
    const unsigned any_bad = __ballot_sync(0xffffffffu, bad);
    sm.w[lane] = wk;
    if (lane == 0) {
      Acc* out = a.partials + static_cast<size_t>(ctrl) * a.partials_ctrl_stride +
                 static_cast<size_t>(chunk) * a.partial_stride;
      out[0] = rho;
      out[1] = eta;
      out[2] = any_bad ? 1.0 : 0.0;
      out[3] = 0.0;
    }
  }
  __syncthreads();
  // numerators: t-pairs distributed over the roles, eps regenerated
  {
    const Acc wk = sm.w[lane];
    Acc* out = a.partials + static_cast<size_t>(ctrl) * a.partials_ctrl_stride +
               static_cast<size_t>(chunk) * a.partial_stride + kPartialHeader;
    NoiseStream<float, Mode> ns2 = make_noise<float, Mode>(a, ctrl, valid ? k : 0);
    for (int tp = role; 2 * tp < T; tp += L) {
      for (int t = 2 * tp; t < 2 * tp + 2 && t < T; ++t) {
        float e0 = 0.f, e1 = 0.f;
        if (valid) {
          ns2.eps(t, e0, e1);
          if (zm) {
            e0 = e0 - s_plan[2 * t];
            e1 = e1 - s_plan[2 * t + 1];
          }
        }
        const Acc n0 = warp_sum(wk * static_cast<Acc>(e0));
        const Acc n1 = warp_sum(wk * static_cast<Acc>(e1));
        if (lane == 0) {
          out[2 * t] = n0;
          out[2 * t + 1] = n1;
        }
      }
    }
  }
}

}  // namespace mppi_dev
