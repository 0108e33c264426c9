// rollout_tc_pair.cuh — the tensor-core rollout (rollout_tc.cuh) with one
// 16-sample chunk per warp PAIR, for launches that fit one wave (H = 32).
//
// Why: a single-chunk warp's step is a chain of pipe-bound phases (layer-1
// HMMAs, 16 SFU ex2 per lane, layer-2 HMMAs, ...), each waiting on the last,
// with the per-sample scalar work (noise, coupling, cost, costmap taps,
// pose) issued in between by the same in-order warp.  At c0/c1 the grid has
// 1-2 such warps per scheduler, so that chain is the iteration time.  Here
// the two warps of a pair split the hidden units of layers 1-2 (n-tiles
// 2h, 2h+1 = units 16h .. 16h+15 for warp half h) and the scalar work:
//   * half 0, the STATE warp: pose + costmap taps, the state inputs, layer 3,
//     the Euler update, the running cost, the softmin partials;
//   * half 1, the CONTROL warp: noise, v = clamp(u + eps), the coupling,
//     eps' for the numerators, the control inputs.
// Each warp's layer-l activation is exactly the k-tile h of layer l+1's A
// operand; the two trade theirs through shared memory (three 64-thread
// named-barrier handoffs per step).  Every product, accumulation order and
// rounding is the single-warp kernel's, so the costs and partials are
// bit-identical to rollout_tc_kernel<32, MT = 1> (checked by the GPU tests).
// eps' stays on chip (the one-wave variant only); the numerators are summed
// per (t, c) element over the chunk's rows in that kernel's lane order.
#pragma once

#include "rollout_tc.cuh"

namespace mppi_dev {

struct TcPairStage {
  uint32_t in[2][64];        // layer-1 A operand, tc_in_word layout (TcStage)
  uint32_t xa[2][2][8][32];  // [layer 2 / 3][k-tile (= warp half)][ahi 0..3, alo 0..3][lane]
  float4 out[16];            // layer-3 outputs per sample row (state warp)
  double wk[16];             // softmin weight of each row (numerator pass)
};

__device__ __forceinline__ void tc_pair_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

// grid = (ceil(chunks / NP), controllers), block = 64 * NP (NP pairs).
// Dynamic smem: plan (2T + 2 floats), then eps' [NP][T][16] float2 and the
// coupling terms [NP][T][16] float (tc_pair_smem_bytes).
__host__ __device__ constexpr size_t tc_pair_smem_bytes(int T, int np) {
  return ((sizeof(float) * (2 * T + 2) + 15) & ~size_t(15)) + static_cast<size_t>(np) * T * 16 * (8 + 4);
}

template <int NP, int Mode, bool STAB>
__global__ void __launch_bounds__(64 * NP, NP == 1 ? 7 : 4) rollout_tc_pair_kernel(const __grid_constant__ RolloutArgs<float> a,
                                                                           const uint32_t* __restrict__ frag) {
  constexpr int H = 32;
  using L = TcLayout<H>;
  constexpr int SW = tc_sw_rcp<H>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int T = a.T;
  float* s_plan = reinterpret_cast<float*>(smem_raw);
  float2* s_eps_all = reinterpret_cast<float2*>(smem_raw + ((sizeof(float) * (2 * T + 2) + 15) & ~size_t(15)));
  float* s_coup_all = reinterpret_cast<float*>(s_eps_all + static_cast<size_t>(NP) * T * 16);
  __shared__ __align__(16) TcPairStage s_stage[NP];

  const int ctrl = blockIdx.y;
  if (a.abort_flag[static_cast<size_t>(ctrl) * a.abort_stride] != 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, half = warp & 1;
  const int g = lane >> 2, t4 = lane & 3;
  const int bar_id = 1 + pair;
  const int chunk = a.chunk0 + blockIdx.x * NP + pair;
  for (int i = threadIdx.x; i < 2 * T + 2; i += 64 * NP)
    s_plan[i] = (i < 2 * T) ? a.plan[static_cast<size_t>(ctrl) * 2 * T + i] : 0.f;

  // this warp's hidden half of layers 1-2; layer 3 whole (state warp)
  uint32_t w1[4], w2[2][2][4], w3[8];
  float b2[2][4], b3[4];
#pragma unroll
  for (int jj = 0; jj < 2; ++jj) {
    const int j = 2 * half + jj;
    w1[2 * jj] = frag[(L::W1 + 2 * j) * 32 + lane];
    w1[2 * jj + 1] = frag[(L::W1 + 2 * j + 1) * 32 + lane];
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
#pragma unroll
      for (int i = 0; i < 4; ++i) w2[kk][jj][i] = frag[(L::W2 + (kk * L::NJ + j) * 4 + i) * 32 + lane];
    b2[jj][0] = __uint_as_float(frag[(L::B2 + 2 * j) * 32 + lane]);
    b2[jj][1] = __uint_as_float(frag[(L::B2 + 2 * j + 1) * 32 + lane]);
    b2[jj][2] = tc_ld_opaque(frag + (L::B2 + 2 * j) * 32 + lane);
    b2[jj][3] = tc_ld_opaque(frag + (L::B2 + 2 * j + 1) * 32 + lane);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) w3[i] = frag[(L::W3 + i) * 32 + lane];
  b3[0] = __uint_as_float(frag[L::B3 * 32 + lane]);
  b3[1] = __uint_as_float(frag[(L::B3 + 1) * 32 + lane]);
  b3[2] = tc_ld_opaque(frag + L::B3 * 32 + lane);
  b3[3] = tc_ld_opaque(frag + (L::B3 + 1) * 32 + lane);

  TcPairStage& st = s_stage[pair];
  if (half == 1 && lane < 16) {  // the constant-one input column (k = 6: bias of layer 1)
    const int w = tc_in_word(lane & 7, 3, lane >> 3);
    st.in[0][w] = h2_bits(__floats2half2_rn(1.f, 0.f));
    st.in[1][w] = 0u;
  }

  // ---- owner lanes (lanes t >= 2 mirror t - 2, as rollout_tc_kernel MT = 1)
  const int row_own = g + 8 * (t4 & 1);
  const int hrow = t4 & 1;
  const bool dup = t4 >= 2;
  const int k = chunk * 16 + row_own;
  const bool active = chunk < a.chunk_end;
  const bool valid = (k < a.K) && !dup && active;
  const bool zm = k >= a.zero_start;
  const int kn = (k < a.K) ? k : 0;
  const float dt = a.sys.dt;
  const float dt3 = dt * __uint_as_float(frag[L::SC * 32 + lane]);  // dt 2^-s (exact): layer 3 is 2^s-scaled
  const CostDev<float> cp = a.sys.cost;
  const float inv_s0 = 1.0f / a.sigma0, inv_s1 = 1.0f / a.sigma1;
  const float gml = a.gamma - a.lambda, half_lambda = 0.5f * a.lambda;
  float2* s_eps = s_eps_all + static_cast<size_t>(pair) * T * 16;
  float* s_coup = s_coup_all + static_cast<size_t>(pair) * T * 16;
  __syncthreads();  // s_plan, stage constants
  cudaTriggerProgrammaticLaunchCompletion();  // one wave: the tail may launch and wait

  // ---- control warp: noise, v_t = g(u_t + eps_t), coupling (controller.cpp:86-101)
  NoiseStream<float, Mode> ns = make_noise<float, Mode>(a, ctrl, kn);
  const uint64_t seed = a.seeds[ctrl], iteration = a.iters[ctrl];
  float zc0 = 0.f, zc1 = 0.f;
  float v0c = 0.f, v1c = 0.f;
  auto produce_v = [&](int t, bool even) {
    float e0, e1;
    if constexpr (Mode == kPhilox) {
      if (even) {
        const uint4 d = philox_draw(seed, iteration, static_cast<uint32_t>(kn), static_cast<uint32_t>(t) >> 1);
        float z0, z1;
        philox_box_muller(d.x, d.y, z0, z1);
        philox_box_muller(d.z, d.w, zc0, zc1);
        e0 = a.scale0 * z0;
        e1 = a.scale1 * z1;
      } else {
        e0 = a.scale0 * zc0;
        e1 = a.scale1 * zc1;
      }
    } else {
      ns.eps(t, e0, e1);
    }
    const float u0 = s_plan[2 * t], u1 = s_plan[2 * t + 1];
    e0 = zm ? e0 - u0 : e0;
    e1 = zm ? e1 - u1 : e1;
    if (!dup) s_eps[t * 16 + row_own] = make_float2(e0, e1);  // owners only (predicated)
    const float v0 = u0 + e0, v1 = u1 + e1;
    const float uv = __fmul_rn(__fmul_rn(u0, v0), inv_s0) + __fmul_rn(__fmul_rn(u1, v1), inv_s1);
    const float uu = __fmul_rn(__fmul_rn(u0, u0), inv_s0) + __fmul_rn(__fmul_rn(u1, u1), inv_s1);
    const float coup = zm ? __fadd_rn(__fmul_rn(gml, uv), __fmul_rn(half_lambda, uu)) : __fmul_rn(a.gamma, uv);
    if (!dup) s_coup[t * 16 + row_own] = coup;
    v0c = clamp_r(v0, a.sys.lo0, a.sys.hi0);
    v1c = clamp_r(v1, a.sys.lo1, a.sys.hi1);
  };
  auto stage_v = [&] {
    uint32_t hi, lo;
    split2(v0c, v1c, hi, lo);
    if (!dup) {
      st.in[0][tc_in_word(g, 2, hrow)] = hi;
      st.in[1][tc_in_word(g, 2, hrow)] = lo;
    }
  };

  // ---- state warp: the 7-state, costmap taps, cost
  cudaGridDependencySynchronize();  // x0 (a no-op unless launched after the x0 fetch)
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
  float p_roll = 0.f, p_vx = 0.f, p_vy = 0.f;

  if (half == 1) {
    produce_v(0, true);
    stage_v();
  }

  auto step = [&](int t, auto even_tag) {
    constexpr bool EVEN = decltype(even_tag)::value;
    MapTaps<float> q_next{};
    if (half == 0) {
      // pose of x_{t+1} (Euler split from the old state, dynamics.cpp:137-148)
      // and its costmap taps, a step ahead of their use
      float sn, cs;
      tc_sincos(th, sn, cs);
      px = add_rn(px, mul_rn(sub_rn(mul_rn(cs, vx), mul_rn(sn, vy)), dt));
      py = add_rn(py, mul_rn(add_rn(mul_rn(sn, vx), mul_rn(cs, vy)), dt));
      th = add_rn(th, mul_rn(thd, dt));
      q_next = map_fetch(map, px, py);
      uint32_t hi0, lo0, hi1, lo1;
      split2(roll, vx, hi0, lo0);
      split2(vy, thd, hi1, lo1);
      if (!dup) {  // owners only (predicated): no two lanes write one word
        st.in[0][tc_in_word(g, 0, hrow)] = hi0;
        st.in[1][tc_in_word(g, 0, hrow)] = lo0;
        st.in[0][tc_in_word(g, 1, hrow)] = hi1;
        st.in[1][tc_in_word(g, 1, hrow)] = lo1;
      }
    }
    tc_pair_bar(bar_id);  // (1) inputs of step t staged
    // ---- layer 1, this warp's two n-tiles (as tc_mlp)
    uint32_t ahi[4], alo[4];
    {
      const int w = tc_in_word(g, t4, 0);
      const uint2 ah = *reinterpret_cast<const uint2*>(&st.in[0][w]);
      const uint2 al = *reinterpret_cast<const uint2*>(&st.in[1][w]);
      float d1[2][4];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        Acc2 acc;
#pragma unroll
        for (int i = 0; i < 4; ++i) acc.m[i] = acc.c[i] = 0.f;
        mma_k8(acc.c, al.x, al.y, w1[2 * jj]);
        mma_k8(acc.c, ah.x, ah.y, w1[2 * jj + 1]);
        mma_k8(acc.m, ah.x, ah.y, w1[2 * jj]);
        acc2_sum(acc, d1[jj]);
      }
      acc_to_a<SW>(d1[0], d1[1], ahi, alo);  // k-tile `half` of layer 2
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        st.xa[0][half][i][lane] = ahi[i];
        st.xa[0][half][4 + i][lane] = alo[i];
      }
    }
    // ---- side work while the partner finishes its half
    if (half == 0) {
      // running cost of step t-1 on x_t (taps fetched last step)
      const float h = map_interp(q);
      const float rc = tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[t > 0 ? t - 1 : 0], cp);
      if (t > 0) cost += static_cast<Acc>(add_rn(rc, s_coup[(t - 1) * 16 + row_own]));
    } else {
      if (t + 1 < T) produce_v(t + 1, !EVEN);
    }
    tc_pair_bar(bar_id);  // (2) layer-2 A operand complete
    // ---- layer 2, this warp's two n-tiles, k-tiles 0 then 1 (as tc_mlp)
    {
      uint32_t k0h[4], k0l[4], k1h[4], k1l[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t ph = st.xa[0][half ^ 1][i][lane], pl = st.xa[0][half ^ 1][4 + i][lane];
        k0h[i] = half ? ph : ahi[i];
        k0l[i] = half ? pl : alo[i];
        k1h[i] = half ? ahi[i] : ph;
        k1l[i] = half ? alo[i] : pl;
      }
      Acc2 a2[2];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int i = 0; i < 4; ++i) a2[jj].c[i] = 0.f;
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const uint32_t* b = w2[0][jj];
        mma_k16(a2[jj].c, k0l, b[0], b[2]);
        mma_k16(a2[jj].c, k0h, b[1], b[3]);
        mma_k16_c(a2[jj].m, k0h, b[0], b[2], b2[jj]);
      }
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const uint32_t* b = w2[1][jj];
        mma_k16(a2[jj].c, k1l, b[0], b[2]);
        mma_k16(a2[jj].c, k1h, b[1], b[3]);
        mma_k16(a2[jj].m, k1h, b[0], b[2]);
      }
      float d2[2][4];
      acc2_sum(a2[0], d2[0]);
      acc2_sum(a2[1], d2[1]);
      acc_to_a<SW>(d2[0], d2[1], ahi, alo);  // k-tile `half` of layer 3
    }
    if (half == 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        st.xa[1][1][i][lane] = ahi[i];
        st.xa[1][1][4 + i][lane] = alo[i];
      }
      if (t + 1 < T) stage_v();  // both warps have read this step's inputs (barrier 2)
    }
    tc_pair_bar(bar_id);  // (3) layer-3 k-tile 1 complete
    if (half == 0) {
      // ---- layer 3 (k-tile 0 own, k-tile 1 from the control warp; as tc_mlp)
      Acc2 a3;
      float c3[2][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) c3[0][i] = c3[1][i] = 0.f;
      uint32_t phi[4], plo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        phi[i] = st.xa[1][1][i][lane];
        plo[i] = st.xa[1][1][4 + i][lane];
      }
      mma_k16(c3[0], alo, w3[0], w3[2]);
      mma_k16(c3[0], ahi, w3[1], w3[3]);
      mma_k16_c(a3.m, ahi, w3[0], w3[2], b3);
      mma_k16(c3[1], plo, w3[4], w3[6]);
      mma_k16(c3[1], phi, w3[5], w3[7]);
      mma_k16(a3.m, phi, w3[4], w3[6]);
      tc_sum_cross<2>(c3, a3.c);
      float d3[4];
      acc2_sum(a3, d3);
      if (t4 < 2) {
        reinterpret_cast<float2*>(&st.out[g])[t4] = make_float2(d3[0], d3[1]);
        reinterpret_cast<float2*>(&st.out[g + 8])[t4] = make_float2(d3[2], d3[3]);
      }
      __syncwarp();
      const float4 d = st.out[row_own];
      roll = add_rn(roll, mul_rn(d.x, dt3));
      vx = add_rn(vx, mul_rn(d.y, dt3));
      vy = add_rn(vy, mul_rn(d.z, dt3));
      thd = add_rn(thd, mul_rn(d.w, dt3));
      q = q_next;
      p_roll = roll;
      p_vx = vx;
      p_vy = vy;
    }
  };
  int t = 0;
  for (; t + 1 < T; t += 2) {
    step(t, std::true_type{});
    step(t + 1, std::false_type{});
  }
  if (t < T) step(t, std::true_type{});

  // ---- terminal cost and the chunk softmin partials (state warp)
  Acc* out = a.partials + static_cast<size_t>(ctrl) * a.partials_ctrl_stride +
             static_cast<size_t>(chunk) * a.partial_stride;
  MPPI_DCHECK(!active || static_cast<long long>(chunk + 1) * a.partial_stride <= a.partials_ctrl_stride);
  MPPI_DCHECK(!valid || k < a.K);
  if (half == 0) {
    const float h = map_interp(q);
    cost += static_cast<Acc>(
        add_rn(tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[T - 1], cp), s_coup[(T - 1) * 16 + row_own]));
    if (a.sys.with_terminal) cost += static_cast<Acc>(tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[T], cp));
    if (valid) a.costs[static_cast<size_t>(ctrl) * a.K + k] = cost;
    const bool bad = valid && !isfinite(cost);
    const Acc rho = warp_min(valid ? cost : Acc(INFINITY));
    const Acc wk = valid ? exp(-(cost - rho) / a.dlambda) : 0.0;
    const Acc eta = warp_sum(wk);
    const unsigned any_bad = __ballot_sync(0xffffffffu, bad);
    if (lane == 0) MPPI_STAMP_MAX(0);  // K1: last state warp through the rollout
    if (lane == 0 && active) {
      out[0] = rho;
      out[1] = eta;
      out[2] = any_bad ? 1.0 : 0.0;
      out[3] = 0.0;
    }
    if (!dup) st.wk[row_own] = wk;
  }
  tc_pair_bar(bar_id);
  // numerators: element e = 2t + c, in the single-warp kernel's order (rows
  // 0..7 and rows 8..15 as two sequential sums of rounded products, then
  // their sum plus the mirror lanes' zeros), so the chunk rows are
  // bit-identical whichever K1 variant a rank's grid size selects
  for (int e = 32 * half + lane; e < 2 * T; e += 64) {
    const int tt = e >> 1, c = e & 1;
    Acc sa = 0.0, sb = 0.0;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float2 ea = s_eps[tt * 16 + r], eb = s_eps[tt * 16 + r + 8];
      sa = __dadd_rn(sa, __dmul_rn(st.wk[r], static_cast<Acc>(c ? ea.y : ea.x)));
      sb = __dadd_rn(sb, __dmul_rn(st.wk[r + 8], static_cast<Acc>(c ? eb.y : eb.x)));
    }
    if (active) out[kPartialHeader + e] = __dadd_rn(__dadd_rn(sa, sb), 0.0);
  }
}

}  // namespace mppi_dev
