// rollout_tc_split.cuh — the tensor-core rollout (rollout_tc.cuh) with one
// 16-sample chunk per warp PAIR split by SAMPLES: warp half h runs chunk rows
// 8h .. 8h+7, for launches that fit one wave (H = 32).
//
// Why: at c0/c1 a single-chunk warp's step is a chain of pipe-bound phases
// (layer-1 HMMAs, 16 ex2 + 16 reciprocals per lane, layer-2 HMMAs, ...), and
// with 1-2 such warps per scheduler that chain is the iteration time
// (profiles/README.md).  The warp pair of rollout_tc_pair.cuh halves the
// chain by splitting the hidden units, but trades activations through shared
// memory behind three barriers per step.  Here each warp owns 8 samples
// outright and needs no partner until the softmin partials:
//   * layers 1-2 put the samples on the mma N dimension (n8) and the weights
//     on M (A operand = the single-warp kernel's B fragment words of n-tiles
//     2i, 2i+1 of the same lane, no data movement): 8 activations per lane
//     per layer instead of 16;
//   * the activations go from accumulator layout (hidden g, samples 2t, 2t+1)
//     to the next B operand (hidden 2t, 2t+1, sample g) with one
//     movmatrix.trans per 8x8 fp16 block (hi and lo words);
//   * layer 3 is the single-warp kernel's (samples on M, outputs on N), its
//     A operand rows g+8 zero;
//   * the four lanes of a quad run sample g's scalar path (noise, pose,
//     costmap, cost) — lane t feeds input pair t of layer 1 directly from
//     registers (selp), and the outputs reach the quad by four shuffles: no
//     shared-memory stage, no barrier and no branch in the step loop;
//   * optionally (PF, sparse sampling) an L2 prefetch of the costmap two
//     steps ahead (map_prefetch_l2).
// Used while its warps fit one per scheduler (tc_launch.cuh split_fits).
// Every product, accumulation order and rounding is the single-warp kernel's
// (a dot product's tensor-core sum does not depend on which operand holds
// which factor; the reciprocal rule of tc_sw_rcp<32> — SFU for chunk rows
// 0..7, FMA pipe for rows 8..15 — becomes per warp), so costs and partials
// are bit-identical to rollout_tc_kernel<32, MT = 1> (GPU tests).
#pragma once

#include "rollout_tc.cuh"

namespace mppi_dev {

__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// p ? a : b as one selp (never a branch)
__device__ __forceinline__ float fsel_if(int p, float a, float b) {
  float r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\tselp.f32 %0, %1, %2, q;\n\t}" : "=f"(r) : "f"(a), "f"(b), "r"(p));
  return r;
}

// L2 prefetch of the costmap rows under the position extrapolated one more
// step, (2 p_{t+1} - p_t): the taps of x_{t+2} are read a step later, and with
// the L2 cold (every newly visited line an HBM miss) that latency is about a
// step.  Only cache state changes; the taps are still read by map_fetch.
__device__ __forceinline__ void map_prefetch_l2(const MapDev<float>& m, float px, float py) {
  float gx = mul_rn(sub_rn(px, m.x0), m.inv_res);
  float gy = mul_rn(sub_rn(py, m.y0), m.inv_res);
  gx = fminf(fmaxf(gx, 0.f), static_cast<float>(m.width - 2));
  gy = fminf(fmaxf(gy, 0.f), static_cast<float>(m.height - 2));
  const float* p = m.values + static_cast<size_t>(static_cast<int>(gy)) * m.width + static_cast<int>(gx);
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p + m.width));
}

// accumulator tile (rows g, g+8 = hidden units; columns 2t, 2t+1 = samples)
// -> activation -> fp16 hi/lo words transposed to (hidden 2t, 2t+1; sample g):
// h0/l0 from rows g (the k-slice's first 8 units), h1/l1 from rows g+8
template <bool SWR>
__device__ __forceinline__ void split_act_t(const float (&d)[4], uint32_t& h0, uint32_t& l0, uint32_t& h1,
                                            uint32_t& l1) {
  const float2 r0 = act_r2<SWR>(d[0], d[1]), r1 = act_r2<SWR>(d[2], d[3]);
  split2(r0.x, r0.y, h0, l0);
  split2(r1.x, r1.y, h1, l1);
  h0 = movm_t(h0);
  l0 = movm_t(l0);
  h1 = movm_t(h1);
  l1 = movm_t(l1);
}

// dynamic smem: plan (2T + 2 floats), then eps' [NP][T][16] float2
__host__ __device__ constexpr size_t tc_split_smem_bytes(int T, int np) {
  return ((sizeof(float) * (2 * T + 2) + 15) & ~size_t(15)) + static_cast<size_t>(np) * T * 16 * 8;
}

struct TcSplitShared {
  double wk[16];
  double rho[2];
  unsigned bad[2];
};

// The rollout of one warp half (HALF: chunk rows 8 HALF .. 8 HALF + 7).
template <int NP, int Mode, bool STAB, bool PF, int HALF>
__device__ __forceinline__ void tc_split_half(const RolloutArgs<float>& a, const uint32_t* __restrict__ frag,
                                              float* s_plan, float2* s_eps, TcSplitShared& sh, int chunk,
                                              int bar_id) {
  constexpr int H = 32;
  using L = TcLayout<H>;
  constexpr bool SWR = HALF == 1;  // tc_sw_rcp<32>() = 0b1010: rows g + 8 take the FMA-pipe reciprocal
  static_assert(tc_sw_rcp<32>() == 10, "the split kernel assumes the row-g SFU / row-g+8 FMA reciprocal rule");
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int ctrl = blockIdx.y;
  const int T = a.T;

  // ---- weights: layers 1-2 as A fragments (rows = hidden units), layer 3 as B
  uint32_t w1h[2][2], w1l[2][2];   // [m-tile][a0, a1]
  uint32_t w2h[2][2][4], w2l[2][2][4];  // [m-tile][k-tile][a0..a3]
  uint32_t w3[8];
  float b2[2][4], b3[4];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int j = 2 * mi + r;
      w1h[mi][r] = frag[(L::W1 + 2 * j) * 32 + lane];
      w1l[mi][r] = frag[(L::W1 + 2 * j + 1) * 32 + lane];
    }
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {  // a0/a2 from n-tile 2mi, a1/a3 from 2mi + 1
        const int base = L::W2 + (kk * L::NJ + 2 * mi + r) * 4;
        w2h[mi][kk][r] = frag[(base + 0) * 32 + lane];
        w2l[mi][kk][r] = frag[(base + 1) * 32 + lane];
        w2h[mi][kk][2 + r] = frag[(base + 2) * 32 + lane];
        w2l[mi][kk][2 + r] = frag[(base + 3) * 32 + lane];
      }
    }
    // bias of hidden 16 mi + g (+ 8): column 8 j + 2 t' + c of the B2 words
    // with j = 2 mi (+1), t' = g >> 1, c = g & 1 — held by lane t' of any group
    const int src = g >> 1;
    float bv[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float c0 = __shfl_sync(0xffffffffu, __uint_as_float(frag[(L::B2 + 2 * (2 * mi + r)) * 32 + lane]), src);
      const float c1 = __shfl_sync(0xffffffffu, __uint_as_float(frag[(L::B2 + 2 * (2 * mi + r) + 1) * 32 + lane]), src);
      bv[r] = (g & 1) ? c1 : c0;
    }
    b2[mi][0] = b2[mi][1] = bv[0];
    b2[mi][2] = b2[mi][3] = bv[1];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) w3[i] = frag[(L::W3 + i) * 32 + lane];
  b3[0] = __uint_as_float(frag[L::B3 * 32 + lane]);
  b3[1] = __uint_as_float(frag[(L::B3 + 1) * 32 + lane]);
  b3[2] = tc_ld_opaque(frag + L::B3 * 32 + lane);
  b3[3] = tc_ld_opaque(frag + (L::B3 + 1) * 32 + lane);

  // ---- the quad's sample
  const int row = 8 * HALF + g;
  const bool own = t4 == 0;
  const int k = chunk * 16 + row;
  const bool active = chunk < a.chunk_end;
  const bool valid = (k < a.K) && own && active;
  const bool zm = k >= a.zero_start;
  const int kn = (k < a.K) ? k : 0;
  const float dt = a.sys.dt;
  const float dt3 = dt * __uint_as_float(frag[L::SC * 32 + lane]);
  const CostDev<float> cp = a.sys.cost;
  const float inv_s0 = 1.0f / a.sigma0, inv_s1 = 1.0f / a.sigma1;
  const float gml = a.gamma - a.lambda, half_lambda = 0.5f * a.lambda;

  NoiseStream<float, Mode> ns = make_noise<float, Mode>(a, ctrl, kn);
  const uint64_t seed = a.seeds[ctrl], iteration = a.iters[ctrl];
  float zc0 = 0.f, zc1 = 0.f;
  float v0c, v1c, coup_t;
  const uint32_t s_eps_base = static_cast<uint32_t>(__cvta_generic_to_shared(s_eps + row));
  // v_t = g(u_t + eps_t) and the coupling of step t (controller.cpp:86-101).
  // (At one warp per scheduler the noise draws here cost less than a
  // prologue computing the whole batch up front: c0 72.2 vs 73.3 us;
  // profiles/r02d.)
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
      ns.eps(min(t, T - 1), e0, e1);
    }
    const float u0 = s_plan[2 * t], u1 = s_plan[2 * t + 1];
    e0 = zm ? e0 - u0 : e0;
    e1 = zm ? e1 - u1 : e1;
    // owner-only store as a predicated st.shared (a C++ `if` on the lane
    // index compiles to a divergent branch + reconvergence in every step)
    {
      const uint32_t addr = s_eps_base + 8u * static_cast<uint32_t>(t * 16);
      asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.shared.v2.f32 [%0], {%1, %2};\n\t}" ::"r"(addr),
                   "f"(e0), "f"(e1), "r"(static_cast<int>(t < T && own))
                   : "memory");
    }
    const float v0 = u0 + e0, v1 = u1 + e1;
    const float uv = __fmul_rn(__fmul_rn(u0, v0), inv_s0) + __fmul_rn(__fmul_rn(u1, v1), inv_s1);
    const float uu = __fmul_rn(__fmul_rn(u0, u0), inv_s0) + __fmul_rn(__fmul_rn(u1, u1), inv_s1);
    coup_t = zm ? __fadd_rn(__fmul_rn(gml, uv), __fmul_rn(half_lambda, uu)) : __fmul_rn(a.gamma, uv);
    v0c = clamp_r(v0, a.sys.lo0, a.sys.hi0);
    v1c = clamp_r(v1, a.sys.lo1, a.sys.hi1);
  };

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
  float p_roll = 0.f, p_vx = 0.f, p_vy = 0.f, p_coup = 0.f;
  const int quad0 = lane & ~3;
  const int sel_0 = t4 == 0, sel_2 = t4 == 2, sel_lo = t4 < 2;
  produce_v(0, true);

  auto step = [&](int t, auto even_tag) {
    constexpr bool EVEN = decltype(even_tag)::value;
    // pose of x_{t+1} and its costmap taps, a step ahead (as rollout_tc_kernel)
    float sn, cs;
    tc_sincos(th, sn, cs);
    const float px_old = px, py_old = py;
    px = add_rn(px, mul_rn(sub_rn(mul_rn(cs, vx), mul_rn(sn, vy)), dt));
    py = add_rn(py, mul_rn(add_rn(mul_rn(sn, vx), mul_rn(cs, vy)), dt));
    th = add_rn(th, mul_rn(thd, dt));
    const MapTaps<float> q_next = map_fetch(map, px, py);
    if constexpr (PF) map_prefetch_l2(map, 2.f * px - px_old, 2.f * py - py_old);
    // ---- layer 1: B operand = input pair t4 of sample g: (roll, vx), (vy, thd), (v0, v1), (1, 0)
    uint32_t xh, xl;
    {
      // (selp: the ternaries on the lane index compiled to divergent branches)
      const float bx = fsel_if(sel_lo, fsel_if(sel_0, roll, vy), fsel_if(sel_2, v0c, 1.f));
      const float by = fsel_if(sel_lo, fsel_if(sel_0, vx, thd), fsel_if(sel_2, v1c, 0.f));
      split2(bx, by, xh, xl);
    }
    uint32_t x2h[2][2], x2l[2][2];  // layer-2 B operand [k-tile][b0, b1]
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      Acc2 acc;
#pragma unroll
      for (int i = 0; i < 4; ++i) acc.m[i] = acc.c[i] = 0.f;
      mma_k8(acc.c, w1h[mi][0], w1h[mi][1], xl);  // W hi * x lo
      mma_k8(acc.c, w1l[mi][0], w1l[mi][1], xh);  // W lo * x hi
      mma_k8(acc.m, w1h[mi][0], w1h[mi][1], xh);  // W hi * x hi
      float d1[4];
      acc2_sum(acc, d1);
      split_act_t<SWR>(d1, x2h[mi][0], x2l[mi][0], x2h[mi][1], x2l[mi][1]);
    }
    // running cost of step t-1 on x_t (taps fetched last step)
    {
      const float h = map_interp(q);
      const float rc = tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[t > 0 ? t - 1 : 0], cp);
      cost += (t > 0) ? static_cast<Acc>(add_rn(rc, p_coup)) : 0.0;
      p_coup = coup_t;
    }
    // ---- layer 2: per m-tile (hidden 16 mi ..), k-tiles 0 then 1
    Acc2 a2[2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int i = 0; i < 4; ++i) a2[mi].c[i] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const uint32_t bl[2] = {x2l[kk][0], x2l[kk][1]}, bh[2] = {x2h[kk][0], x2h[kk][1]};
        mma_k16(a2[mi].c, w2h[mi][kk], bl[0], bl[1]);  // W hi * act lo
        mma_k16(a2[mi].c, w2l[mi][kk], bh[0], bh[1]);  // W lo * act hi
        if (kk == 0)
          mma_k16_c(a2[mi].m, w2h[mi][kk], bh[0], bh[1], b2[mi]);
        else
          mma_k16(a2[mi].m, w2h[mi][kk], bh[0], bh[1]);
      }
    }
    uint32_t a3h[2][4], a3l[2][4];  // layer-3 A operand [k-tile][a0..a3], rows g + 8 zero
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      float d2[4];
      acc2_sum(a2[mi], d2);
      split_act_t<SWR>(d2, a3h[mi][0], a3l[mi][0], a3h[mi][2], a3l[mi][2]);
      a3h[mi][1] = a3h[mi][3] = a3l[mi][1] = a3l[mi][3] = 0u;
    }
    produce_v(t + 1, !EVEN);
    // ---- layer 3 (as tc_mlp: per-k-tile cross accumulators)
    Acc2 a3;
    float c3[2][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) c3[0][i] = c3[1][i] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int b = kk * 4;
      mma_k16(c3[kk], a3l[kk], w3[b], w3[b + 2]);
      mma_k16(c3[kk], a3h[kk], w3[b + 1], w3[b + 3]);
      if (kk == 0)
        mma_k16_c(a3.m, a3h[kk], w3[b], w3[b + 2], b3);
      else
        mma_k16(a3.m, a3h[kk], w3[b], w3[b + 2]);
    }
    tc_sum_cross<2>(c3, a3.c);
    float d3[4];
    acc2_sum(a3, d3);
    // outputs 0, 1 in lane t = 0 and 2, 3 in lane t = 1 of the quad
    const float dr = __shfl_sync(0xffffffffu, d3[0], quad0);
    const float dvx = __shfl_sync(0xffffffffu, d3[1], quad0);
    const float dvy = __shfl_sync(0xffffffffu, d3[0], quad0 + 1);
    const float dw = __shfl_sync(0xffffffffu, d3[1], quad0 + 1);
    roll = add_rn(roll, mul_rn(dr, dt3));
    vx = add_rn(vx, mul_rn(dvx, dt3));
    vy = add_rn(vy, mul_rn(dvy, dt3));
    thd = add_rn(thd, mul_rn(dw, dt3));
    q = q_next;
    p_roll = roll;
    p_vx = vx;
    p_vy = vy;
  };
  int t = 0;
  for (; t + 1 < T; t += 2) {
    step(t, std::true_type{});
    step(t + 1, std::false_type{});
  }
  if (t < T) step(t, std::true_type{});

  // ---- terminal cost; the chunk's softmin partials in the single-warp order
  {
    const float h = map_interp(q);
    cost += static_cast<Acc>(add_rn(tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[T - 1], cp), p_coup));
    if (a.sys.with_terminal) cost += static_cast<Acc>(tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[T], cp));
  }
  MPPI_DCHECK(!valid || (k >= 0 && k < a.K));
  if (valid) a.costs[static_cast<size_t>(ctrl) * a.K + k] = cost;
  const unsigned bad = __ballot_sync(0xffffffffu, valid && !isfinite(cost));
  const Acc rho_h = warp_min(valid ? cost : Acc(INFINITY));
  if (lane == 0) {
    sh.rho[HALF] = rho_h;
    sh.bad[HALF] = bad;
  }
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(64) : "memory");
  const Acc rho = sh.rho[0] < sh.rho[1] ? sh.rho[0] : sh.rho[1];
  const Acc wk = valid ? exp(-(cost - rho) / a.dlambda) : 0.0;
  if (own) sh.wk[row] = wk;
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(64) : "memory");
  Acc* out = a.partials + static_cast<size_t>(ctrl) * a.partials_ctrl_stride +
             static_cast<size_t>(chunk) * a.partial_stride;
  MPPI_DCHECK(!active || static_cast<long long>(chunk + 1) * a.partial_stride <= a.partials_ctrl_stride);
  if constexpr (HALF == 0) {
    // eta with the single-warp kernel's lane layout and butterfly order
    // (lane (g, t): row g for t = 0, row g + 8 for t = 1, zero for t >= 2)
    const Acc eta = warp_sum(t4 == 0 ? sh.wk[g] : t4 == 1 ? sh.wk[g + 8] : 0.0);
    if (lane == 0) MPPI_STAMP_MAX(0);
    if (lane == 0 && active) {
      out[0] = rho;
      out[1] = eta;
      out[2] = (sh.bad[0] | sh.bad[1]) ? 1.0 : 0.0;
      out[3] = 0.0;
    }
  }
  for (int e = 32 * HALF + lane; e < 2 * T; e += 64) {
    const int tt = e >> 1, c = e & 1;
    Acc sa = 0.0, sb = 0.0;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float2 ea = s_eps[tt * 16 + r], eb = s_eps[tt * 16 + r + 8];
      sa = __dadd_rn(sa, __dmul_rn(sh.wk[r], static_cast<Acc>(c ? ea.y : ea.x)));
      sb = __dadd_rn(sb, __dmul_rn(sh.wk[r + 8], static_cast<Acc>(c ? eb.y : eb.x)));
    }
    if (active) out[kPartialHeader + e] = __dadd_rn(__dadd_rn(sa, sb), 0.0);
  }
}

// Resident CTAs per SM the register budget is sized for: 1 (no cap, ~200
// registers, no spills; the kernel runs at <= 2 CTAs per SM); a 7-CTA cap
// (c1's one wave) spills in the step loop
#ifndef MPPI_SPLIT_MINB
#define MPPI_SPLIT_MINB 1
#endif
// grid = (ceil(chunks / NP), controllers), block = 64 * NP (NP warp pairs)
// PF: the two-steps-ahead L2 costmap prefetch (map_prefetch_l2)
template <int NP, int Mode, bool STAB, bool PF>
__global__ void __launch_bounds__(64 * NP, MPPI_SPLIT_MINB) rollout_tc_split_kernel(const __grid_constant__ RolloutArgs<float> a,
                                                                           const uint32_t* __restrict__ frag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int T = a.T;
  float* s_plan = reinterpret_cast<float*>(smem_raw);
  float2* s_eps_all = reinterpret_cast<float2*>(smem_raw + ((sizeof(float) * (2 * T + 2) + 15) & ~size_t(15)));
  __shared__ TcSplitShared s_sh[NP];
  const int ctrl = blockIdx.y;
  if (a.abort_flag[static_cast<size_t>(ctrl) * a.abort_stride] != 0) return;
  const int warp = threadIdx.x >> 5;
  const int pair = warp >> 1, half = warp & 1;
  const int chunk = a.chunk0 + blockIdx.x * NP + pair;
  for (int i = threadIdx.x; i < 2 * T + 2; i += 64 * NP)
    s_plan[i] = (i < 2 * T) ? a.plan[static_cast<size_t>(ctrl) * 2 * T + i] : 0.f;
  __syncthreads();
  cudaTriggerProgrammaticLaunchCompletion();  // one wave: the dependent may launch and wait
  float2* s_eps = s_eps_all + static_cast<size_t>(pair) * T * 16;
  if (half == 0)
    tc_split_half<NP, Mode, STAB, PF, 0>(a, frag, s_plan, s_eps, s_sh[pair], chunk, 1 + pair);
  else
    tc_split_half<NP, Mode, STAB, PF, 1>(a, frag, s_plan, s_eps, s_sh[pair], chunk, 1 + pair);
}

}  // namespace mppi_dev
