// rollout_tc.cuh — K1 tensor-core variant: the dynamics MLP of a tile of
// samples on the tensor cores (warp-level mma.sync, fp16x3 split, fp32
// accumulate), everything else per sample in fp32 on the CUDA cores.
//
// Why: the FFMA2 kernel (rollout_ws.cuh) issues ~1 770 warp-instructions per
// 32-sample step, 768 of them FFMA2 and ~380 weight loads; at the BASELINE
// c1 size it is latency-bound (1.7 warps per scheduler) and at large K it is
// register/issue-bound at ~50 % of the FP32 pipe (profiles/r01).  One
// HMMA.16816 does 2 048 MACs in 8 issue-cycles of an SM sub-partition (B200,
// tools/probes/mma_probe.cu: 548 TFLOP/s f16, 276 TFLOP/s tf32 for mma.sync),
// so even three of them per product (hi*hi + hi*lo + lo*hi) beat FFMA2 by ~2x
// on the MLP, and the weights live in registers — no weight traffic at all.
//
// Numerics.  Every operand x is split as x = hi + lo with hi = fp16(x),
// lo = fp16(x - hi); the three products keep ~22 significant bits and the
// tensor core accumulates in fp32, so the MLP error is of the order of an fp32
// FMA evaluation (checked against the float restatement in the parity tests).
// tanh is folded into the layers: with k = 2 log2(e),
//   tanh(z) = 1 + 2 s,  s = -1 / (1 + 2^(k z)),
// so layer 1 multiplies by k*W1 (bias k*b1 through a constant-one input),
// layer 2 by 2k*W2 with bias k*(b2 + W2 1), layer 3 by 2*W3 with bias
// b3 + W3 1, and each activation costs one ex2, one add and one rcp.
//
// Layout (per warp, MT m16 tiles = 16*MT samples = one chunk):
//   A (activations) = rows = samples, B (weights, registers) = columns =
//   hidden units.  The m16n8 f32 accumulator of layer l is, element for
//   element, the A fragment of layer l+1 (rows g, g+8; k = 2t, 2t+1, 2t+8,
//   2t+9), so no data moves between layers.  Inputs enter and outputs leave
//   through a per-warp shared-memory stage.  Lane (g = lane/4, t = lane%4) owns
//   sample row g + 8 (t&1) of tile t>>1 (MT = 2), or of tile 0 with lanes
//   t >= 2 mirroring t - 2 (MT = 1): the owner runs the per-sample state,
//   noise, costmap and cost exactly as the FFMA2 kernel's roles do.
#pragma once

#include <cuda_fp16.h>

#include "rollout.cuh"
#include "tail.cuh"

namespace mppi_dev {

// Per-lane fragment words, stored [word][lane] (coalesced load at kernel start),
// for H hidden units (NJ = H/8 output n-tiles, NK = H/16 input k-tiles):
//   W1 .. : B1 (k8 x n8) n-tile j: hi = 2j, lo = 2j+1
//   W2 .. : B2 (k16 x n8): W2 + ((kk*NJ + j)*2 + r)*2 + hl    (r: b0/b1)
//   W3 .. : B3 (k16 x n8, outputs 0..3): W3 + (kk*2 + r)*2 + hl
//   B2 .. : bias2 (fp32 bits): B2 + j*2 + c, column 8j + 2t + c
//   B3 .. : bias3 (fp32 bits): column 2t + c (zero for t >= 2)
//   SC    : 2^-s (fp32 bits, every lane): layer 3 runs on 2^s-scaled weights
// H = 32 keeps every fragment in registers; at H = 64 the 128 layer-2 words
// live in shared memory (one LDS.128 per (kk, j), shared by the CTA's warps).
//
// Layer-3 scaling: 2 W3 (~0.08 for the BASELINE Xavier x 0.1 output layer)
// would leave the lo halves of its fp16 split (~4e-5) in the fp16 subnormal
// range below 6.1e-5, which keeps ~2^-24 absolute, not 11 significant bits:
// the output layer would carry ~10x the rounding of an fp32 evaluation.  The
// host scales W3 and its bias by the power of two s that brings max |2 W3|
// into [0.5, 1) (tc_build_fragments), which is exact, and the kernel folds
// 2^-s into the dt of the dynamic block: RN(d 2^s * dt 2^-s) = RN(d dt).
template <int H>
struct TcLayout {
  static constexpr int NJ = H / 8, NK = H / 16;
  static constexpr int W1 = 0, W2 = 2 * NJ, W3 = W2 + 4 * NK * NJ, B2 = W3 + 4 * NK, B3 = B2 + 2 * NJ;
  static constexpr int SC = B3 + 2;
  static constexpr int WORDS = SC + 1;
  static constexpr bool W2_SMEM = H > 32;
};
constexpr int kTcWords = TcLayout<32>::WORDS;  // 59
constexpr int kTcH = 32;

__device__ __forceinline__ void mma_k8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(b0));
}
__device__ __forceinline__ void mma_k16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// D = A B + C with C left intact (a bias quad feeds the first product directly)
__device__ __forceinline__ void mma_k16_c(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                          const float (&c)[4]) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c[0]), "f"(c[1]), "f"(c[2]), "f"(c[3]));
}

// A load the compiler cannot merge with an identical one: the repeated words
// of the bias quads {c, c+1, c, c+1} then stay in four live registers instead
// of being re-assembled with moves every step.
__device__ __forceinline__ float tc_ld_opaque(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return __uint_as_float(v);
}

__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// st.shared.b32 under a predicate, at a shared-window address: the owners'
// stage stores stay predicated instructions (a C++ `if` around them compiled
// to a branch with a reconvergence point in every step), and the address
// needs no generic-to-shared conversion inside the step loop
__device__ __forceinline__ void sts32_if(uint32_t addr, uint32_t v, bool p) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.b32 [%0], %1;\n\t}" ::"r"(addr), "r"(v),
               "r"(static_cast<int>(p))
               : "memory");
}

// (x, y) -> fp16x2 hi and lo words: hi = fp16(x), lo = fp16(x - hi).
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x, y);
  const float2 hf = __half22float2(h);
  const float2 r = __ffma2_rn(hf, make_float2(-1.f, -1.f), make_float2(x, y));
  hi = h2_bits(h);
  lo = h2_bits(__floats2half2_rn(r.x, r.y));
}

__device__ __forceinline__ float tc_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float tc_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// -1/d for 1 <= d <= 2^126 + 1 on the FMA pipe: bit-trick seed (|rel err| <=
// 5.1 %, the sign set by the wrapping subtraction; always a normal number in
// this range), one cubic Newton step (1.3e-4), one quadratic step (~2e-8,
// below half an fp32 ulp before rounding).  Negated so no FFMA2 operand
// needs a negation.
__device__ __forceinline__ float2 nrcp2_fma(float2 d) {
  float2 s = make_float2(__uint_as_float(0xFEF311C3u - __float_as_uint(d.x)),
                         __uint_as_float(0xFEF311C3u - __float_as_uint(d.y)));
  const float2 one = make_float2(1.f, 1.f);
  float2 e = __ffma2_rn(d, s, one);      // 1 - d/|d| (relative error of the seed)
  const float2 q = __ffma2_rn(e, e, e);  // e + e^2
  s = __ffma2_rn(s, q, s);               // s (1 + e + e^2)
  e = __ffma2_rn(d, s, one);
  return __ffma2_rn(s, e, s);
}
// s = -1 / (1 + 2^y) on a pair (tanh(z) = 1 + 2s with y = k z; the weights
// are folded accordingly, tc_build_fragments).  The ex2 runs on the SFU; the
// reciprocal on the SFU too unless SW, where it runs on the FMA pipe: at 4 SFU
// lanes per scheduler a warp-wide MUFU holds the pipe 8 cycles, and two per
// activation were the longest serial resource of a step.  SW clamps y at 126
// first (2^y must stay finite for the Newton residual).
template <bool SW = false>
__device__ __forceinline__ float2 act_r2(float y0, float y1) {
  if constexpr (SW) {
    const float2 d = __fadd2_rn(make_float2(tc_ex2(fminf(y0, 126.f)), tc_ex2(fminf(y1, 126.f))), make_float2(1.f, 1.f));
    return nrcp2_fma(d);
  } else {
    const float2 d = __fadd2_rn(make_float2(tc_ex2(y0), tc_ex2(y1)), make_float2(1.f, 1.f));
    return make_float2(tc_rcp(-d.x), tc_rcp(-d.y));
  }
}

// Which of the four activation pairs of acc_to_a take the FMA-pipe
// reciprocal (bit mask).  Measured (profiles/README.md): half at H = 32
// balances the SFU against the issue slots (c0 -5 %, c1 -1 %, K = 262144
// unchanged); at H = 64 the issue slots are the binding resource and the
// SFU reciprocal is faster (all-FMA: +11 % at c2).
template <int H>
__host__ __device__ constexpr int tc_sw_rcp() {
#ifdef MPPI_TC_SW_RCP
  return MPPI_TC_SW_RCP;
#else
  return H == 32 ? 10 : 0;
#endif
}
// Accumulator (n-tiles 2kk, 2kk+1) -> activation -> A fragment hi/lo of k-tile kk.
template <int SW>  // bit i: pair i of the four uses the FMA-pipe reciprocal
__device__ __forceinline__ void acc_to_a(const float (&d0)[4], const float (&d1)[4], uint32_t (&ahi)[4],
                                         uint32_t (&alo)[4]) {
  const float2 r00 = act_r2<(SW & 1) != 0>(d0[0], d0[1]), r01 = act_r2<(SW & 2) != 0>(d0[2], d0[3]);
  const float2 r10 = act_r2<(SW & 4) != 0>(d1[0], d1[1]), r11 = act_r2<(SW & 8) != 0>(d1[2], d1[3]);
  split2(r00.x, r00.y, ahi[0], alo[0]);  // row g,   k = 2t, 2t+1
  split2(r01.x, r01.y, ahi[1], alo[1]);  // row g+8, k = 2t, 2t+1
  split2(r10.x, r10.y, ahi[2], alo[2]);  // row g,   k = 2t+8, 2t+9
  split2(r11.x, r11.y, ahi[3], alo[3]);  // row g+8, k = 2t+8, 2t+9
}

// Branch-free sincos for the pose update: Cody-Waite reduction by pi/2 and
// near-minimax polynomials on [-pi/4, pi/4] (<= ~1 ulp there; no slow path,
// so the step body stays one basic block the scheduler can interleave).
__device__ __forceinline__ void tc_sincos(float x, float& s, float& c) {
  const float q = rintf(x * 0.636619772f);
  float r = __fmaf_rn(q, -1.57079625e+00f, x);
  r = __fmaf_rn(q, -7.54978942e-08f, r);
  r = __fmaf_rn(q, -5.39030253e-15f, r);
  const float z = r * r;
  float ps = __fmaf_rn(-1.95159533e-04f, z, 8.33216589e-03f);
  ps = __fmaf_rn(ps, z, -1.66666552e-01f);
  const float sr = __fmaf_rn(r * z, ps, r);
  float pc = __fmaf_rn(2.43892027e-05f, z, -1.38867483e-03f);
  pc = __fmaf_rn(pc, z, 4.16666232e-02f);
  pc = __fmaf_rn(pc, z, -0.5f);
  const float cr = __fmaf_rn(z, pc, 1.0f);
  const int iq = static_cast<int>(q);
  const float s0 = (iq & 1) ? cr : sr;
  const float c0 = (iq & 1) ? sr : cr;
  s = (iq & 2) ? -s0 : s0;
  c = ((iq + 1) & 2) ? -c0 : c0;
}

// state_cost (costs.cpp:29-43) + the BASELINE crash term, branch-free, same
// rounded operation sequence as state_cost_h (model.cuh).
template <bool STAB>
__device__ __forceinline__ float tc_state_cost(float h, float roll, float vx, float vy, float decay_t,
                                               const CostDev<float>& cp) {
  const float track = add_rn(h, (h > cp.boundary_threshold) ? mul_rn(decay_t, cp.impulse) : 0.f);
  const float dv = sub_rn(vx, cp.v_des);
  float c = add_rn(mul_rn(cp.alpha_track, track), mul_rn(cp.alpha_speed, mul_rn(dv, dv)));
  if constexpr (STAB) {
    const float zeta = (fabsf(vx) < 0.01f) ? 0.f : -atanf(__fdiv_rn(vy, fabsf(vx)));
    const float stab = add_rn(mul_rn(zeta, zeta), (fabsf(zeta) > cp.slip_limit) ? cp.impulse : 0.f);
    c = add_rn(c, mul_rn(cp.alpha_stab, stab));
  }
  const bool crash = cp.crash_penalty != 0.f && (h > cp.crash_threshold || fabsf(roll) > cp.roll_limit);
  return add_rn(c, crash ? cp.crash_penalty : 0.f);
}

// Two fp32 m16n8 accumulators per output tile: `m` takes hi*hi (and the
// bias), `c` the two cross terms; they are added once at the end, so the
// full-magnitude accumulator sees 1-2 tensor-core roundings per layer instead
// of 6, and the three product chains run in parallel.
struct Acc2 {
  float m[4], c[4];
};
__device__ __forceinline__ void acc2_sum(const Acc2& a, float (&d)[4]) {
  const float2 x = __fadd2_rn(make_float2(a.m[0], a.m[1]), make_float2(a.c[0], a.c[1]));
  const float2 y = __fadd2_rn(make_float2(a.m[2], a.m[3]), make_float2(a.c[2], a.c[3]));
  d[0] = x.x;
  d[1] = x.y;
  d[2] = y.x;
  d[3] = y.y;
}

// The layer-1 A operand in fragment order: plane hl (0 hi, 1 lo), word
// tc_in_word(g, p, h) holds the fp16x2 input pair p of sample row g + 8h, so
// lane (g, t) reads its {row g, row g+8} operand pair as one LDS.64 straight
// into the HMMA source registers.  Pairs: (roll,vx), (vy,thd), (v0,v1), (1,0).
// The pair index is XOR-swizzled by g >> 2 so the owners' 32-bit stores are
// bank-conflict-free as well as the reads.
__device__ __forceinline__ int tc_in_word(int g, int p, int h) { return g * 8 + 2 * (p ^ (g >> 2)) + h; }
// c = sum of the per-k-tile cross-term accumulators, in k-tile order
template <int NK>
__device__ __forceinline__ void tc_sum_cross(const float (&c)[NK][4], float (&out)[4]) {
  float2 x = make_float2(c[0][0], c[0][1]), y = make_float2(c[0][2], c[0][3]);
#pragma unroll
  for (int kk = 1; kk < NK; ++kk) {
    x = __fadd2_rn(x, make_float2(c[kk][0], c[kk][1]));
    y = __fadd2_rn(y, make_float2(c[kk][2], c[kk][3]));
  }
  out[0] = x.x;
  out[1] = x.y;
  out[2] = y.x;
  out[3] = y.y;
}

template <int MT>
struct TcStage {
  uint32_t in[MT][2][64];  // [tile][hi/lo][tc_in_word]
  float4 out[MT][16];      // layer-3 outputs per sample row
};
constexpr int kTcTB = 16;  // timesteps per block of the numerator reduction
constexpr int kTcRedStride = 33;  // doubles per row (padding: conflict-free column reads)
// doubles of numerator scratch per warp: the staged reduction of regenerated
// eps', or the chunk's 16 softmin weights when eps' is on chip
__host__ __device__ constexpr int tc_red_doubles(bool store) { return store ? 16 : 2 * kTcTB * kTcRedStride; }

// MLP of one step for MT tiles: inputs from the stage, outputs d3 (fp32).
// side1 / side2: independent per-sample work of the step, placed between the
// layers so the scheduler interleaves it with the tensor-core chains (it
// otherwise lands after the MLP as a separate dependent block).  b2frag(kk, j)
// returns the layer-2 B fragment words (b0 hi, b0 lo, b1 hi, b1 lo).
template <int H, int MT, class B2Frag, class Side1, class Side2>
__device__ __forceinline__ void tc_mlp(const TcStage<MT>& st, int g, int t4, const uint32_t (&w1)[2 * (H / 8)],
                                       B2Frag&& b2frag, const uint32_t (&w3)[4 * (H / 16)],
                                       const float (&b2)[H / 8][4], const float (&b3)[4], float (&d3)[MT][4],
                                       Side1&& side1, Side2&& side2) {
  constexpr int NJ = H / 8, NK = H / 16;
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    // ---- layer 1 (k8): A rows g, g+8; k = 2t, 2t+1 (bias through the constant-one column)
    const int w = tc_in_word(g, t4, 0);
    const uint2 ah = *reinterpret_cast<const uint2*>(&st.in[m][0][w]);  // hi: rows g, g+8
    const uint2 al = *reinterpret_cast<const uint2*>(&st.in[m][1][w]);  // lo
    float d1[NJ][4];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      Acc2 a;
#pragma unroll
      for (int i = 0; i < 4; ++i) a.m[i] = a.c[i] = 0.f;
      mma_k8(a.c, al.x, al.y, w1[2 * j]);      // lo * hi
      mma_k8(a.c, ah.x, ah.y, w1[2 * j + 1]);  // hi * lo
      mma_k8(a.m, ah.x, ah.y, w1[2 * j]);      // hi * hi
      acc2_sum(a, d1[j]);
    }
    if (m == MT - 1) side1();
    // ---- layer 2 (NK x k16)
    Acc2 a2[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
#pragma unroll
      for (int i = 0; i < 4; ++i) a2[j].c[i] = 0.f;
    }
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
      uint32_t ahi[4], alo[4];
      acc_to_a<tc_sw_rcp<H>()>(d1[2 * kk], d1[2 * kk + 1], ahi, alo);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const uint4 b = b2frag(kk, j);  // b0 hi, b0 lo, b1 hi, b1 lo
        mma_k16(a2[j].c, alo, b.x, b.z);
        mma_k16(a2[j].c, ahi, b.y, b.w);
        if (kk == 0)
          mma_k16_c(a2[j].m, ahi, b.x, b.z, b2[j]);  // the bias enters as C
        else
          mma_k16(a2[j].m, ahi, b.x, b.z);
      }
    }
    float d2[NJ][4];
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc2_sum(a2[j], d2[j]);
    if (m == MT - 1) side2();
    // ---- layer 3 (NK x k16, n = 8: outputs 0..3)
    // (the last layer ends the step's dependent chain: its cross terms
    // accumulate per k-tile, two chains of two instead of one of 2*NK)
    Acc2 a3;
    float c3[NK][4];
#pragma unroll
    for (int kk = 0; kk < NK; ++kk)
#pragma unroll
      for (int i = 0; i < 4; ++i) c3[kk][i] = 0.f;
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
      uint32_t ahi[4], alo[4];
      acc_to_a<tc_sw_rcp<H>()>(d2[2 * kk], d2[2 * kk + 1], ahi, alo);
      const int b = kk * 4;
      mma_k16(c3[kk], alo, w3[b], w3[b + 2]);
      mma_k16(c3[kk], ahi, w3[b + 1], w3[b + 3]);
      if (kk == 0)
        mma_k16_c(a3.m, ahi, w3[b], w3[b + 2], b3);
      else
        mma_k16(a3.m, ahi, w3[b], w3[b + 2]);
    }
    tc_sum_cross<NK>(c3, a3.c);
    acc2_sum(a3, d3[m]);
  }
}

// grid = (ceil(chunks / NW), controllers), block = 32 * NW; one warp = one
// chunk of 16*MT samples.  Dynamic smem: plan (2T + 2 floats), then the
// numerator reduction buffers (NW x 2*kTcTB x kTcRedStride doubles).
// Resident CTAs per SM the register budget is sized for (measured,
// profiles/README.md): MT = 2 three (168 registers; four spills); MT = 1 at
// H = 32 three (158 registers, no spills: the group-merge CTAs of the
// programmatic-dependent launch then fit beside two K1 CTAs, c1 -1.3 %);
// H = 64 two (its layer-2 chain needs the registers: three is +8 % at c2).
template <int H, int MT>
__host__ __device__ constexpr int tc_min_ctas() {
  return (MT == 2 || H == 32) ? 3 : 2;
}
// PST: the owners' stage stores as predicated st.shared (sts32_if) instead of
// a C++ `if` (a branch and a reconvergence point per step): measured -7 % K1
// at <= 1 warp per scheduler (K = 4096, 8192), +1 % at c1's 1.7 (tc_launch.cuh
// picks it by the grid size; same arithmetic, bit-identical results).
template <int H, int MT, int NW, int Mode, bool STAB, bool STORE, bool TRACE, bool PST = false>
__global__ void __launch_bounds__(32 * NW, tc_min_ctas<H, MT>()) rollout_tc_kernel(const __grid_constant__ RolloutArgs<float> a,
                                                            const uint32_t* __restrict__ frag) {
  constexpr int CH = 16 * MT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int T = a.T;
  float* s_plan = reinterpret_cast<float*>(smem_raw);
  double* s_red_all = reinterpret_cast<double*>(smem_raw + ((sizeof(float) * (2 * T + 2) + 15) & ~size_t(15)));
  // STORE: the rollout keeps eps' (the batch as rollout_batch leaves it) of
  // its samples on chip, [warp][t][sample] float2, for the numerator pass —
  // used when the whole grid fits one wave with this footprint (small K);
  // otherwise eps' is regenerated from the counters.
  float2* s_eps_all = reinterpret_cast<float2*>(s_red_all + static_cast<size_t>(NW) * tc_red_doubles(STORE));
  __shared__ __align__(16) TcStage<MT> s_stage[NW];

  const int ctrl = blockIdx.y;
  if (a.abort_flag[static_cast<size_t>(ctrl) * a.abort_stride] != 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int chunk = a.chunk0 + blockIdx.x * NW + warp;
  for (int i = threadIdx.x; i < 2 * T + 2; i += 32 * NW)
    s_plan[i] = (i < 2 * T) ? a.plan[static_cast<size_t>(ctrl) * 2 * T + i] : 0.f;

  // weights + biases into registers (loop-invariant for the whole rollout);
  // at H = 64 the layer-2 fragments go to shared memory instead
  using L = TcLayout<H>;
  uint32_t w1[2 * L::NJ], w3[4 * L::NK];
  uint32_t w2r[L::W2_SMEM ? 1 : 4 * L::NK * L::NJ];
  float b2[L::NJ][4], b3[4];  // bias quads in accumulator order {c, c+1, c, c+1}
  __shared__ __align__(16) uint4 s_w2[L::W2_SMEM ? L::NK * L::NJ : 1][32];
#pragma unroll
  for (int i = 0; i < 2 * L::NJ; ++i) w1[i] = frag[(L::W1 + i) * 32 + lane];
  if constexpr (L::W2_SMEM) {
    for (int f = warp; f < L::NK * L::NJ; f += NW)
      s_w2[f][lane] = make_uint4(frag[(L::W2 + 4 * f) * 32 + lane], frag[(L::W2 + 4 * f + 1) * 32 + lane],
                                 frag[(L::W2 + 4 * f + 2) * 32 + lane], frag[(L::W2 + 4 * f + 3) * 32 + lane]);
  } else {
#pragma unroll
    for (int i = 0; i < 4 * L::NK * L::NJ; ++i) w2r[i] = frag[(L::W2 + i) * 32 + lane];
  }
#pragma unroll
  for (int i = 0; i < 4 * L::NK; ++i) w3[i] = frag[(L::W3 + i) * 32 + lane];
#pragma unroll
  for (int j = 0; j < L::NJ; ++j) {
    b2[j][0] = __uint_as_float(frag[(L::B2 + 2 * j) * 32 + lane]);
    b2[j][1] = __uint_as_float(frag[(L::B2 + 2 * j + 1) * 32 + lane]);
    b2[j][2] = tc_ld_opaque(frag + (L::B2 + 2 * j) * 32 + lane);
    b2[j][3] = tc_ld_opaque(frag + (L::B2 + 2 * j + 1) * 32 + lane);
  }
  b3[0] = __uint_as_float(frag[L::B3 * 32 + lane]);
  b3[1] = __uint_as_float(frag[(L::B3 + 1) * 32 + lane]);
  b3[2] = tc_ld_opaque(frag + L::B3 * 32 + lane);
  b3[3] = tc_ld_opaque(frag + (L::B3 + 1) * 32 + lane);
  auto b2frag = [&](int kk, int j) -> uint4 {
    if constexpr (L::W2_SMEM) {
      return s_w2[kk * L::NJ + j][lane];
    } else {
      const int b = (kk * L::NJ + j) * 4;
      return make_uint4(w2r[b], w2r[b + 1], w2r[b + 2], w2r[b + 3]);
    }
  };

  TcStage<MT>& st = s_stage[warp];
  // the constant-one input column (k = 6: bias of layer 1), written once
  for (int i = lane; i < CH; i += 32) {
    const int w = tc_in_word(i & 7, 3, (i >> 3) & 1);
    st.in[i >> 4][0][w] = h2_bits(__floats2half2_rn(1.f, 0.f));
    st.in[i >> 4][1][w] = 0u;
  }

  // ---- owner: the sample this lane runs the scalar path for
  const int m_own = (MT == 2) ? (t4 >> 1) : 0;
  const int row_own = g + 8 * (t4 & 1);
  const bool dup = (MT == 1) && (t4 >= 2);  // MT = 1: lanes t >= 2 mirror t - 2
  const int k = chunk * CH + 16 * m_own + row_own;
  // warps past the rank's last chunk (last CTA only) run without writing
  // anything (they keep the warp-synchronous code uniform)
  const bool active = chunk < a.chunk_end;
  const bool valid = (k < a.K) && !dup && active;
  const bool zm = k >= a.zero_start;
  const int kn = (k < a.K) ? k : 0;  // noise counter (in range for every lane)
  const float dt = a.sys.dt;
  const float dt3 = dt * __uint_as_float(frag[L::SC * 32 + lane]);  // dt 2^-s (exact)
  const CostDev<float> cp = a.sys.cost;
  const float inv_s0 = 1.0f / a.sigma0, inv_s1 = 1.0f / a.sigma1;
  const float gml = a.gamma - a.lambda, half_lambda = 0.5f * a.lambda;
  __syncthreads();  // s_plan, stage constants
  // a one-wave grid (the on-chip eps' variant) lets its dependent tail kernel
  // launch now: the tail's CTAs wait in cudaGridDependencySynchronize for
  // this grid's completion, but their launch latency is hidden
  if constexpr (STORE) cudaTriggerProgrammaticLaunchCompletion();

  // Noise: Philox draws one 128-bit block per step pair; the other modes (parity)
  // go through the generic per-step stream.
  NoiseStream<float, Mode> ns = make_noise<float, Mode>(a, ctrl, kn);
  const uint64_t seed = a.seeds[ctrl], iteration = a.iters[ctrl];
  float zc0 = 0.f, zc1 = 0.f;  // Philox: the odd step of the current draw
  auto eps_at = [&](int t, bool even, float& e0, float& e1) {
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
  };
  // v_t = g(u_t + eps_t) and the coupling of step t (controller.cpp:86-101)
  float v0c, v1c, coup_t;
  float2* s_eps = STORE ? s_eps_all + static_cast<size_t>(warp) * T * CH : nullptr;
  const int s_own = 16 * m_own + row_own;
  auto produce_v = [&](int t, bool even) {
    float e0, e1;
    eps_at(t, even, e0, e1);
    const float u0 = s_plan[2 * t], u1 = s_plan[2 * t + 1];
    e0 = zm ? e0 - u0 : e0;
    e1 = zm ? e1 - u1 : e1;
    if constexpr (STORE) {
      if (t < T && !dup) s_eps[t * CH + s_own] = make_float2(e0, e1);  // owners only (predicated)
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
  const bool trace = a.trace_states != nullptr && valid && k == a.trace_k;
  // this lane's stage-input words (shared-window byte addresses)
  const uint32_t s_in_hi = static_cast<uint32_t>(__cvta_generic_to_shared(&st.in[m_own][0][0]));
  const uint32_t s_in_lo = static_cast<uint32_t>(__cvta_generic_to_shared(&st.in[m_own][1][0]));
  const uint32_t w_in0 = 4u * tc_in_word(g, 0, t4 & 1), w_in1 = 4u * tc_in_word(g, 1, t4 & 1),
                 w_in2 = 4u * tc_in_word(g, 2, t4 & 1);
  produce_v(0, true);

  // One step; EVEN = parity of t (compile-time, so the Philox draw of the
  // next pair is unconditional code in the odd step).
  auto step = [&](int t, auto even_tag) {
    constexpr bool EVEN = decltype(even_tag)::value;
    // pose of x_{t+1}: the Euler split (dynamics.cpp:137-148) reads only the
    // old state, so it runs before the MLP and the costmap taps of x_{t+1}
    // are in flight for a whole step before its cost consumes them
    float sn, cs;
    tc_sincos(th, sn, cs);
    px = add_rn(px, mul_rn(sub_rn(mul_rn(cs, vx), mul_rn(sn, vy)), dt));
    py = add_rn(py, mul_rn(add_rn(mul_rn(sn, vx), mul_rn(cs, vy)), dt));
    th = add_rn(th, mul_rn(thd, dt));
    const MapTaps<float> q_next = map_fetch(map, px, py);
    // stage this step's inputs (the owners' predicated stores: the MT = 1
    // mirror lanes compute the same values and store nothing, so no two
    // lanes write one word and no branch splits the step's basic block)
    {
      uint32_t hi0, lo0, hi1, lo1, hi2, lo2;
      split2(roll, vx, hi0, lo0);
      split2(vy, thd, hi1, lo1);
      split2(v0c, v1c, hi2, lo2);
      if constexpr (PST) {
        sts32_if(s_in_hi + w_in0, hi0, !dup);
        sts32_if(s_in_lo + w_in0, lo0, !dup);
        sts32_if(s_in_hi + w_in1, hi1, !dup);
        sts32_if(s_in_lo + w_in1, lo1, !dup);
        sts32_if(s_in_hi + w_in2, hi2, !dup);
        sts32_if(s_in_lo + w_in2, lo2, !dup);
      } else if (!dup) {
        uint32_t* hi_plane = st.in[m_own][0];
        uint32_t* lo_plane = st.in[m_own][1];
        const int h = t4 & 1;
        hi_plane[tc_in_word(g, 0, h)] = hi0;
        lo_plane[tc_in_word(g, 0, h)] = lo0;
        hi_plane[tc_in_word(g, 1, h)] = hi1;
        lo_plane[tc_in_word(g, 1, h)] = lo1;
        hi_plane[tc_in_word(g, 2, h)] = hi2;
        lo_plane[tc_in_word(g, 2, h)] = lo2;
      }
    }
    __syncwarp();
    float d3[MT][4];
    // independent of this step's MLP (overlaps it): running cost of step t-1
    // on x_t (taps fetched last step), and v_{t+1}
    tc_mlp<H, MT>(st, g, t4, w1, b2frag, w3, b2, b3, d3,
               [&] {
                 const float h = map_interp(q);
                 const float rc = tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[t > 0 ? t - 1 : 0], cp);
                 cost += (t > 0) ? static_cast<Acc>(add_rn(rc, p_coup)) : 0.0;
                 p_coup = coup_t;
               },
               [&] { produce_v(t + 1, !EVEN); });
    // outputs to their owners: columns 2t, 2t+1 live in lanes t = 0, 1
    if (t4 < 2) {
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        reinterpret_cast<float2*>(&st.out[m][g])[t4] = make_float2(d3[m][0], d3[m][1]);
        reinterpret_cast<float2*>(&st.out[m][g + 8])[t4] = make_float2(d3[m][2], d3[m][3]);
      }
    }
    __syncwarp();
    const float4 d = st.out[m_own][row_own];
    // the dynamic block of the Euler split
    roll = add_rn(roll, mul_rn(d.x, dt3));
    vx = add_rn(vx, mul_rn(d.y, dt3));
    vy = add_rn(vy, mul_rn(d.z, dt3));
    thd = add_rn(thd, mul_rn(d.w, dt3));
    q = q_next;  // consumed by the next step's cost
    p_roll = roll;
    p_vx = vx;
    p_vy = vy;
    if (TRACE && trace) {
      float* so = a.trace_states + (t + 1) * 7;
      so[0] = px; so[1] = py; so[2] = th; so[3] = roll; so[4] = vx; so[5] = vy; so[6] = thd;
    }
  };
  int t = 0;
  for (; t + 1 < T; t += 2) {
    step(t, std::true_type{});
    step(t + 1, std::false_type{});
  }
  if (t < T) step(t, std::true_type{});

  // ---- terminal cost and the chunk softmin partials
  {
    const float h = map_interp(q);
    cost += static_cast<Acc>(add_rn(tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[T - 1], cp), p_coup));
    if (a.sys.with_terminal) cost += static_cast<Acc>(tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[T], cp));
  }
  MPPI_DCHECK(!valid || (k >= 0 && k < a.K));
  if (valid) a.costs[static_cast<size_t>(ctrl) * a.K + k] = cost;
  const bool bad = valid && !isfinite(cost);
  const Acc rho = warp_min(valid ? cost : Acc(INFINITY));
  const Acc wk = valid ? exp(-(cost - rho) / a.dlambda) : 0.0;
  const Acc eta = warp_sum(wk);
  const unsigned any_bad = __ballot_sync(0xffffffffu, bad);
  Acc* out = a.partials + static_cast<size_t>(ctrl) * a.partials_ctrl_stride +
             static_cast<size_t>(chunk) * a.partial_stride;
  MPPI_DCHECK(!active || (chunk >= a.chunk0 && static_cast<long long>(chunk + 1) * a.partial_stride <=
                                                    a.partials_ctrl_stride));
  MPPI_DCHECK(a.partial_stride == kPartialHeader + 2 * T);
  if (lane == 0) MPPI_STAMP_MAX(0);  // K1: last warp through the rollout
  if (lane == 0 && active) {
    out[0] = rho;
    out[1] = eta;
    out[2] = any_bad ? 1.0 : 0.0;
    out[3] = 0.0;
  }
  // numerators over the regenerated batch (eps' = eps - U for zero-mean):
  // blocks of kTcTB steps, products staged [t][c][lane] in shared memory and
  // summed per (t, c) over the lanes in ascending lane order by one lane each.
  double* red = s_red_all + static_cast<size_t>(warp) * tc_red_doubles(STORE);
  if constexpr (STORE && MT == 1) {
    // eps' is on chip: each lane sums whole (t, c) elements over the chunk's
    // rows with the staged reduction's order below (rows 0..7 and rows 8..15
    // as two sequential sums of rounded products, then their sum plus the
    // mirror lanes' zero sums), so the partials are bit-identical to it and
    // to the warp-pair kernel's: which variant a launch picks (it depends on
    // the rank's grid size) never changes a result.
    if (!dup) red[row_own] = wk;
    __syncwarp();
    for (int e = lane; e < 2 * T; e += 32) {
      const int tt = e >> 1, c = e & 1;
      Acc sa = 0.0, sb = 0.0;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const float2 ea = s_eps[tt * CH + r], eb = s_eps[tt * CH + r + 8];
        sa = __dadd_rn(sa, __dmul_rn(red[r], static_cast<Acc>(c ? ea.y : ea.x)));
        sb = __dadd_rn(sb, __dmul_rn(red[r + 8], static_cast<Acc>(c ? eb.y : eb.x)));
      }
      if (active) out[kPartialHeader + e] = __dadd_rn(__dadd_rn(sa, sb), 0.0);
    }
    __syncwarp();
  } else {
  if constexpr (Mode != kPhilox) ns = make_noise<float, Mode>(a, ctrl, kn);
  for (int tb = 0; tb < T; tb += kTcTB) {
#pragma unroll 2
    for (int j = 0; j < kTcTB; ++j) {
      const int tt = tb + j;
      float e0 = 0.f, e1 = 0.f;
      if (tt < T) {
        if constexpr (STORE) {
          const float2 ev = s_eps[tt * CH + s_own];
          e0 = ev.x;
          e1 = ev.y;
        } else {
          eps_at(tt, (tt & 1) == 0, e0, e1);
          e0 = zm ? e0 - s_plan[2 * tt] : e0;
          e1 = zm ? e1 - s_plan[2 * tt + 1] : e1;
        }
      }
      red[(2 * j) * kTcRedStride + lane] = __dmul_rn(wk, static_cast<Acc>(e0));
      red[(2 * j + 1) * kTcRedStride + lane] = __dmul_rn(wk, static_cast<Acc>(e1));
    }
    __syncwarp();
    // four interleaved partial sums (lanes l = 4i + q), then q = 0..3: a
    // fixed order with an 8-deep dependent chain instead of 32.  At MT = 1
    // q = 0 holds rows 0..7, q = 1 rows 8..15 and q = 2, 3 the mirror lanes'
    // zeros — the order of the on-chip eps' path above.
    Acc s4[4] = {0.0, 0.0, 0.0, 0.0};
    const double* col = red + lane * kTcRedStride;
#pragma unroll
    for (int l = 0; l < 32; l += 4) {
#pragma unroll
      for (int q = 0; q < 4; ++q) s4[q] = __dadd_rn(s4[q], col[l + q]);
    }
    const Acc s = __dadd_rn(__dadd_rn(s4[0], s4[1]), __dadd_rn(s4[2], s4[3]));
    if (active && tb + (lane >> 1) < T) out[kPartialHeader + 2 * tb + lane] = s;
    __syncwarp();
  }
  }
}

}  // namespace mppi_dev
