// rollout_umma.cuh — K1 on the 5th-generation tensor cores (tcgen05 / TMEM),
// H = 32 and 64, for the throughput configurations.
//
// One CTA of 128 threads owns a chunk of 128 samples, ONE SAMPLE PER THREAD:
// thread r runs sample r's whole scalar path (Philox noise, coupling, clamp,
// Euler split, costmap, cost — no mirror lanes) and owns row r of every
// per-layer M = 128 tile.  Per step and layer the threads stage their rows
// of the A operand (fp16 hi and lo of the layer input) in shared memory in
// the canonical K-major no-swizzle UMMA layout, one elected thread issues the
// layer's tcgen05.mma (M = 128, N = H or 16, K = 16 per slice; hi*hi into one TMEM
// accumulator, hi*lo + lo*hi into another, as the mma.sync kernel's m/c
// split), commits them to an mbarrier, and every thread reads its row back
// with tcgen05.ld (TMEM lane = thread).  Weights (B operands, fp16 hi/lo,
// tanh folded as in rollout_tc.cuh) stay in shared memory for the whole
// rollout; the accumulators use 2H TMEM columns per CTA.
//
// Compared with the mma.sync kernel this removes the warp-issued HMMAs, the
// fragment bookkeeping and the mirror-lane duplication of the scalar path; it
// adds three CTA barriers + three mbarrier waits per step, so it is meant for
// grids of several CTAs per SM (c2-c4 sizes), where they hide each other's
// waits.  Results agree with the other K1 variants to fp32 rounding (not
// bitwise: the accumulation inside the tensor core differs).
#pragma once

#include <cuda_fp16.h>

#include "rollout_tc.cuh"

namespace mppi_dev {

constexpr int kUmmaThreads = 128;  // samples (= TMEM lanes, = MMA M) per CTA
// bit p: pair p of every 8 activations takes the FMA-pipe reciprocal (the rest
// the SFU); H = 64 defaults to the SFU for all of them, as the mma.sync kernel
template <int H>
__host__ __device__ constexpr int umma_sw_rcp() {
#ifdef MPPI_UMMA_SW
  return MPPI_UMMA_SW;
#else
  return H == 32 ? 10 : 0;
#endif
}
// 128-sample tiles per CTA (default one).  With two, a CTA runs two
// independent MMA pipelines (256 threads, a named barrier per tile) sharing
// ONE shared-memory copy of the weights: at H = 64 the weights are 24 KB of
// the 66 KB per-tile footprint, so CTA pairs hold four tiles per SM where
// single-tile CTAs fit three.  Measured (-DMPPI_UMMA_TPC=2, H = 64, 128
// registers): c2 K1 1165 -> 1118 us (one wave instead of 1.15), but
// K = 32768 +17 % and K = 131072 +13 %.  So the launcher picks the two-tile
// CTAs at H = 64 only when they fit the grid in one wave and single tiles
// do not (umma_launch.cuh: the c2 band, 445 .. 592 tiles per controller set).
template <int H>
__host__ __device__ constexpr int umma_tiles_per_cta() {
#ifdef MPPI_UMMA_TPC
  return MPPI_UMMA_TPC;
#else
  return 1;
#endif
}
// resident CTAs per SM the register budget is sized for: four tiles at H = 32
// (128 registers), three at H = 64 (its shared-memory footprint allows no
// more), two two-tile CTAs
template <int H, int TPC = umma_tiles_per_cta<H>()>
__host__ __device__ constexpr int umma_min_ctas() {
#ifdef MPPI_UMMA_CTAS
  return MPPI_UMMA_CTAS;
#else
  return TPC == 2 ? 2 : (H == 32 ? 4 : 3);
#endif
}
// accumulators per tile: [0, H) hi*hi, [H, 2H) cross terms
template <int H, int TPC = umma_tiles_per_cta<H>()>
__host__ __device__ constexpr int umma_tmem_cols() { return 2 * H * TPC; }

// Byte offset of element (row, k) of a K = 16 fp16 tile in the canonical
// K-major, no-swizzle layout: 8-row x 16-byte core matrices, the two K halves
// 128 B apart (LBO), 8-row groups 256 B apart (SBO).
__host__ __device__ constexpr uint32_t umma_tile_offset(int row, int k) {
  return static_cast<uint32_t>((row & 7) * 16 + (row >> 3) * 256 + (k >> 3) * 128 + (k & 7) * 2);
}
constexpr uint32_t kUmmaTileA = 128 * 32;  // bytes of an M = 128, K = 16 fp16 tile
// Weight image (host-built, copied to shared memory as is): fp16 B tiles in
// the layout above (N rows x K = 16 per slice; layers 2/3 have H/16 K slices),
// then the fp32 bias vectors and the layer-3 scale.
template <int H>
struct UmmaLayout {
  static constexpr int NK = H / 16;                                         // K slices of layers 2 and 3
  static constexpr uint32_t W1_HI = 0, W1_LO = 32 * H;                      // N = H, K = 16
  static constexpr uint32_t W2_HI = 64 * H, W2_LO = W2_HI + NK * 32 * H;    // NK slices x (32 H) B
  static constexpr uint32_t W3_HI = W2_LO + NK * 32 * H, W3_LO = W3_HI + NK * 512;  // N = 16: NK x 512 B
  static constexpr uint32_t B2 = W3_LO + NK * 512;                          // H floats
  static constexpr uint32_t B3 = B2 + 4 * H;                                // 4 floats (+ pad)
  static constexpr uint32_t SC = B3 + 16;                                   // 2^-s (1 float)
  static constexpr uint32_t BYTES = ((SC + 4) + 15) & ~15u;
};

// UMMA shared-memory descriptor (K-major, SWIZZLE_NONE, LBO 128 B, SBO 256 B, version 1).
__device__ __forceinline__ uint64_t umma_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(128 >> 4) << 16;
  d |= static_cast<uint64_t>(256 >> 4) << 32;
  d |= 1ull << 46;  // version (sm_100)
  return d;        // base offset 0, lbo mode 0, layout type 0 (no swizzle)
}
// Instruction descriptor: F16 x F16 -> F32, K-major A and B, M = 128, N.
__host__ __device__ constexpr uint32_t umma_idesc(int n) {
  return (1u << 4) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(mbar), "r"(phase), "r"(0x989680u)  // suspend-time hint: sleep until the phase completes
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tc05_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc05_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void proxy_fence_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 16 / 4 consecutive fp32 TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// One hidden layer from TMEM to the next layer's A operand, two K slices
// (32 hidden units) at a time: this thread's row of the hi*hi and cross
// accumulators of both slices first (one tcgen05.wait), then per unit the sum
// (+ the bias when BIAS), the activation (tanh folded: s = -1/(1 + 2^y), pairs on the
// SFU or the FMA-pipe reciprocal per SW), the fp16 hi/lo split, and the rows
// of the A tiles (hi and lo planes) — the 16 activation pairs of a group are
// independent chains the scheduler interleaves.
template <int H, int SW, bool BIAS>
__device__ __forceinline__ void umma_layer_to_a(uint32_t t_lane, const float* __restrict__ bias, uint32_t a_hi,
                                                uint32_t a_lo, int row) {
#pragma unroll
  for (int s0 = 0; s0 < H / 16; s0 += 2) {
    float y[32];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float m16[16], c16[16];
      tmem_ld16(t_lane + 16 * (s0 + q), m16);
      tmem_ld16(t_lane + H + 16 * (s0 + q), c16);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        float2 z = __fadd2_rn(make_float2(m16[j], m16[j + 1]), make_float2(c16[j], c16[j + 1]));
        if constexpr (BIAS) z = __fadd2_rn(z, make_float2(bias[16 * (s0 + q) + j], bias[16 * (s0 + q) + j + 1]));
        y[16 * q + j] = z.x;
        y[16 * q + j + 1] = z.y;
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // K halves of slice s0 + q: hidden 16 (s0 + q) + 8h .. +7
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int j = 16 * q + 8 * h + 2 * p;
          const float2 r = ((SW >> p) & 1) ? act_r2<true>(y[j], y[j + 1]) : act_r2<false>(y[j], y[j + 1]);
          split2(r.x, r.y, hw[p], lw[p]);
        }
        const uint32_t off = static_cast<uint32_t>(s0 + q) * kUmmaTileA + umma_tile_offset(row, 8 * h);
        sts128(a_hi + off, hw[0], hw[1], hw[2], hw[3]);
        sts128(a_lo + off, lw[0], lw[1], lw[2], lw[3]);
      }
    }
  }
}

// grid = (ceil(chunks / TPC), controllers), block = 128 TPC, tile i of a CTA
// = chunk blockIdx.x TPC + i of 128 samples.  Dynamic smem: plan (2T + 2
// floats) | weight image (UmmaLayout<H>) | per tile: A tiles: layer 1 hi/lo
// (2 x 4 KB), layers 2/3 hi/lo x H/16 K slices, with the numerator staging
// (kTcTB x 2 x 128 doubles) aliased on them after the rollout.
template <int H>
__host__ __device__ constexpr size_t umma_tile_region_bytes() {
  const size_t tiles = (2 + 2 * (H / 16)) * kUmmaTileA;
  const size_t stage = sizeof(double) * kTcTB * 2 * kUmmaThreads;
  return tiles > stage ? tiles : stage;
}
template <int H, int TPC = umma_tiles_per_cta<H>()>
__host__ __device__ constexpr size_t umma_smem_bytes(int T) {
  const size_t plan = (sizeof(float) * (2 * T + 2) + 127) & ~size_t(127);
  return plan + UmmaLayout<H>::BYTES + TPC * umma_tile_region_bytes<H>() + 128;
}
// a named barrier over the 128 threads of tile `tile` (ids 1 ..; 0 is __syncthreads)
__device__ __forceinline__ void umma_tile_bar(int tile) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + tile), "n"(kUmmaThreads) : "memory");
}

template <int H, int Mode, bool STAB, bool TRACE, int TPC = umma_tiles_per_cta<H>()>
__global__ void __launch_bounds__(kUmmaThreads * TPC, umma_min_ctas<H, TPC>()) rollout_umma_kernel(
    const __grid_constant__ RolloutArgs<float> a, const unsigned char* __restrict__ wimg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_taddr;
  __shared__ __align__(8) unsigned long long s_mbar_all[TPC];
  __shared__ double s_red_all[TPC][kUmmaThreads / 32];
  __shared__ int s_bad_all[TPC];
  const int T = a.T;
  // tid: this thread's row (sample) of its tile; warp: its warp within the
  // tile (= its TMEM lane quarter)
  const int tile = TPC == 1 ? 0 : static_cast<int>(threadIdx.x) / kUmmaThreads;
  const int tid = TPC == 1 ? static_cast<int>(threadIdx.x) : static_cast<int>(threadIdx.x) % kUmmaThreads;
  const int warp = tid >> 5, lane = tid & 31;
  const int ctrl = blockIdx.y;
  if (a.abort_flag[static_cast<size_t>(ctrl) * a.abort_stride] != 0) return;
  const int chunk = a.chunk0 + blockIdx.x * TPC + tile;
  // a tile past the rank's last chunk (last CTA only) runs without writing
  const bool active = TPC == 1 || chunk < a.chunk_end;  // (single-tile grids hold exactly the rank's chunks)
  const int k = chunk * kUmmaThreads + tid;
  const bool valid = active && k < a.K;
  double* s_red = s_red_all[tile];
  int& s_bad = s_bad_all[tile];
  const bool zm = k >= a.zero_start;
  const int kn = valid ? k : 0;

  float* s_plan = reinterpret_cast<float*>(smem_raw);
  unsigned char* s_w = smem_raw + ((sizeof(float) * (2 * T + 2) + 127) & ~size_t(127));
  using UL = UmmaLayout<H>;
  constexpr int NK = UL::NK;
  constexpr int SW = umma_sw_rcp<H>();
  unsigned char* s_tiles = s_w + UL::BYTES;
  s_tiles = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(s_tiles) + 127) & ~uintptr_t(127));
  s_tiles += static_cast<size_t>(tile) * umma_tile_region_bytes<H>();
  const uint32_t w_addr = static_cast<uint32_t>(__cvta_generic_to_shared(s_w));
  const uint32_t a1_hi = static_cast<uint32_t>(__cvta_generic_to_shared(s_tiles));
  const uint32_t a1_lo = a1_hi + kUmmaTileA;
  const uint32_t a2_hi = a1_lo + kUmmaTileA;        // NK K slices
  const uint32_t a2_lo = a2_hi + NK * kUmmaTileA;   // NK K slices
  const uint32_t mbar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar_all[tile]));

  for (int i = threadIdx.x; i < 2 * T + 2; i += kUmmaThreads * TPC)
    s_plan[i] = (i < 2 * T) ? a.plan[static_cast<size_t>(ctrl) * 2 * T + i] : 0.f;
  {
    const uint4* src = reinterpret_cast<const uint4*>(wimg);
    uint4* dst = reinterpret_cast<uint4*>(s_w);
    for (int i = threadIdx.x; i < static_cast<int>(UL::BYTES / 16); i += kUmmaThreads * TPC) dst[i] = src[i];
  }
  // the constant-one input (k = 6, the layer-1 bias column) and the zero K
  // half (k = 8 .. 15) of this thread's layer-1 rows, written once
  sts128(a1_hi + umma_tile_offset(tid, 8), 0u, 0u, 0u, 0u);
  sts128(a1_lo + umma_tile_offset(tid, 8), 0u, 0u, 0u, 0u);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&s_taddr))),
                 "n"(umma_tmem_cols<H, TPC>()));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  tc05_before_sync();
  __syncthreads();
  tc05_after_sync();
  const uint32_t taddr = s_taddr + static_cast<uint32_t>(2 * H * tile);  // this tile's accumulator columns
  const uint32_t t_lane = taddr + (static_cast<uint32_t>(32 * warp) << 16);  // this warp's TMEM lanes
  const uint32_t idH = umma_idesc(H), id16 = umma_idesc(16);
  const uint32_t one_h = h2_bits(__floats2half2_rn(1.f, 0.f));
  const float* s_b2 = reinterpret_cast<const float*>(s_w + UL::B2);
  const float* s_b3 = reinterpret_cast<const float*>(s_w + UL::B3);
  const float dt = a.sys.dt;
  const float dt3 = dt * *reinterpret_cast<const float*>(s_w + UL::SC);  // dt 2^-s (exact)
  const CostDev<float> cp = a.sys.cost;
  const float inv_s0 = 1.0f / a.sigma0, inv_s1 = 1.0f / a.sigma1;
  const float gml = a.gamma - a.lambda, half_lambda = 0.5f * a.lambda;
  uint32_t phase = 0;

  // noise and the coupling of step t (controller.cpp:86-101)
  NoiseStream<float, Mode> ns = make_noise<float, Mode>(a, ctrl, kn);
  const uint64_t seed = a.seeds[ctrl], iteration = a.iters[ctrl];
  float zc0 = 0.f, zc1 = 0.f;
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
  float v0c, v1c, coup_t;
  auto produce_v = [&](int t, bool even) {
    float e0, e1;
    eps_at(t, even, e0, e1);
    const float u0 = s_plan[2 * t], u1 = s_plan[2 * t + 1];
    e0 = zm ? e0 - u0 : e0;
    e1 = zm ? e1 - u1 : e1;
    const float v0 = u0 + e0, v1 = u1 + e1;
    const float uv = __fmul_rn(__fmul_rn(u0, v0), inv_s0) + __fmul_rn(__fmul_rn(u1, v1), inv_s1);
    const float uu = __fmul_rn(__fmul_rn(u0, u0), inv_s0) + __fmul_rn(__fmul_rn(u1, u1), inv_s1);
    coup_t = zm ? __fadd_rn(__fmul_rn(gml, uv), __fmul_rn(half_lambda, uu)) : __fmul_rn(a.gamma, uv);
    v0c = clamp_r(v0, a.sys.lo0, a.sys.hi0);
    v1c = clamp_r(v1, a.sys.lo1, a.sys.hi1);
  };

  cudaGridDependencySynchronize();  // x0 (written by the step graph's x0 fetch, whose programmatic dependent this is)
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
  const bool trace = TRACE && a.trace_states != nullptr && valid && k == a.trace_k;
  produce_v(0, true);
  auto stage_v = [&] {
    uint32_t h2, l2;
    split2(v0c, v1c, h2, l2);
    sts64(a1_hi + umma_tile_offset(tid, 4), h2, one_h);
    sts64(a1_lo + umma_tile_offset(tid, 4), l2, 0u);
  };
  stage_v();

  // one layer's MMAs by the elected thread: D_m = A_hi B_hi, D_c = A_hi B_lo + A_lo B_hi
  // (descriptors built once: A tiles and weight tiles never move)
  const uint64_t d_a1h = umma_desc(a1_hi), d_a1l = umma_desc(a1_lo);
  // (slice s of a tile sequence is its base descriptor + s * bytes / 16: the
  // start-address field holds addr >> 4 and never carries out of 14 bits)
  const uint64_t d_a2h = umma_desc(a2_hi), d_a2l = umma_desc(a2_lo);
  const uint64_t d_w1h = umma_desc(w_addr + UL::W1_HI), d_w1l = umma_desc(w_addr + UL::W1_LO);
  const uint64_t d_w2h = umma_desc(w_addr + UL::W2_HI), d_w2l = umma_desc(w_addr + UL::W2_LO);
  const uint64_t d_w3h = umma_desc(w_addr + UL::W3_HI), d_w3l = umma_desc(w_addr + UL::W3_LO);
  constexpr uint64_t kSliceA = kUmmaTileA >> 4, kSliceW2 = (32 * H) >> 4, kSliceW3 = 512 >> 4;
  auto sync_for_mma = [&] {
    proxy_fence_smem();
    tc05_before_sync();
    if constexpr (TPC == 1) __syncthreads();
    else umma_tile_bar(tile);
  };
  auto issue1 = [&] {
    sync_for_mma();
    if (tid == 0) {
      tc05_after_sync();
      umma_f16(taddr, d_a1h, d_w1h, idH, 0);
      umma_f16(taddr + H, d_a1h, d_w1l, idH, 0);
      umma_f16(taddr + H, d_a1l, d_w1h, idH, 1);
      umma_commit(mbar);
    }
  };
  auto issue23 = [&](uint64_t bh, uint64_t bl, uint64_t slice_w, uint32_t idesc) {
    sync_for_mma();
    if (tid == 0) {
      tc05_after_sync();
#pragma unroll
      for (int s = 0; s < NK; ++s) {
        const uint64_t ah = d_a2h + s * kSliceA, al = d_a2l + s * kSliceA;
        const uint64_t wh = bh + s * slice_w, wl = bl + s * slice_w;
        umma_f16(taddr, ah, wh, idesc, s > 0);
        umma_f16(taddr + H, ah, wl, idesc, s > 0);
        umma_f16(taddr + H, al, wh, idesc, 1);
      }
      umma_commit(mbar);
    }
  };
  auto wait_mma = [&] {
    mbar_wait(mbar, phase);
    phase ^= 1u;
    tc05_after_sync();
  };

  auto step = [&](int t, auto even_tag) {
    constexpr bool EVEN = decltype(even_tag)::value;
    // layer-1 state inputs (roll, vx, vy, thd) of this thread's row; the
    // control half (v0, v1, 1, 0) was staged during the previous step's layer 3
    {
      uint32_t h0, l0, h1, l1;
      split2(roll, vx, h0, l0);
      split2(vy, thd, h1, l1);
      sts64(a1_hi + umma_tile_offset(tid, 0), h0, h1);
      sts64(a1_lo + umma_tile_offset(tid, 0), l0, l1);
    }
    issue1();
    // side work while layer 1 runs: the pose of x_{t+1} (the Euler split reads
    // only the old state) and its costmap taps, the running cost of step t-1 on x_t
    float sn, cs;
    tc_sincos(th, sn, cs);
    px = add_rn(px, mul_rn(sub_rn(mul_rn(cs, vx), mul_rn(sn, vy)), dt));
    py = add_rn(py, mul_rn(add_rn(mul_rn(sn, vx), mul_rn(cs, vy)), dt));
    th = add_rn(th, mul_rn(thd, dt));
    const MapTaps<float> q_next = map_fetch(map, px, py);
    {
      const float h = map_interp(q);
      const float rc = tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[t > 0 ? t - 1 : 0], cp);
      cost += (t > 0) ? static_cast<Acc>(add_rn(rc, p_coup)) : 0.0;
      p_coup = coup_t;
    }
    wait_mma();
    umma_layer_to_a<H, SW, false>(t_lane, nullptr, a2_hi, a2_lo, tid);
    issue23(d_w2h, d_w2l, kSliceW2, idH);
    produce_v(t + 1, !EVEN);
    wait_mma();
    umma_layer_to_a<H, SW, true>(t_lane, s_b2, a2_hi, a2_lo, tid);  // (layer 2's MMAs have completed: the tiles are free)
    issue23(d_w3h, d_w3l, kSliceW3, id16);
    stage_v();  // v_{t+1} into the next step's layer-1 row (layer 1's tile is free)
    wait_mma();
    float om[4], oc[4];
    tmem_ld4(t_lane, om);
    tmem_ld4(t_lane + H, oc);
    tmem_wait_ld();
    float d[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) d[o] = __fadd_rn(__fadd_rn(om[o], oc[o]), s_b3[o]);
    // the dynamic block of the Euler split (layer 3 is 2^s-scaled: dt3 = dt 2^-s)
    roll = add_rn(roll, mul_rn(d[0], dt3));
    vx = add_rn(vx, mul_rn(d[1], dt3));
    vy = add_rn(vy, mul_rn(d[2], dt3));
    thd = add_rn(thd, mul_rn(d[3], dt3));
    q = q_next;
    p_roll = roll;
    p_vx = vx;
    p_vy = vy;
    if (TRACE && trace) {
      float* so = a.trace_states + (t + 1) * 7;
      so[0] = px; so[1] = py; so[2] = th; so[3] = roll; so[4] = vx; so[5] = vy; so[6] = thd;
    }
  };
  int t = 0;
#pragma unroll 1
  for (; t + 1 < T; t += 2) {
    step(t, std::true_type{});
    step(t + 1, std::false_type{});
  }
  if (t < T) step(t, std::true_type{});
  // ---- terminal cost and the chunk softmin partials (rho, eta, bad, numerators)
  {
    const float h = map_interp(q);
    cost += static_cast<Acc>(add_rn(tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[T - 1], cp), p_coup));
    if (a.sys.with_terminal) cost += static_cast<Acc>(tc_state_cost<STAB>(h, p_roll, p_vx, p_vy, a.sys.decay_pow[T], cp));
  }
  MPPI_DCHECK(!valid || k < a.K);
  if (valid) a.costs[static_cast<size_t>(ctrl) * a.K + k] = cost;
  if (tid == 0) s_bad = 0;
  tc05_before_sync();
  __syncthreads();
  if (threadIdx.x < 32)  // (the allocating warp frees every tile's columns)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_taddr), "n"(umma_tmem_cols<H, TPC>()));
  if (valid && !isfinite(cost)) s_bad = 1;
  // rho = min, eta = sum exp(-(S - rho) / lambda) over the chunk (warps in order)
  Acc m = warp_min(valid ? cost : Acc(INFINITY));
  if (lane == 0) s_red[warp] = m;
  __syncthreads();
  Acc rho = s_red[0];
#pragma unroll
  for (int w = 1; w < kUmmaThreads / 32; ++w) rho = (s_red[w] < rho) ? s_red[w] : rho;
  const Acc wk = valid ? exp(-(cost - rho) / a.dlambda) : 0.0;
  const Acc ew = warp_sum(wk);
  __syncthreads();
  if (lane == 0) s_red[warp] = ew;
  __syncthreads();
  Acc* out = a.partials + static_cast<size_t>(ctrl) * a.partials_ctrl_stride +
             static_cast<size_t>(chunk) * a.partial_stride;
  MPPI_DCHECK(!active || static_cast<long long>(chunk + 1) * a.partial_stride <= a.partials_ctrl_stride);
  if (tid == 0 && active) {
    Acc eta = s_red[0];
#pragma unroll
    for (int w = 1; w < kUmmaThreads / 32; ++w) eta = eta + s_red[w];
    out[0] = rho;
    out[1] = eta;
    out[2] = s_bad ? 1.0 : 0.0;
    out[3] = 0.0;
  }
  // numerators over the regenerated batch: blocks of kTcTB steps, products
  // staged [t][c][sample] in shared memory (aliasing the A tiles), then each
  // (t, c) summed over the 128 samples by four threads in fixed stripes
  // (samples q, q + 4, ...) and the four stripe sums added in order
  double* stage = reinterpret_cast<double*>(s_tiles);
  if constexpr (Mode != kPhilox) ns = make_noise<float, Mode>(a, ctrl, kn);
  for (int tb = 0; tb < T; tb += kTcTB) {
    __syncthreads();  // previous block consumed
#pragma unroll 2
    for (int j = 0; j < kTcTB; ++j) {
      const int tt = tb + j;
      float e0 = 0.f, e1 = 0.f;
      if (tt < T) {
        eps_at(tt, (tt & 1) == 0, e0, e1);
        e0 = zm ? e0 - s_plan[2 * tt] : e0;
        e1 = zm ? e1 - s_plan[2 * tt + 1] : e1;
      }
      stage[(2 * j) * kUmmaThreads + tid] = __dmul_rn(wk, static_cast<Acc>(e0));
      stage[(2 * j + 1) * kUmmaThreads + tid] = __dmul_rn(wk, static_cast<Acc>(e1));
    }
    __syncthreads();
    {
      const int e = tid >> 2, qs = tid & 3;  // element e (= 2 j + c) of this block, stripe qs
      Acc s = 0.0;
      const double* col = stage + static_cast<size_t>(e) * kUmmaThreads;
#pragma unroll 8
      for (int r = qs; r < kUmmaThreads; r += 4) s = __dadd_rn(s, col[r]);
      const Acc s1 = __shfl_xor_sync(0xffffffffu, s, 1);
      const Acc s2 = __shfl_xor_sync(0xffffffffu, s, 2);
      const Acc s3 = __shfl_xor_sync(0xffffffffu, s, 3);
      if (qs == 0 && active && tb + (e >> 1) < T) {
        // stripes 0, 1, 2, 3 of element e live in lanes 4e' .. 4e' + 3 of this warp
        out[kPartialHeader + 2 * tb + e] = __dadd_rn(__dadd_rn(s, s1), __dadd_rn(s2, s3));
      }
    }
  }
}

}  // namespace mppi_dev
