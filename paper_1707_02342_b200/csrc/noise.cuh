// noise.cuh — counter-based Gaussian perturbations generated in registers.
//
// Two generators, both pure functions of (seed, iteration, k, t) so a kernel
// can regenerate any eps_k[t] instead of storing the K x T x 2 batch:
//  * the reference stream — splitmix64 chain + Box-Muller in double
//    (proj/include/mppi/sampler.hpp:15-54, sampler.cpp:21-31), bit-compatible
//    in the integer hash;
//  * Philox4x32-10 (production), one 128-bit draw per two timesteps.
#pragma once

#include "common.cuh"

namespace mppi_dev {

constexpr uint64_t kStreamPerturbations = 0x706572747572626full;  // sampler.hpp:57

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// The part of counter_hash (sampler.hpp:22-32) that depends only on
// (seed, iteration) is hoisted out of the per-sample loop by the callers.
__host__ __device__ __forceinline__ uint64_t ref_hash_prefix(uint64_t seed, uint64_t iteration) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ kStreamPerturbations);
  return splitmix64(h ^ iteration);
}
__device__ __forceinline__ void ref_normal_pair(uint64_t prefix, uint64_t k, uint64_t t,
                                                double& z0, double& z1) {
  uint64_t h = splitmix64(prefix ^ k);
  h = splitmix64(h ^ t);
  h = splitmix64(h ^ 0ull);  // pair index 0: m = 2 has one Box-Muller pair per (k, t)
  const double u1 = static_cast<double>((h >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(splitmix64(h) >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double phi = (2.0 * 3.14159265358979323846) * u2;
  double s, c;
  sincos(phi, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// Philox4x32-10 (Salmon et al., SC'11).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// Box-Muller of one Philox half-draw: u1 = ((a>>8)+1) 2^-24 in (0,1],
// u2 = (b>>8) 2^-24 in [0,1) (both exact in fp32).
//
// fp32 (the production noise of the fp32 kernels) on the SFU, branch-free:
//  * -ln(u1): MUFU.LG2 * ln 2, except within 2^-6 of 1 where its absolute
//    error (~2^-22) would dominate the small result; there the series
//    x + x^2/2 + x^3/3 + x^4/4 of x = 1 - u1 (exact) is used;
//  * r = sqrt.approx(2 (-ln u1));
//  * (cos, sin)(2 pi u2) = -(cos, sin)(2 pi u2 - pi): MUFU.SIN/COS on [-pi, pi)
//    (abs. error ~2^-21).
// Every draw stays within ~1e-6 of the double-precision Box-Muller of the same
// integers (the oracle's definition, checked by the Philox parity test).
__device__ __forceinline__ void philox_box_muller(uint32_t a, uint32_t b, float& z0, float& z1) {
  const float u1 = static_cast<float>((a >> 8) + 1u) * 0x1.0p-24f;
  const float u2 = static_cast<float>(b >> 8) * 0x1.0p-24f;
  const float x = 1.0f - u1;  // exact: u1 is a multiple of 2^-24 in (0, 1]
  const float series = x * __fmaf_rn(x, __fmaf_rn(x, __fmaf_rn(x, 0.25f, 0.33333334f), 0.5f), 1.0f);
  float lg;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(u1));
  const float nlog = (x < 0.015625f) ? series : -0.69314718f * lg;
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(2.0f * nlog));
  const float phi = __fmaf_rn(u2, 6.28318531f, -3.14159265f);
  float s, c;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(phi));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(phi));
  z0 = -r * c;
  z1 = -r * s;
}
__device__ __forceinline__ void philox_box_muller(uint32_t a, uint32_t b, double& z0, double& z1) {
  const double u1 = static_cast<double>((a >> 8) + 1u) * 0x1.0p-24;
  const double u2 = static_cast<double>(b >> 8) * 0x1.0p-24;
  const double r = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// Philox counter layout: ctr = (t/2, k, iter_lo, iter_hi), key = seed; lanes
// (x, y) of the draw feed even t, (z, w) odd t.
__device__ __forceinline__ uint4 philox_draw(uint64_t seed, uint64_t iteration, uint32_t k,
                                             uint32_t t_pair) {
  return philox4x32_10(make_uint4(t_pair, k, static_cast<uint32_t>(iteration),
                                  static_cast<uint32_t>(iteration >> 32)),
                       static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

enum NoiseMode { kInjected = 0, kRefSplitmix = 1, kPhilox = 2 };

// Per-thread noise source for one sample k of one controller.  eps(t) must be
// called with t = 0, 1, 2, ... in order (Philox caches the odd half-draw).
template <class R, int Mode>
struct NoiseStream {
  // all modes: sqrt(sigma_c) rounded to R, and in double for the reference stream
  R scale0, scale1;
  double dscale0, dscale1;
  // injected: device layout [T][K][2]
  const R* inj;
  int K;
  uint32_t k;
  // ref splitmix
  uint64_t prefix;
  // philox
  uint64_t seed, iteration;
  R z2, z3;  // odd-step half of the current Philox draw

  __device__ __forceinline__ void eps(int t, R& e0, R& e1) {
    if constexpr (Mode == kInjected) {
      const R* p = inj + (static_cast<size_t>(t) * K + k) * 2;
      e0 = p[0];
      e1 = p[1];
    } else if constexpr (Mode == kRefSplitmix) {
      double z0, z1;
      ref_normal_pair(prefix, k, static_cast<uint64_t>(t), z0, z1);
      // eps(t,c) = sqrt(sigma_c) * z in double, rounded once (sampler.cpp:33-34)
      e0 = static_cast<R>(dscale0 * z0);
      e1 = static_cast<R>(dscale1 * z1);
    } else {
      if ((t & 1) == 0) {
        const uint4 d = philox_draw(seed, iteration, k, static_cast<uint32_t>(t) >> 1);
        R z0, z1;
        philox_box_muller(d.x, d.y, z0, z1);
        philox_box_muller(d.z, d.w, z2, z3);
        e0 = scale0 * z0;
        e1 = scale1 * z1;
      } else {
        e0 = scale0 * z2;
        e1 = scale1 * z3;
      }
    }
  }
};

}  // namespace mppi_dev
