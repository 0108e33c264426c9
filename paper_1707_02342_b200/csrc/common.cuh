// common.cuh — shared device helpers for the B200 IT-MPPI kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include <type_traits>

namespace mppi_dev {

// Device-side invariant checks of a debug build (-DMPPI_DEVICE_CHECKS): every
// global write of the hot path checks its index against the buffer it owns
// and traps otherwise (compute-sanitizer is not available on the GPU pool;
// tools/gpu_device_checks.sh runs the GPU tests on this build).
#ifdef MPPI_DEVICE_CHECKS
#define MPPI_DCHECK(cond)                                                                         \
  do {                                                                                            \
    if (!(cond)) {                                                                                \
      printf("MPPI_DCHECK failed %s:%d block (%d,%d,%d) thread %d: %s\n", __FILE__, __LINE__,     \
             blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x, #cond);                             \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define MPPI_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

// Rounded (never contracted) arithmetic.  The state update and the cost use
// these so the fp32/fp64 device paths perform the same operation sequence as
// the oracle restatement (oracle/mppi_oracle.cpp, built with
// -ffp-contract=off); only the MLP uses explicit fused multiply-adds, in both.
template <class R> __device__ __forceinline__ R mul_rn(R a, R b);
template <class R> __device__ __forceinline__ R add_rn(R a, R b);
template <class R> __device__ __forceinline__ R sub_rn(R a, R b);
template <> __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
template <> __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ float fma_r(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_r(double a, double b, double c) { return __fma_rn(a, b, c); }

__device__ __forceinline__ float div_r(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_r(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ float tanh_r(float x) { return tanhf(x); }
__device__ __forceinline__ double tanh_r(double x) { return tanh(x); }
__device__ __forceinline__ float exp_r(float x) { return expf(x); }
__device__ __forceinline__ double exp_r(double x) { return exp(x); }
__device__ __forceinline__ float sqrt_r(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ double sqrt_r(double x) { return __dsqrt_rn(x); }
__device__ __forceinline__ float atan_r(float x) { return atanf(x); }
__device__ __forceinline__ double atan_r(double x) { return atan(x); }
__device__ __forceinline__ float tan_r(float x) { return tanf(x); }
__device__ __forceinline__ double tan_r(double x) { return tan(x); }
__device__ __forceinline__ float sin_r(float x) { return sinf(x); }
__device__ __forceinline__ double sin_r(double x) { return sin(x); }
__device__ __forceinline__ float abs_r(float x) { return fabsf(x); }
__device__ __forceinline__ double abs_r(double x) { return fabs(x); }
__device__ __forceinline__ void sincos_r(float x, float* s, float* c) { sincosf(x, s, c); }
__device__ __forceinline__ void sincos_r(double x, double* s, double* c) { sincos(x, s, c); }
__device__ __forceinline__ bool isfinite_r(float x) { return isfinite(x); }
__device__ __forceinline__ bool isfinite_r(double x) { return isfinite(x); }

// std::clamp semantics (dynamics.cpp:13-16): NaN passes through unchanged —
// fminf/fmaxf would silently replace it, so comparisons are explicit.
template <class R>
__device__ __forceinline__ R clamp_r(R v, R lo, R hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}

// Timeline stamps of a profiling build (-DMPPI_STAMPS): %globaltimer at the
// phase boundaries of one iteration (K1 end, group merge, tail phases),
// printed by the tail.  Slot i holds the max (ends) or min (starts) over CTAs.
#ifdef MPPI_STAMPS
__device__ unsigned long long g_stamps[16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define MPPI_STAMP_MAX(i) atomicMax(&::mppi_dev::g_stamps[i], ::mppi_dev::gtimer())
#define MPPI_STAMP_MIN(i) atomicMin(&::mppi_dev::g_stamps[i], ::mppi_dev::gtimer())
#else
#define MPPI_STAMP_MAX(i) \
  do {                    \
  } while (0)
#define MPPI_STAMP_MIN(i) \
  do {                    \
  } while (0)
#endif

template <class R>
__device__ __forceinline__ R warp_sum(R v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <class R>
__device__ __forceinline__ R warp_min(R v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const R w = __shfl_xor_sync(0xffffffffu, v, o);
    v = (w < v) ? w : v;
  }
  return v;
}

}  // namespace mppi_dev
