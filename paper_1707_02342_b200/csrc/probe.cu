// probe.cu — FP32 FMA throughput microbenchmark (the roofline denominator).
//
// MEASURED_PEAKS.json holds HBM and bf16 tensor peaks only; the rollout is
// bound by the CUDA-core FP32 pipe, so its peak is measured here on the box:
// independent FMA chains in registers, one variant with scalar FFMA and one
// with Blackwell's paired FFMA2 (fma.rn.f32x2), full-chip grid.  The best
// variant is the denominator reported by bench.py.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/mppi_gpu.h"
#include "host_util.hpp"

namespace {

constexpr int kChains = 16;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) ffma_probe(float* out, float b, float c) {
  float a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = static_cast<float>(threadIdx.x + i);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = __fmaf_rn(a[i], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 1234.5f) out[threadIdx.x] = s;  // never true; keeps the chains live
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void __launch_bounds__(256) ffma2_probe(float* out, float b, float c) {
  unsigned long long a[kChains / 2];
  const float2 bb = make_float2(b, b), cc = make_float2(c, c);
  const unsigned long long B = *reinterpret_cast<const unsigned long long*>(&bb);
  const unsigned long long Cc = *reinterpret_cast<const unsigned long long*>(&cc);
#pragma unroll
  for (int i = 0; i < kChains / 2; ++i) {
    const float2 v = make_float2(static_cast<float>(threadIdx.x + i), static_cast<float>(i));
    a[i] = *reinterpret_cast<const unsigned long long*>(&v);
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains / 2; ++i) a[i] = ffma2(a[i], B, Cc);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains / 2; ++i) {
    const float2 v = *reinterpret_cast<const float2*>(&a[i]);
    s += v.x + v.y;
  }
  if (s == 1234.5f) out[threadIdx.x] = s;
}

}  // namespace

extern "C" int mppi_gpu_fp32_peak_probe(int device, double* tflops_out, double* sm_clock_mhz_out) {
  auto fail = [](const char* what, cudaError_t e) {
    mppi_host::last_error() = std::string(what) + ": " + cudaGetErrorString(e);
    return MPPI_ERR_CUDA;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail("cudaSetDevice", e);
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, device);
  float* out = nullptr;
  if ((e = cudaMalloc(&out, 1024 * sizeof(float))) != cudaSuccess) return fail("cudaMalloc", e);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256;
  const double flops = 2.0 * kChains * static_cast<double>(kIters) * blocks * threads;
  double best = 0.0;
  for (int variant = 0; variant < 2; ++variant) {
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(a);
      if (variant == 0) ffma_probe<<<blocks, threads>>>(out, 0.999f, 0.001f);
      else ffma2_probe<<<blocks, threads>>>(out, 0.999f, 0.001f);
      cudaEventRecord(b);
      if ((e = cudaEventSynchronize(b)) != cudaSuccess) {
        cudaFree(out);
        return fail("probe kernel", e);
      }
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms > 0.f) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  if (tflops_out) *tflops_out = best;
  if (sm_clock_mhz_out) *sm_clock_mhz_out = clk_khz / 1000.0;
  return MPPI_OK;
}
