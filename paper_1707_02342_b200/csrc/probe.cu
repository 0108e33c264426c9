// probe.cu — pipe throughput microbenchmarks (the roofline denominators).
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

// Warp-level mma.sync m16n8k16 f16 x f16 -> f32 (the instruction of the
// tensor-core K1), independent accumulators per warp.
__global__ void __launch_bounds__(256) hmma_probe(float* out, uint32_t a0, uint32_t b0) {
  float d[kChains / 2][4];
#pragma unroll
  for (int i = 0; i < kChains / 2; ++i) d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0.f;
  const uint32_t a1 = a0 ^ threadIdx.x, b1 = b0 ^ threadIdx.x;
  for (int it = 0; it < kIters / 8; ++it) {
#pragma unroll
    for (int i = 0; i < kChains / 2; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
                   : "r"(a0), "r"(a1), "r"(a0), "r"(a1), "r"(b0), "r"(b1));
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains / 2; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

// MUFU ex2 (the SFU / XU pipe: the activation's exponential), independent chains.
__global__ void __launch_bounds__(256) mufu_probe(float* out, float x0) {
  float a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = x0 + 1e-3f * (threadIdx.x + i);
  for (int it = 0; it < kIters / 8; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += a[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

}  // namespace

// mma.sync f16 (TFLOP/s, 2 x 16 x 8 x 16 per instruction) and MUFU ex2
// (G lane-ops/s) throughput on `device`: the tensor and SFU ceilings of the
// tensor-core K1, reported beside the FP32 one.
extern "C" int mppi_gpu_pipe_peak_probe(int device, double* hmma_tflops_out, double* mufu_gops_out) {
  auto fail = [](const char* what, cudaError_t e) {
    mppi_host::last_error() = std::string(what) + ": " + cudaGetErrorString(e);
    return MPPI_ERR_CUDA;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail("cudaSetDevice", e);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  if ((e = cudaMalloc(&out, 1024 * sizeof(float))) != cudaSuccess) return fail("cudaMalloc", e);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256;
  const double warps = blocks * (threads / 32.0);
  const double hmma_flop = warps * (kIters / 8) * (kChains / 2) * 2.0 * 16 * 8 * 16;
  const double mufu_ops = static_cast<double>(blocks) * threads * (kIters / 8) * kChains;
  double best[2] = {0.0, 0.0};
  for (int variant = 0; variant < 2; ++variant) {
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(a);
      if (variant == 0) hmma_probe<<<blocks, threads>>>(out, 0x3c003c00u, 0x38003800u);
      else mufu_probe<<<blocks, threads>>>(out, -1.0f);
      cudaEventRecord(b);
      if ((e = cudaEventSynchronize(b)) != cudaSuccess) {
        cudaFree(out);
        return fail("probe kernel", e);
      }
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      const double v = (variant == 0 ? hmma_flop / 1e12 : mufu_ops / 1e9) / (ms * 1e-3);
      if (rep > 0 && ms > 0.f) best[variant] = std::max(best[variant], v);
    }
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  if (hmma_tflops_out) *hmma_tflops_out = best[0];
  if (mufu_gops_out) *mufu_gops_out = best[1];
  return MPPI_OK;
}

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
