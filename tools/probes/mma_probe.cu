// Microbenchmark (design input for the tensor-core rollout): throughput and
// latency of legacy warp-level mma.sync on sm_100a (tf32 m16n8k8, bf16
// m16n8k16), FFMA2 and MUFU ex2, measured with clock64 / cudaEvents.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int CHAINS, bool BF16>
__global__ void mma_tput(float* out, int iters, long long* cyc) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
  float d[CHAINS][4] = {};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (BF16) mma_bf16(d[c], a, b);
      else mma_tf32(d[c], a, b);
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void ffma2_tput(float* out, int iters, long long* cyc) {
  float2 acc[8];
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x, i);
  const float2 w = make_float2(1.0001f, 0.9999f), x = make_float2(1e-3f, 2e-3f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = __ffma2_rn(acc[i], w, x);
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void ex2_tput(float* out, int iters, long long* cyc) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-4f + i * 1e-3f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <class F>
void run(const char* name, F launch, int blocks, int threads, int iters, double ops_per_thread_iter) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long));
  launch(out, 10, cyc, blocks, threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launch(out, iters, cyc, blocks, threads);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double ops = ops_per_thread_iter * iters * double(blocks) * threads;
  std::printf("%-28s blocks=%4d thr=%4d  %8.3f ms  %9.2f Tops/s  cycles/iter(block0)=%.2f  %s\n", name, blocks, threads, ms,
              ops / (ms * 1e-3) / 1e12, double(c) / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::printf("SMs %d\n", sms);
  const int it = 20000;
  // tf32 m16n8k8: 2*16*8*8 = 2048 flop per warp-mma -> 64 flop per thread
  for (int w : {1, 4, 8, 16}) {
    run("tf32 mma x8 chains", [](float* o, int n, long long* c, int b, int t) { mma_tput<8, false><<<b, t>>>(o, n, c); },
        sms, 32 * w, it, 8 * 64);
  }
  run("tf32 mma 1 chain (latency)", [](float* o, int n, long long* c, int b, int t) { mma_tput<1, false><<<b, t>>>(o, n, c); },
      sms, 32, it, 64);
  run("tf32 mma 4 chains", [](float* o, int n, long long* c, int b, int t) { mma_tput<4, false><<<b, t>>>(o, n, c); },
      sms, 32, it, 4 * 64);
  for (int w : {1, 4, 16}) {
    run("bf16 mma x8 chains", [](float* o, int n, long long* c, int b, int t) { mma_tput<8, true><<<b, t>>>(o, n, c); },
        sms, 32 * w, it, 8 * 128);
  }
  run("bf16 mma 1 chain (latency)", [](float* o, int n, long long* c, int b, int t) { mma_tput<1, true><<<b, t>>>(o, n, c); },
      sms, 32, it, 128);
  for (int w : {4, 16}) {
    run("ffma2 x8", [](float* o, int n, long long* c, int b, int t) { ffma2_tput<<<b, t>>>(o, n, c); }, sms, 32 * w, it,
        8 * 4);
  }
  for (int w : {4, 16}) {
    run("ex2 x8 (ops = ex2/s)", [](float* o, int n, long long* c, int b, int t) { ex2_tput<<<b, t>>>(o, n, c); }, sms,
        32 * w, it, 8);
  }
  return 0;
}
