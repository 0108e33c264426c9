// handle.cuh — the controller handle for one arithmetic type R: device
// buffers, launch plumbing, captured CUDA graphs and the NCCL sample-shard
// exchange.  Instantiated once per precision (handle_f32.cu, handle_f64.cu).
//
// The host side of the drop-in boundary.  It owns all device memory of one
// control loop (or fleet), one CUDA stream, the captured CUDA graphs of the
// iteration, and (multi-GPU) the NCCL communicator of its sample shard.  No
// CPU fallback exists: every compute entry point launches device kernels and
// fails with MPPI_ERR_CUDA when no device is usable.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "epilogue.cuh"
#include "group.cuh"
#include "rollout_tc.cuh"
#include "rollout_umma.cuh"
#include "cem.cuh"
#include "ws_launch.hpp"
#include "errors.hpp"
#include "handle_iface.hpp"
#include "host_util.hpp"
#include "nccl_api.hpp"

namespace mppi_host {

using namespace mppi_dev;

// -------------------------------------------------------- device buffers ----
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    if (count == 0) return;
    CUDA_TRY(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
};
template <class T>
struct HostPinned {
  T* p = nullptr;
  size_t n = 0;
  ~HostPinned() {
    if (p) cudaFreeHost(p);
  }
  void alloc(size_t count) {
    if (count <= n && p) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    CUDA_TRY(cudaMallocHost(&p, count * sizeof(T)));
    n = count;
  }
};

constexpr int kBlock = 128;      // samples per chunk / K1 CTA

// Per-lane mma.sync fragment table of the tensor-core rollout
// (rollout_tc.cuh, word map there): weights folded with the tanh identity
// tanh(z) = 1 + 2s, s = -1 / (1 + 2^(kz)), k = 2 log2 e, then split hi/lo in fp16.
template <class R, int H>
std::vector<uint32_t> tc_build_fragments(const MlpParams<R, H>& w) {
  using L = mppi_dev::TcLayout<H>;
  const double kk2 = 2.0 / std::log(2.0);
  auto W1 = [&](int n, int i) { return static_cast<double>(w.w1t[i][n]); };
  auto W2 = [&](int n, int i) { return static_cast<double>(w.w2t[i][n]); };
  auto W3 = [&](int n, int i) { return static_cast<double>(w.w3t[i][n]); };
  auto B1 = [&](int kin, int n) -> double {  // k8 x n32
    if (kin < 6) return kk2 * W1(n, kin);
    if (kin == 6) return kk2 * static_cast<double>(w.b1[n]);
    return 0.0;
  };
  // the layer inputs are s = -1/(1 + 2^(kz)) = (tanh z - 1) / 2
  auto B2 = [&](int i, int n) -> double { return 2.0 * kk2 * W2(n, i); };
  // layer 3 on 2^s-scaled weights, max |2 W3| 2^s in [0.5, 1) (TcLayout: keeps
  // the lo halves of the fp16 split out of the subnormal range)
  double w3max = 0.0;
  for (int n = 0; n < 4; ++n)
    for (int i = 0; i < H; ++i) w3max = std::max(w3max, std::abs(2.0 * W3(n, i)));
  int s3 = 0;
  while (s3 < 12 && w3max > 0.0 && w3max * std::ldexp(1.0, s3 + 1) < 1.0) ++s3;
  if (const char* e = std::getenv("MPPI_TC_W3_SHIFT")) s3 = std::max(0, std::min(12, std::atoi(e)));  // A/B only
  const double sc3 = std::ldexp(1.0, s3);
  auto B3 = [&](int i, int n) -> double { return n < 4 ? sc3 * 2.0 * W3(n, i) : 0.0; };
  auto hl = [](double x, int which) -> uint16_t {
    const __half h = __double2half(x);
    if (which == 0) return __half_as_ushort(h);
    return __half_as_ushort(__double2half(x - static_cast<double>(__half2float(h))));
  };
  auto pack = [&](double lo_k, double hi_k, int which) -> uint32_t {
    return static_cast<uint32_t>(hl(lo_k, which)) | (static_cast<uint32_t>(hl(hi_k, which)) << 16);
  };
  std::vector<uint32_t> f(static_cast<size_t>(L::WORDS) * 32, 0u);
  auto put = [&](int word, int lane, uint32_t v) { f[static_cast<size_t>(word) * 32 + lane] = v; };
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    for (int j = 0; j < L::NJ; ++j)
      for (int which = 0; which < 2; ++which)
        put(L::W1 + 2 * j + which, lane, pack(B1(2 * t, 8 * j + g), B1(2 * t + 1, 8 * j + g), which));
    for (int kk = 0; kk < L::NK; ++kk)
      for (int j = 0; j < L::NJ; ++j)
        for (int r = 0; r < 2; ++r)
          for (int which = 0; which < 2; ++which) {
            const int i0 = 16 * kk + 2 * t + 8 * r;
            put(L::W2 + ((kk * L::NJ + j) * 2 + r) * 2 + which, lane,
                pack(B2(i0, 8 * j + g), B2(i0 + 1, 8 * j + g), which));
          }
    for (int kk = 0; kk < L::NK; ++kk)
      for (int r = 0; r < 2; ++r)
        for (int which = 0; which < 2; ++which) {
          const int i0 = 16 * kk + 2 * t + 8 * r;
          put(L::W3 + (kk * 2 + r) * 2 + which, lane, pack(B3(i0, g), B3(i0 + 1, g), which));
        }
    for (int j = 0; j < L::NJ; ++j)
      for (int c = 0; c < 2; ++c) {
        const int n = 8 * j + 2 * t + c;
        double sum = 0.0;
        for (int i = 0; i < H; ++i) sum += W2(n, i);
        const float v = static_cast<float>(kk2 * (static_cast<double>(w.b2[n]) + sum));
        uint32_t bits;
        std::memcpy(&bits, &v, 4);
        put(L::B2 + 2 * j + c, lane, bits);
      }
    for (int c = 0; c < 2; ++c) {
      const int n = 2 * t + c;
      float v = 0.f;
      if (n < 4) {
        double sum = 0.0;
        for (int i = 0; i < H; ++i) sum += W3(n, i);
        v = static_cast<float>(sc3 * (static_cast<double>(w.b3[n]) + sum));
      }
      uint32_t bits;
      std::memcpy(&bits, &v, 4);
      put(L::B3 + c, lane, bits);
    }
    {
      const float inv = static_cast<float>(std::ldexp(1.0, -s3));
      uint32_t bits;
      std::memcpy(&bits, &inv, 4);
      put(L::SC, lane, bits);
    }
  }
  return f;
}
// The weight image of the tcgen05 rollout (rollout_umma.cuh, UmmaLayout): the
// same folded weights as tc_build_fragments (layer 3 on 2^s-scaled weights),
// as fp16 hi / lo B tiles in the canonical K-major layout, plus the layer-2/3
// bias vectors (added after the accumulator read-back) and 2^-s.
template <class R, int H>
std::vector<unsigned char> umma_build_image(const MlpParams<R, H>& w) {
  using U = mppi_dev::UmmaLayout<H>;
  const double kk2 = 2.0 / std::log(2.0);
  auto W1 = [&](int n, int i) { return static_cast<double>(w.w1t[i][n]); };
  auto W2 = [&](int n, int i) { return static_cast<double>(w.w2t[i][n]); };
  auto W3 = [&](int n, int i) { return static_cast<double>(w.w3t[i][n]); };
  double w3max = 0.0;
  for (int n = 0; n < 4; ++n)
    for (int i = 0; i < H; ++i) w3max = std::max(w3max, std::abs(2.0 * W3(n, i)));
  int s3 = 0;
  while (s3 < 12 && w3max > 0.0 && w3max * std::ldexp(1.0, s3 + 1) < 1.0) ++s3;
  if (const char* e = std::getenv("MPPI_TC_W3_SHIFT")) s3 = std::max(0, std::min(12, std::atoi(e)));
  const double sc3 = std::ldexp(1.0, s3);
  std::vector<unsigned char> img(U::BYTES, 0);
  auto put_half = [&](uint32_t base, int row, int k, double v, bool lo) {
    const __half h = __double2half(v);
    const __half x = lo ? __double2half(v - static_cast<double>(__half2float(h))) : h;
    const uint16_t bits = __half_as_ushort(x);
    std::memcpy(&img[base + mppi_dev::umma_tile_offset(row, k)], &bits, 2);
  };
  for (int lo = 0; lo < 2; ++lo) {
    for (int n = 0; n < H; ++n)
      for (int k = 0; k < 16; ++k) {
        const double v = k < 6 ? kk2 * W1(n, k) : (k == 6 ? kk2 * static_cast<double>(w.b1[n]) : 0.0);
        put_half(lo ? U::W1_LO : U::W1_HI, n, k, v, lo != 0);
      }
    for (int s = 0; s < U::NK; ++s)
      for (int n = 0; n < H; ++n)
        for (int k = 0; k < 16; ++k)
          put_half((lo ? U::W2_LO : U::W2_HI) + 32 * H * s, n, k, 2.0 * kk2 * W2(n, 16 * s + k), lo != 0);
    for (int s = 0; s < U::NK; ++s)
      for (int n = 0; n < 16; ++n)
        for (int k = 0; k < 16; ++k)
          put_half((lo ? U::W3_LO : U::W3_HI) + 512 * s, n, k, n < 4 ? sc3 * 2.0 * W3(n, 16 * s + k) : 0.0,
                   lo != 0);
  }
  for (int n = 0; n < H; ++n) {
    double sum = 0.0;
    for (int i = 0; i < H; ++i) sum += W2(n, i);
    const float v = static_cast<float>(kk2 * (static_cast<double>(w.b2[n]) + sum));
    std::memcpy(&img[U::B2 + 4 * n], &v, 4);
  }
  for (int o = 0; o < 4; ++o) {
    double sum = 0.0;
    for (int i = 0; i < H; ++i) sum += W3(o, i);
    const float v = static_cast<float>(sc3 * (static_cast<double>(w.b3[o]) + sum));
    std::memcpy(&img[U::B3 + 4 * o], &v, 4);
  }
  const float inv = static_cast<float>(std::ldexp(1.0, -s3));
  std::memcpy(&img[U::SC], &inv, 4);
  return img;
}

constexpr int kEpiBlock = 512;   // K2 CTA

template <class R>
struct Handle final : HandleBase {
  // ---- HandleBase adaptors
  int device_index() const override { return device; }
  int controllers() const override { return C; }
  const mppi_gpu_config& config() const override { return cfg; }
  void set_map_f64(int c, const double* v, int w, int h, double x0, double y0, double res) override {
    set_map(c, v, w, h, x0, y0, res);
  }
  void set_map_f32(int c, const float* v, int w, int h, double x0, double y0, double res) override {
    set_map(c, v, w, h, x0, y0, res);
  }
  void* stream_ptr() const override { return reinterpret_cast<void*>(stream); }
  uint64_t launch_count() const override { return launches; }
  void set_profile(bool on) override { profile = on; }
  void read_profile(double* ms, uint64_t* n, bool reset) override {
    if (ms) *ms = prof_ms;
    if (n) *n = prof_launches;
    if (reset) {
      prof_ms = 0;
      prof_launches = 0;
    }
  }
  std::string variant_name() const override {
    char buf[256];
    if (use_umma)
      std::snprintf(buf, sizeof(buf), "rollout_umma_kernel<f32,H=%d,noise=%d> (tcgen05.mma f16x3 M=128, TMEM accumulators, chunk 128, %d chunks, %d groups, group merge + tail kernels)",
                    H, cfg.noise_mode, n_chunks, n_groups);
    else if (use_tc && tc_pair_used == 2)
      std::snprintf(buf, sizeof(buf), "rollout_tc_split_kernel<f32,H=%d,noise=%d> (mma.sync f16x3, 8 samples per warp on the n dimension, chunk 16 per warp pair, %d chunks, %d groups, group merge + tail kernels)",
                    H, cfg.noise_mode, n_chunks, n_groups);
    else if (use_tc && tc_pair_used == 1)
      std::snprintf(buf, sizeof(buf), "rollout_tc_pair_kernel<f32,H=%d,noise=%d> (mma.sync f16x3, chunk 16 per warp pair, %d chunks, %d groups, group merge + tail kernels)",
                    H, cfg.noise_mode, n_chunks, n_groups);
    else if (use_tc)
      std::snprintf(buf, sizeof(buf), "rollout_tc_kernel<f32,H=%d,MT=%d,noise=%d> (mma.sync f16x3, chunk %d, %d chunks, %d groups, group merge + tail kernels)",
                    H, tc_mt, cfg.noise_mode, chunk_samples, n_chunks, n_groups);
    else if (use_ws)
      std::snprintf(buf, sizeof(buf), "rollout_ws_kernel<f32,H=%d,L=%d,noise=%d,%s> (chunk 32, %d chunks, %d groups)", H, ws_L,
                    cfg.noise_mode, ws_smem_w ? "smem-weights" : "const-weights", n_chunks, n_groups);
    else
      std::snprintf(buf, sizeof(buf), "rollout_kernel<%s,H=%d,%s,noise=%d,block=%d>",
                    std::is_same<R, double>::value ? "f64" : "f32", H,
                    cfg.system == MPPI_SYSTEM_QUADRATIC ? "quadratic"
                    : (cfg.system == MPPI_SYSTEM_VEHICLE_BASIS     ? "vehicle_basis"
                       : cfg.system == MPPI_SYSTEM_VEHICLE_BICYCLE ? "vehicle_bicycle"
                                                                   : "vehicle_mlp"),
                    cfg.noise_mode, kBlock);
    return buf;
  }

  mppi_gpu_config cfg{};
  int K = 0, T = 0, C = 1, H = 32, device = 0;
  // chunks of chunk_samples samples; fixed groups of chunks (group.cuh), the
  // unit of the multi-rank exchange; this rank's groups [group_lo, group_hi)
  // = chunks [chunk_lo, chunk_hi)
  int n_chunks = 0, chunk_lo = 0, chunk_hi = 0;
  int n_groups = 0, group_lo = 0, group_hi = 0;
  // K1 variant: warp-specialised fp32 kernel (chunk = 32 samples, L warps per
  // chunk) for the vehicle model, generic one-sample-per-thread kernel
  // (chunk = kBlock) otherwise.
  bool use_ws = false;
  int ws_L = 1, chunk_samples = kBlock;
  bool ws_smem_w = true;  // weights staged in shared memory (vs constant bank)
  // tensor-core K1 (rollout_tc.cuh): fp32 vehicle model, H = 32; chunk = 16*tc_mt
  bool use_tc = false;
  bool use_umma = false;  // K1 on tcgen05 / TMEM (rollout_umma.cuh); the tensor-core tail as use_tc
  DevBuf<unsigned char> d_umma;
  int tc_mt = 2;
  int tc_pair_used = -1;  // whether this handle's last K1 launch was the warp-pair kernel (-1: none yet)
  DevBuf<uint32_t> d_tcfrag;
  // tensor-core tail (tail.cuh): merge of the group rows + epilogue, one CTA per controller
  DevBuf<unsigned char> d_plantw;  // MlpParams<float, H> (the plant step of the tail)
  int graph_kernels[4] = {0, 0, 0, 0};
  bool graph_direct[4] = {false, false, false, false};  // the graph's tail publishes the host status itself
  bool status_direct = false;      // capture in progress: the tail writes h_status itself
  bool k1_pdl = false;             // capture in progress: K1 follows the x0 fetch kernel (PDL)
  // sample sharding: NCCL all-gather of the group rows, or (in one process)
  // peer copies from the other handles of a local group
  enum { kExNone = 0, kExNccl = 1, kExLocal = 2 };
  int rank = 0, world = 1, exchange_mode = kExNone;
  std::vector<Handle<R>*> local_peers;
  int zero_start = 0;
  int partial_stride = 0;
  long long partials_ctrl_stride = 0;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  std::vector<double> sg;
  uint64_t launches = 0;

  // weights (host copies; by-value kernel parameters) + device copy for the
  // by-pointer variant
  ThetaDev<R> theta_r{};  // VEHICLE_BASIS coefficients
  BicycleDev<R> bike_r{};  // VEHICLE_BICYCLE parameters
  std::unique_ptr<MlpParams<R, 32>> w32;
  std::unique_ptr<MlpParams<R, 64>> w64;
  DevBuf<MlpParams<R, 64>> d_w64;
  bool has_mlp = false, has_map = false, has_noise = false;

  // device state
  DevBuf<R> d_plan, d_x0, d_inj, d_decay;
  DevBuf<Acc> d_costs, d_partials, d_groups, d_agg, d_w, d_rho_eta;
  DevBuf<R> d_states, d_utrace, d_xtrace;
  DevBuf<double> d_eps_ref;
  DevBuf<uint64_t> d_iters, d_seeds, d_trace_base;
  DevBuf<int> d_abort, d_bad;
  DevBuf<StepStatus> d_status;
  DevBuf<const R*> d_map_ptrs;
  DevBuf<R> d_map_shared;
  std::vector<std::unique_ptr<DevBuf<R>>> d_map_fleet;
  DevBuf<unsigned char> d_flush;
  int map_w = 0, map_h = 0;
  double map_x0 = 0, map_y0 = 0, map_res = 1;
  HostPinned<R> h_x0;
  HostPinned<StepStatus> h_status;
  std::vector<unsigned long long> seq_want;
  std::vector<uint64_t> h_iters;

  // last parity batch (for update_plan / rollout_states)
  bool batch_valid = false, batch_injected = false;
  uint64_t batch_iteration = 0;

  // profiling
  bool profile = false;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_it0 = nullptr, ev_it1 = nullptr, ev_x0 = nullptr, ev_x1 = nullptr;
  double prof_ms = 0, prof_x_ms = 0;
  uint64_t prof_launches = 0, prof_x_n = 0;

  // graphs: 0 = step (compute+slide), 1 = compute only, 2 = closed-loop iteration
  cudaGraphExec_t graph[4] = {nullptr, nullptr, nullptr, nullptr};
  uint64_t n_before_capture = 0;
  bool graph_trace[4] = {false, false, false, false};

  explicit Handle(const mppi_gpu_config& c) : cfg(c) {
    validate_config(c);
    K = c.samples;
    T = c.horizon_steps;
    C = c.n_controllers;
    H = c.mlp_hidden;
    device = c.device;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw Error(MPPI_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    }
    if (device < 0 || device >= ndev) throw_invalid("config.device out of range");
    CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreate(&ev_a));
    CUDA_TRY(cudaEventCreate(&ev_b));
    CUDA_TRY(cudaEventCreate(&ev_it0));
    CUDA_TRY(cudaEventCreate(&ev_it1));
    CUDA_TRY(cudaEventCreate(&ev_x0));
    CUDA_TRY(cudaEventCreate(&ev_x1));
    choose_variant();
    n_chunks = (K + chunk_samples - 1) / chunk_samples;
    chunk_lo = 0;
    chunk_hi = n_chunks;
    n_groups = group_count(n_chunks);
    group_lo = 0;
    group_hi = n_groups;
    zero_start = K - static_cast<int>(std::lround(c.explore_fraction * K));
    partial_stride = kPartialHeader + 2 * T;
    partials_ctrl_stride = static_cast<long long>(n_chunks) * partial_stride;
    if (c.sg_window != 0) sg = mppi_host::sg_coefficients(c.sg_window, c.sg_degree);

    d_plan.alloc(static_cast<size_t>(C) * 2 * T);
    CUDA_TRY(cudaMemset(d_plan.p, 0, d_plan.n * sizeof(R)));
    d_x0.alloc(static_cast<size_t>(C) * 8);
    CUDA_TRY(cudaMemset(d_x0.p, 0, d_x0.n * sizeof(R)));
    d_costs.alloc(static_cast<size_t>(C) * K);
    if (c.weight_rule == MPPI_WEIGHT_CEM) d_w.alloc(K);  // (allocated before any graph capture)
    d_partials.alloc(static_cast<size_t>(C) * partials_ctrl_stride);
    d_groups.alloc(static_cast<size_t>(C) * n_groups * partial_stride);
    d_agg.alloc(static_cast<size_t>(2) * T);
    d_iters.alloc(C);
    CUDA_TRY(cudaMemset(d_iters.p, 0, C * sizeof(uint64_t)));
    h_iters.assign(C, 0);
    d_trace_base.alloc(C);
    d_seeds.alloc(C);
    std::vector<uint64_t> seeds(C);
    // keyed by the GLOBAL controller index (a fleet sharded over ranks keeps
    // one noise stream per controller whatever the rank count)
    for (int i = 0; i < C; ++i) seeds[i] = c.seed + static_cast<uint64_t>(c.controller_offset) + static_cast<uint64_t>(i);
    CUDA_TRY(cudaMemcpy(d_seeds.p, seeds.data(), C * sizeof(uint64_t), cudaMemcpyHostToDevice));
    d_abort.alloc(C);
    CUDA_TRY(cudaMemset(d_abort.p, 0, C * sizeof(int)));
    d_bad.alloc(1);
    d_rho_eta.alloc(2);
    d_status.alloc(C);
    CUDA_TRY(cudaMemset(d_status.p, 0, C * sizeof(StepStatus)));
    h_status.alloc(C);
    std::memset(h_status.p, 0, sizeof(StepStatus) * C);
    h_x0.alloc(static_cast<size_t>(C) * 8);
    std::memset(h_x0.p, 0, sizeof(R) * C * 8);
    // decay^t table (std::pow, costs.cpp:35)
    std::vector<R> decay(T + 1);
    for (int t = 0; t <= T; ++t) decay[t] = static_cast<R>(std::pow(c.cost.decay, t));
    d_decay.alloc(T + 1);
    CUDA_TRY(cudaMemcpy(d_decay.p, decay.data(), (T + 1) * sizeof(R), cudaMemcpyHostToDevice));
    d_map_ptrs.alloc(C);
    CUDA_TRY(cudaMemset(d_map_ptrs.p, 0, C * sizeof(const R*)));
    if (c.system == MPPI_SYSTEM_QUADRATIC) has_mlp = true, has_map = true;
    w32 = std::make_unique<MlpParams<R, 32>>();
    w64 = std::make_unique<MlpParams<R, 64>>();
    std::memset(w32.get(), 0, sizeof(MlpParams<R, 32>));
    std::memset(w64.get(), 0, sizeof(MlpParams<R, 64>));
  }

  ~Handle() override {
    for (auto& g : graph)
      if (g) cudaGraphExecDestroy(g);
    if (comm) nccl().CommDestroy(comm);
    leave_local_group();
    if (ev_x0) cudaEventDestroy(ev_x0);
    if (ev_x1) cudaEventDestroy(ev_x1);
    if (ev_a) cudaEventDestroy(ev_a);
    if (ev_b) cudaEventDestroy(ev_b);
    if (ev_it0) cudaEventDestroy(ev_it0);
    if (ev_it1) cudaEventDestroy(ev_it1);
    if (stream) cudaStreamDestroy(stream);
  }

  void choose_variant() {
    const char* kv = std::getenv("MPPI_KERNEL");
    const std::string kernel = kv ? kv : "";
    const bool force_generic = kernel == "generic";
    const bool f32_vehicle = std::is_same<R, float>::value && cfg.system == MPPI_SYSTEM_VEHICLE_MLP;
    // default K1 for the fp32 vehicle model: tensor cores at H = 32 and 64
    // (MPPI_KERNEL=ws: the FFMA2 warp-specialised kernel, generic: one thread
    // per sample)
    use_tc = f32_vehicle && !force_generic && kernel != "ws";
    // From 32 768 samples on (counting every controller of a fleet): K1 on
    // tcgen05 / TMEM, one sample per thread (rollout_umma.cuh; measured at
    // H = 32 3-10 % faster than the mma.sync kernel there and 1.8x slower at
    // 16 384, where it runs one 4-warp CTA per SM; at H = 64 (c2) 11 %
    // faster; profiles/README.md).  MPPI_KERNEL=umma forces it,
    // MPPI_KERNEL=mma keeps the mma.sync kernel
    const bool umma_default = static_cast<long long>(K) * C >= 32768;
    if (use_tc && (kernel == "umma" || (umma_default && kernel != "mma"))) {
      use_umma = true;
      chunk_samples = mppi_dev::kUmmaThreads;
      return;
    }
    if (use_tc) {
      // one m16 tile per warp while warps are scarce (counting every
      // controller of a fleet), two once the grid fills the GPU several times
      tc_mt = static_cast<long long>(K) * C <= 32768 ? 1 : 2;
      if (H == 64) tc_mt = 1;     // (the H = 64 kernel keeps one tile per warp)
      if (const char* mv = std::getenv("MPPI_TC_MT"); mv && H == 32) tc_mt = std::atoi(mv) == 1 ? 1 : 2;
      chunk_samples = 16 * tc_mt;
      return;
    }
    use_ws = f32_vehicle && !force_generic;
    if (!use_ws) {
      chunk_samples = kBlock;
      return;
    }
    chunk_samples = 32;
    // Split the MLP over L warps until the grid holds ~1024 warps (measured
    // on B200, tools/sweep.py: K=1920 -> L=4, K=16384 -> L=2, K>=65536 ->
    // L=1; L=8 never won).  Weights: shared memory, except for the
    // one-warp-per-chunk kernel at large K where the constant bank wins.
    const long long chunks = (K + 31) / 32;
    int L = 1;
    while (L < 4 && chunks * (2 * L) <= 1024) L *= 2;
    if (H == 64 && L < 2) L = 2;  // the H = 64 kernels split the hidden layer over >= 2 warps
    ws_smem_w = !(L == 1 && chunks >= 2048);
    if (const char* lv = std::getenv("MPPI_WS_L")) {
      const int want = std::atoi(lv);
      if (want == 1 || want == 2 || want == 4 || want == 8) L = want;
    }
    if (const char* sv = std::getenv("MPPI_WS_SMEM_W")) ws_smem_w = std::atoi(sv) != 0;
    if (H == 64 && L < 2) L = 2;
    ws_L = L;
  }
  static void validate_config(const mppi_gpu_config& c) {
    // SamplingParams::validate (types.hpp:105-122)
    if (c.samples < 1) throw_invalid("SamplingParams: samples must be >= 1");
    if (c.horizon_steps < 1) throw_invalid("SamplingParams: horizon_steps must be >= 1");
    if (!(c.dt > 0.0)) throw_invalid("SamplingParams: dt must be > 0");
    for (int i = 0; i < 2; ++i)
      if (!(c.sigma_diag[i] > 0.0) || !std::isfinite(c.sigma_diag[i]))
        throw_invalid("SamplingParams: sigma_diag entries must be finite and > 0");
    if (!(c.lambda > 0.0)) throw_invalid("SamplingParams: lambda must be > 0");
    if (!(c.gamma >= 0.0)) throw_invalid("SamplingParams: gamma must be >= 0");
    if (!(c.explore_fraction >= 0.0 && c.explore_fraction < 1.0))
      throw_invalid("SamplingParams: explore_fraction must be in [0, 1)");
    // ControlBounds::validate (dynamics.hpp:19-28)
    for (int i = 0; i < 2; ++i)
      if (!(c.bounds_lower[i] < c.bounds_upper[i])) throw_invalid("ControlBounds: lower must be < upper");
    if (c.sg_window != 0) {
      if (c.sg_window < 3 || c.sg_window % 2 == 0) throw_invalid("sg_coefficients: window must be odd and >= 3");
      if (c.sg_degree < 0 || c.sg_degree >= c.sg_window) throw_invalid("sg_coefficients: need 0 <= degree < window");
      if (c.sg_window > kMaxSgWindow) throw Error(MPPI_ERR_UNSUPPORTED, "sg window > 63");
    }
    if (c.weight_rule != MPPI_WEIGHT_IT && c.weight_rule != MPPI_WEIGHT_CEM) throw_invalid("weight_rule");
    if (c.weight_rule == MPPI_WEIGHT_CEM) {  // cem_weights (weights.cpp:27-40)
      if (!(c.cem_delta > 0.0 && c.cem_delta < 1.0)) throw_invalid("cem_weights: delta must be in (0, 1)");
      if (std::lround(c.samples * (1.0 - c.cem_delta)) < 1)
        throw_invalid("cem_weights: delta leaves an empty elite set");
      if (c.n_controllers != 1) throw Error(MPPI_ERR_UNSUPPORTED, "the CEM rule runs one controller per handle");
    }
    if (c.noise_mode < 0 || c.noise_mode > 2) throw_invalid("noise_mode");
    if (c.precision != MPPI_FP32 && c.precision != MPPI_FP64) throw_invalid("precision");
    if (c.system != MPPI_SYSTEM_VEHICLE_MLP && c.system != MPPI_SYSTEM_QUADRATIC &&
        c.system != MPPI_SYSTEM_VEHICLE_BASIS && c.system != MPPI_SYSTEM_VEHICLE_BICYCLE)
      throw_invalid("system");
    if (c.mlp_hidden != 32 && c.mlp_hidden != 64) throw_invalid("mlp_hidden must be 32 or 64");
    if (c.n_controllers < 1) throw_invalid("n_controllers must be >= 1");
    if (c.controller_offset < 0) throw_invalid("controller_offset must be >= 0");
    if (c.noise_mode == MPPI_NOISE_INJECTED && c.n_controllers != 1)
      throw Error(MPPI_ERR_UNSUPPORTED, "injected noise supports one controller per handle");
    if (c.horizon_steps > 4096) throw Error(MPPI_ERR_UNSUPPORTED, "horizon_steps > 4096");
    if (!(c.cost.decay > 0.0 && c.cost.decay <= 1.0)) throw_invalid("CostParams: decay must be in (0, 1]");
    if (!(c.cost.alpha_track >= 0.0 && c.cost.alpha_speed >= 0.0 && c.cost.alpha_stab >= 0.0))
      throw_invalid("CostParams: weights must be >= 0");
  }

  int state_dim() const { return cfg.system == MPPI_SYSTEM_QUADRATIC ? 2 : 7; }
  void check_ctrl(int c) const {
    if (c < 0 || c >= C) throw_invalid("controller index out of range");
  }
  void invalidate_graphs() {
    for (auto& g : graph)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
  }
  void require_ready() const {
    if (!has_mlp) throw_invalid("vehicle system: model (MLP weights / basis Theta) not set");
    if (!has_map) throw_invalid("vehicle system: costmap not set");
    if (cfg.noise_mode == MPPI_NOISE_INJECTED && !has_noise) throw_invalid("INJECTED noise: no batch set");
  }

  // ----------------------------------------------------------- set data ---
  void set_mlp(int hidden, const double* w1, const double* b1, const double* w2, const double* b2,
               const double* w3, const double* b3) {
    if (cfg.system != MPPI_SYSTEM_VEHICLE_MLP) throw_invalid("set_dynamics_mlp: system has no MLP");
    if (hidden != H) throw_invalid("set_dynamics_mlp: hidden size must match config.mlp_hidden");
    auto fill = [&](auto& w) {
      for (int j = 0; j < H; ++j) {
        for (int i = 0; i < 6; ++i) w.w1t[i][j] = static_cast<R>(w1[j * 6 + i]);
        w.b1[j] = static_cast<R>(b1[j]);
        w.b2[j] = static_cast<R>(b2[j]);
        for (int i = 0; i < H; ++i) w.w2t[i][j] = static_cast<R>(w2[j * H + i]);
      }
      for (int o = 0; o < 4; ++o) {
        w.b3[o] = static_cast<R>(b3[o]);
        for (int i = 0; i < H; ++i) w.w3t[i][o] = static_cast<R>(w3[o * H + i]);
      }
    };
    for (int i = 0; i < H * 6; ++i)
      if (!std::isfinite(w1[i])) throw_invalid("MLP weights must be finite");
    auto upload_tc = [&](const auto& w) {
      if (!use_tc) return;
      if (use_umma) {
        const std::vector<unsigned char> img = umma_build_image(w);
        d_umma.alloc(img.size());
        CUDA_TRY(cudaMemcpy(d_umma.p, img.data(), img.size(), cudaMemcpyHostToDevice));
      }
      std::vector<uint32_t> frag = tc_build_fragments(w);
      d_tcfrag.alloc(frag.size());
      CUDA_TRY(cudaMemcpy(d_tcfrag.p, frag.data(), frag.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
      d_plantw.alloc(sizeof(w));
      CUDA_TRY(cudaMemcpy(d_plantw.p, &w, sizeof(w), cudaMemcpyHostToDevice));
    };
    if (H == 32) {
      fill(*w32);
      upload_tc(*w32);
    } else {
      fill(*w64);
      upload_tc(*w64);
      if (!kWeightsByValue<R, 64>) {
        d_w64.alloc(1);
        CUDA_TRY(cudaMemcpy(d_w64.p, w64.get(), sizeof(MlpParams<R, 64>), cudaMemcpyHostToDevice));
      }
    }
    has_mlp = true;
    invalidate_graphs();
  }

  // BasisFunctionModel Theta (dynamics.hpp:75-82), theta[b*4 + o]; like
  // load_theta, non-finite entries are rejected (dynamics.cpp:240-242).
  void set_basis(const double* theta) {
    if (cfg.system != MPPI_SYSTEM_VEHICLE_BASIS) throw_invalid("set_dynamics_basis: system is not the basis model");
    for (int i = 0; i < 100; ++i)
      if (!std::isfinite(theta[i])) throw_invalid("set_dynamics_basis: non-finite Theta entry");
    for (int b = 0; b < 25; ++b)
      for (int o = 0; o < 4; ++o) theta_r.c[b][o] = static_cast<R>(theta[b * 4 + o]);
    has_mlp = true;  // the model is set
    invalidate_graphs();
  }

  // BicycleParams::validate (dynamics.hpp:53-61) and the friction circle of
  // brush_tire_force (dynamics.cpp:25-27) at the largest admissible throttle.
  void set_bicycle(const mppi_bicycle_params& p) override {
    if (cfg.system != MPPI_SYSTEM_VEHICLE_BICYCLE) throw_invalid("set_dynamics_bicycle: system is not the bicycle model");
    const double v[9] = {p.mass, p.yaw_inertia, p.a, p.b, p.stiffness, p.mu, p.load, p.steer_scale, p.force_scale};
    for (double x : v)
      if (!(x > 0.0) || !std::isfinite(x)) throw_invalid("BicycleParams: all parameters must be positive");
    const double thr = std::max(std::abs(cfg.bounds_lower[1]), std::abs(cfg.bounds_upper[1]));
    if (p.force_scale * thr > p.mu * p.load)
      throw Error(MPPI_ERR_DOMAIN, "brush_tire_force: |u_F| exceeds the friction circle mu*F_z");
    bike_r = BicycleDev<R>{static_cast<R>(p.mass), static_cast<R>(p.yaw_inertia), static_cast<R>(p.a),
                           static_cast<R>(p.b), static_cast<R>(p.stiffness), static_cast<R>(p.mu),
                           static_cast<R>(p.load), static_cast<R>(p.steer_scale), static_cast<R>(p.force_scale)};
    has_mlp = true;  // the model is set
    invalidate_graphs();
  }

  template <class Src>
  void set_map(int ctrl, const Src* values, int width, int height, double x0, double y0, double res) {
    if (cfg.system == MPPI_SYSTEM_QUADRATIC) throw_invalid("set_costmap: system has no costmap");
    // CostMap::validate (costs.hpp:24-37)
    if (width < 2 || height < 2) throw_invalid("CostMap: width and height must be >= 2");
    if (!(res > 0.0)) throw_invalid("CostMap: resolution must be > 0");
    if (has_map && (width != map_w || height != map_h || x0 != map_x0 || y0 != map_y0 || res != map_res))
      throw_invalid("set_costmap: all maps of a handle share one geometry");
    const size_t n = static_cast<size_t>(width) * height;
    std::vector<R> v(n);
    for (size_t i = 0; i < n; ++i) {
      const double d = static_cast<double>(values[i]);
      if (!std::isfinite(d) || std::abs(d) > 2.5) throw_invalid("CostMap: values must be finite and within +-2.5");
      v[i] = static_cast<R>(d);
    }
    map_w = width;
    map_h = height;
    map_x0 = x0;
    map_y0 = y0;
    map_res = res;
    std::vector<const R*> ptrs(C);
    CUDA_TRY(cudaMemcpy(ptrs.data(), d_map_ptrs.p, C * sizeof(const R*), cudaMemcpyDeviceToHost));
    if (ctrl < 0) {
      d_map_shared.alloc(n);
      CUDA_TRY(cudaMemcpy(d_map_shared.p, v.data(), n * sizeof(R), cudaMemcpyHostToDevice));
      d_map_fleet.clear();
      for (int c = 0; c < C; ++c) ptrs[c] = d_map_shared.p;
    } else {
      check_ctrl(ctrl);
      if (d_map_fleet.size() != static_cast<size_t>(C)) d_map_fleet.resize(C);
      if (!d_map_fleet[ctrl]) d_map_fleet[ctrl] = std::make_unique<DevBuf<R>>();
      d_map_fleet[ctrl]->alloc(n);
      CUDA_TRY(cudaMemcpy(d_map_fleet[ctrl]->p, v.data(), n * sizeof(R), cudaMemcpyHostToDevice));
      ptrs[ctrl] = d_map_fleet[ctrl]->p;
    }
    CUDA_TRY(cudaMemcpy(d_map_ptrs.p, ptrs.data(), C * sizeof(const R*), cudaMemcpyHostToDevice));
    bool all = true;
    for (int c = 0; c < C; ++c) all = all && ptrs[c] != nullptr;
    has_map = all;
    invalidate_graphs();
  }

  void perturb_fleet(double sigma, uint64_t seed) {
    if (!d_map_shared.p) throw_invalid("perturb_fleet_costmaps: set a shared costmap first");
    if (!(sigma >= 0.0)) throw_invalid("perturb_fleet_costmaps: sigma must be >= 0");
    const size_t n = static_cast<size_t>(map_w) * map_h;
    d_map_fleet.clear();
    d_map_fleet.resize(C);
    std::vector<const R*> ptrs(C);
    for (int c = 0; c < C; ++c) {
      d_map_fleet[c] = std::make_unique<DevBuf<R>>();
      d_map_fleet[c]->alloc(n);
      // (stream of the GLOBAL controller index, as the noise seeds)
      perturb_map_kernel<R><<<592, 256, 0, stream>>>(d_map_shared.p, n, c + cfg.controller_offset, sigma, seed,
                                                     d_map_fleet[c]->p);
      ++launches;
      CUDA_TRY(cudaGetLastError());
      ptrs[c] = d_map_fleet[c]->p;
    }
    CUDA_TRY(cudaMemcpyAsync(d_map_ptrs.p, ptrs.data(), C * sizeof(const R*), cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    invalidate_graphs();
  }

  void map_geometry(int* w, int* h, double* x0, double* y0, double* res) const override {
    if (!has_map) throw_invalid("costmap not set");
    *w = map_w;
    *h = map_h;
    *x0 = map_x0;
    *y0 = map_y0;
    *res = map_res;
  }
  void get_map_f32(int ctrl, float* out) override {
    check_ctrl(ctrl);
    if (!has_map) throw_invalid("get_costmap: no costmap set");
    std::vector<const R*> ptrs(C);
    CUDA_TRY(cudaStreamSynchronize(stream));
    CUDA_TRY(cudaMemcpy(ptrs.data(), d_map_ptrs.p, C * sizeof(const R*), cudaMemcpyDeviceToHost));
    const size_t n = static_cast<size_t>(map_w) * map_h;
    std::vector<R> v(n);
    CUDA_TRY(cudaMemcpy(v.data(), ptrs[ctrl], n * sizeof(R), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < n; ++i) out[i] = static_cast<float>(v[i]);
  }
  void set_plan(int ctrl, const double* U) {
    check_ctrl(ctrl);
    std::vector<R> v(2 * T);
    for (int i = 0; i < 2 * T; ++i) {
      if (!std::isfinite(U[i])) throw_invalid("ControlPlan: needs a finite T x m matrix, T >= 1");
      v[i] = static_cast<R>(U[i]);
    }
    CUDA_TRY(cudaMemcpy(d_plan.p + static_cast<size_t>(ctrl) * 2 * T, v.data(), 2 * T * sizeof(R),
                        cudaMemcpyHostToDevice));
  }
  void get_plan(int ctrl, double* U) {
    check_ctrl(ctrl);
    std::vector<R> v(2 * T);
    CUDA_TRY(cudaStreamSynchronize(stream));
    CUDA_TRY(cudaMemcpy(v.data(), d_plan.p + static_cast<size_t>(ctrl) * 2 * T, 2 * T * sizeof(R),
                        cudaMemcpyDeviceToHost));
    for (int i = 0; i < 2 * T; ++i) U[i] = static_cast<double>(v[i]);
  }
  void set_iteration(int ctrl, uint64_t it) {
    check_ctrl(ctrl);
    CUDA_TRY(cudaMemcpy(d_iters.p + ctrl, &it, sizeof(uint64_t), cudaMemcpyHostToDevice));
    h_iters[ctrl] = it;
  }
  uint64_t get_iteration(int ctrl) {
    check_ctrl(ctrl);
    uint64_t it = 0;
    CUDA_TRY(cudaStreamSynchronize(stream));
    CUDA_TRY(cudaMemcpy(&it, d_iters.p + ctrl, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    h_iters[ctrl] = it;
    return it;
  }
  void set_seed(int ctrl, uint64_t seed) {
    check_ctrl(ctrl);
    CUDA_TRY(cudaMemcpy(d_seeds.p + ctrl, &seed, sizeof(uint64_t), cudaMemcpyHostToDevice));
  }
  void upload_injected(const double* eps) {
    const size_t n = static_cast<size_t>(K) * 2 * T;
    for (size_t i = 0; i < n; ++i)
      if (!std::isfinite(eps[i])) throw_invalid("perturbation batch must be finite");
    d_eps_ref.alloc(n);
    d_inj.alloc(n);
    CUDA_TRY(cudaMemcpyAsync(d_eps_ref.p, eps, n * sizeof(double), cudaMemcpyHostToDevice, stream));
    inject_transpose_kernel<R><<<296, 256, 0, stream>>>(d_eps_ref.p, K, T, d_inj.p);
    ++launches;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(stream));
  }
  void set_noise(const double* eps) {
    upload_injected(eps);
    has_noise = true;
  }

  // ------------------------------------------------------------- launch ---
  RolloutArgs<R> rollout_args() const {
    RolloutArgs<R> a{};
    a.K = K;
    a.T = T;
    a.zero_start = zero_start;
    a.chunk0 = chunk_lo;
    a.chunk_end = chunk_hi;
    a.partial_stride = partial_stride;
    a.partials_ctrl_stride = partials_ctrl_stride;
    a.lambda = static_cast<R>(cfg.lambda);
    a.gamma = static_cast<R>(cfg.gamma);
    a.sigma0 = static_cast<R>(cfg.sigma_diag[0]);
    a.sigma1 = static_cast<R>(cfg.sigma_diag[1]);
    a.dlambda = cfg.lambda;
    a.dscale0 = std::sqrt(cfg.sigma_diag[0]);
    a.dscale1 = std::sqrt(cfg.sigma_diag[1]);
    a.scale0 = static_cast<R>(a.dscale0);
    a.scale1 = static_cast<R>(a.dscale1);
    a.sys = system_args();
    a.plan = d_plan.p;
    a.x0 = d_x0.p;
    a.maps = d_map_ptrs.p;
    a.map_w = map_w;
    a.map_h = map_h;
    a.map_x0 = static_cast<R>(map_x0);
    a.map_y0 = static_cast<R>(map_y0);
    a.map_res = static_cast<R>(map_res);
    a.map_inv_res = static_cast<R>(1.0 / map_res);
    a.inj = d_inj.p;
    a.seeds = d_seeds.p;
    a.iters = d_iters.p;
    a.abort_flag = reinterpret_cast<const int*>(d_status.p);  // StepStatus.code is the first field
    static_assert(sizeof(StepStatus) % sizeof(int) == 0, "StepStatus must be a whole number of ints");
    a.abort_stride = static_cast<int>(sizeof(StepStatus) / sizeof(int));
    a.costs = d_costs.p;
    a.pdl = k1_pdl && use_tc ? 1 : 0;
    a.partials = d_partials.p;
    return a;
  }
  SystemArgs<R> system_args() const {
    SystemArgs<R> s{};
    s.dt = static_cast<R>(cfg.dt);
    s.lo0 = static_cast<R>(cfg.bounds_lower[0]);
    s.lo1 = static_cast<R>(cfg.bounds_lower[1]);
    s.hi0 = static_cast<R>(cfg.bounds_upper[0]);
    s.hi1 = static_cast<R>(cfg.bounds_upper[1]);
    const mppi_cost_params& c = cfg.cost;
    s.cost.alpha_track = static_cast<R>(c.alpha_track);
    s.cost.alpha_speed = static_cast<R>(c.alpha_speed);
    s.cost.alpha_stab = static_cast<R>(c.alpha_stab);
    s.cost.v_des = static_cast<R>(c.v_des);
    s.cost.impulse = static_cast<R>(c.impulse);
    s.cost.boundary_threshold = static_cast<R>(c.boundary_threshold);
    s.cost.slip_limit = static_cast<R>(c.slip_limit);
    s.cost.crash_penalty = static_cast<R>(c.crash_penalty);
    s.cost.crash_threshold = static_cast<R>(c.crash_threshold);
    s.cost.roll_limit = static_cast<R>(c.roll_limit);
    s.decay_pow = d_decay.p;
    s.with_terminal = cfg.with_terminal;
    s.quad_cost_scale = static_cast<R>(cfg.quad_cost_scale);
    s.theta = theta_r;
    s.bike = bike_r;
    return s;
  }
  template <int HH>
  WeightHolder<R, HH> holder() const {
    WeightHolder<R, HH> wh;
    if constexpr (kWeightsByValue<R, HH>) {
      if constexpr (HH == 32) wh.w = *w32;
      else wh.w = *w64;
    } else {
      wh.p = d_w64.p;
    }
    return wh;
  }

  // Calls f.template operator()<HH, Sys, Mode>() for the configured variant.
  template <class F>
  void dispatch(int mode, F&& f) const {
    auto by_mode = [&](auto hh, auto sys) {
      using Sys = typename decltype(sys)::type;
      constexpr int HH = decltype(hh)::value;
      switch (mode) {
        case kInjected: f.template operator()<HH, Sys, kInjected>(); break;
        case kRefSplitmix: f.template operator()<HH, Sys, kRefSplitmix>(); break;
        default: f.template operator()<HH, Sys, kPhilox>(); break;
      }
    };
    if (cfg.system == MPPI_SYSTEM_QUADRATIC)
      by_mode(std::integral_constant<int, 32>{}, type_tag<Quadratic<R, 32>>{});
    else if (cfg.system == MPPI_SYSTEM_VEHICLE_BASIS)
      by_mode(std::integral_constant<int, 32>{}, type_tag<VehicleBasis<R, 32>>{});
    else if (cfg.system == MPPI_SYSTEM_VEHICLE_BICYCLE)
      by_mode(std::integral_constant<int, 32>{}, type_tag<VehicleBicycle<R, 32>>{});
    else if (H == 32)
      by_mode(std::integral_constant<int, 32>{}, type_tag<VehicleMlp<R, 32>>{});
    else
      by_mode(std::integral_constant<int, 64>{}, type_tag<VehicleMlp<R, 64>>{});
  }
  template <class T_>
  struct type_tag {
    using type = T_;
  };

  size_t rollout_smem() const { return sizeof(Acc) * (kBlock / 32) * 2 * T + sizeof(R) * 2 * T; }

  void launch_ws(const RolloutArgs<R>& a, int mode, dim3 grid) {
    if constexpr (std::is_same<R, float>::value) {
      const size_t smem = sizeof(float) * 2 * T;
      if (H == 32) CUDA_TRY(launch_rollout_ws_h32(a, holder<32>(), mode, ws_L, ws_smem_w, grid, smem, stream));
      else CUDA_TRY(launch_rollout_ws_h64(a, holder<64>(), mode, ws_L, ws_smem_w, grid, smem, stream));
    }
  }

  // events: bracket the launch with ev_a/ev_b without synchronising (used
  // inside captured graphs; the caller reads the elapsed time afterwards).
  void enqueue_rollout(int mode, bool events = false) {
    const RolloutArgs<R> a = rollout_args();
    const size_t smem = rollout_smem();
    const dim3 grid(chunk_hi - chunk_lo, C);
    if (chunk_hi <= chunk_lo) return;  // a rank without samples (fewer chunks than ranks)
    // inside stream capture an event record is only a dependency edge unless
    // it is marked external; external records become graph event nodes
    if (events) CUDA_TRY(cudaEventRecordWithFlags(ev_a, stream, cudaEventRecordExternal));
    else if (profile) CUDA_TRY(cudaEventRecord(ev_a, stream));
    if (use_umma) {
      if constexpr (std::is_same<R, float>::value)
        CUDA_TRY((H == 32 ? launch_rollout_umma<32> : launch_rollout_umma<64>)(a, d_umma.p, mode, chunk_hi - chunk_lo,
                                                                              C, stream));
    } else if (use_tc) {
      if constexpr (std::is_same<R, float>::value)
        CUDA_TRY((H == 32 ? launch_rollout_tc<32> : launch_rollout_tc<64>)(a, d_tcfrag.p, mode, tc_mt,
                                                                          chunk_hi - chunk_lo, C, stream));
      tc_pair_used = tc_detail::g_tc_last_pair;
    } else if (use_ws) {
      launch_ws(a, mode, grid);
    } else {
      dispatch(mode, [&]<int HH, class Sys, int Mode>() {
        auto kern = rollout_kernel<R, HH, Sys, Mode, kBlock>;
        if (smem > 48 * 1024)
          CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kern<<<grid, kBlock, smem, stream>>>(a, holder<HH>());
      });
    }
    ++launches;
    CUDA_TRY(cudaGetLastError());
    if (events) CUDA_TRY(cudaEventRecordWithFlags(ev_b, stream, cudaEventRecordExternal));
    if (profile && !events) {
      CUDA_TRY(cudaEventRecord(ev_b, stream));
      CUDA_TRY(cudaEventSynchronize(ev_b));
      float ms = 0;
      CUDA_TRY(cudaEventElapsedTime(&ms, ev_a, ev_b));
      prof_ms += ms;
      ++prof_launches;
    }
  }

  // The fixed-group merge of this rank's chunk partials (group.cuh);
  // programmatic dependent of K1 when K1 ran just before it.
  void enqueue_group_merge(bool after_k1) {
    CUDA_TRY(launch_group_merge(d_partials.p, partials_ctrl_stride, n_chunks, n_groups, group_lo, group_hi - group_lo,
                                partial_stride, cfg.lambda, d_groups.p,
                                static_cast<long long>(n_groups) * partial_stride, C, after_k1, stream));
    ++launches;
  }

  // One iteration after the host inputs are staged: K1 over this rank's
  // chunks, the fixed-group merge, [the exchange of group rows], then the
  // merge of the group rows + epilogue (tensor-core path: tail_kernel;
  // otherwise epilogue_kernel).  CEM: K1, the elite selection, the weighted
  // average over the regenerated batch, the epilogue.
  void enqueue_iteration(int mode, bool events, bool slide, bool increment, bool plant, bool trace) {
    if (cfg.weight_rule == MPPI_WEIGHT_CEM) {
      // CEM (controller.cpp:111-116 -> weights.cpp:27-53): K1 for the costs,
      // the device elite selection, update_plan with those weights
      // (ascending-k weighted sum over the regenerated batch), the epilogue
      enqueue_rollout(mode, events);
      cem_weights_kernel<1024><<<1, 1024, 0, stream>>>(d_costs.p, K, cem_elite(), d_w.p, d_rho_eta.p, nullptr,
                                                        d_status.p);
      ++launches;
      CUDA_TRY(cudaGetLastError());
      const RolloutArgs<R> a = rollout_args();
      const int blocks = (T + 127) / 128;
      switch (mode) {
        case kInjected: weighted_agg_kernel<R, kInjected><<<blocks, 128, 0, stream>>>(a, d_w.p, d_agg.p); break;
        case kRefSplitmix: weighted_agg_kernel<R, kRefSplitmix><<<blocks, 128, 0, stream>>>(a, d_w.p, d_agg.p); break;
        default: weighted_agg_kernel<R, kPhilox><<<blocks, 128, 0, stream>>>(a, d_w.p, d_agg.p); break;
      }
      ++launches;
      CUDA_TRY(cudaGetLastError());
      enqueue_epilogue(false, slide, increment, plant, trace, 1);
      return;
    }
    enqueue_front(mode, events);
    enqueue_back(events, slide, increment, plant, trace);
  }
  // K1 + the group merge (everything before the exchange).  (With K1's event
  // nodes around it, the group merge is an ordinary dependent.)
  void enqueue_front(int mode, bool events) {
    const bool k1 = chunk_hi > chunk_lo;
    enqueue_rollout(mode, events);
    enqueue_group_merge(k1 && !events);
  }
  // the exchange, the merge of the group rows and the epilogue
  void enqueue_back(bool events, bool slide, bool increment, bool plant, bool trace) {
    enqueue_exchange(events);
    if (use_tc) {
      if constexpr (std::is_same<R, float>::value) {
        TailArgs ta{};
        ta.plant_w = d_plantw.p;
        ta.e = epilogue_args(true, slide, increment, plant, trace, /*merged_row=*/true);
        if (status_direct) ta.e.status_host = h_status.p;  // mapped pinned (UVA)
        // a programmatic dependent of the group merge unless the exchange sits between
        const bool pdl = world == 1;
        CUDA_TRY((H == 32 ? launch_tail_tc<32> : launch_tail_tc<64>)(
            d_groups.p, n_groups, partial_stride, static_cast<long long>(n_groups) * partial_stride, cfg.lambda, ta,
            C, pdl, stream));
        ++launches;
      }
      return;
    }
    enqueue_epilogue(true, slide, increment, plant, trace, C);
  }

  // The exchange of the group rows: rank r's rows [group_lo, group_hi) to
  // every rank (NCCL all-gather in place, or peer copies in a local group).
  void enqueue_exchange(bool events) {
    if (world <= 1) return;
    const size_t count = static_cast<size_t>(n_groups / world) * partial_stride;
    if (events) CUDA_TRY(cudaEventRecordWithFlags(ev_x0, stream, cudaEventRecordExternal));
    if (exchange_mode == kExNccl) {
      Acc* base = d_groups.p;
      NCCL_TRY(nccl().AllGather(base + static_cast<size_t>(rank) * count, base, count, ncclFloat64, comm, stream));
    } else if (exchange_mode == kExLocal) {
      for (int p = 0; p < world; ++p) {
        if (p == rank) continue;
        const Handle<R>* peer = local_peers[p];
        if (!peer) throw Error(MPPI_ERR_RUNTIME, "local group: a peer handle was destroyed");
        CUDA_TRY(cudaMemcpyPeerAsync(d_groups.p + static_cast<size_t>(p) * count, device,
                                     peer->d_groups.p + static_cast<size_t>(p) * count, peer->device,
                                     count * sizeof(Acc), stream));
      }
    }
    if (events) CUDA_TRY(cudaEventRecordWithFlags(ev_x1, stream, cudaEventRecordExternal));
  }

  EpilogueArgs<R> epilogue_args(bool merge, bool slide, bool increment, bool plant, bool trace,
                                bool merged_row = false) const {
    EpilogueArgs<R> e{};
    e.T = T;
    e.n_chunks = n_groups;  // the rows merged by the epilogue: the group rows
    // rows per shared-memory tile: <= 32 and <= ~96 KB
    e.tile_rows = std::max(1, std::min({32, e.n_chunks, static_cast<int>((96 * 1024) / (8 * partial_stride))}));
    e.partial_stride = partial_stride;
    e.partials_ctrl_stride = static_cast<long long>(n_groups) * partial_stride;
    e.lambda = cfg.lambda;
    e.lo0 = static_cast<R>(cfg.bounds_lower[0]);
    e.lo1 = static_cast<R>(cfg.bounds_lower[1]);
    e.hi0 = static_cast<R>(cfg.bounds_upper[0]);
    e.hi1 = static_cast<R>(cfg.bounds_upper[1]);
    e.sg_window = static_cast<int>(sg.size());
    for (size_t i = 0; i < sg.size(); ++i) e.sg[i] = sg[i];
    e.slide = slide;
    e.increment = increment;
    e.plant = plant;
    e.partials = merge ? d_groups.p : nullptr;
    if (merge && merged_row) {  // the tensor-core tail merges in shared memory (tail.cuh)
      e.partials = nullptr;
      e.n_chunks = 1;
      e.tile_rows = 1;
      e.partials_ctrl_stride = partial_stride;
    }
    e.agg_in = merge ? nullptr : d_agg.p;
    e.plan = d_plan.p;
    e.x0 = d_x0.p;
    e.iters = d_iters.p;
    e.status = d_status.p;
    e.u_trace = trace ? d_utrace.p : nullptr;
    e.x_trace = trace ? d_xtrace.p : nullptr;
    e.trace_base = d_trace_base.p;
    e.n_ctrl = C;
    e.sys = system_args();
    return e;
  }
  void enqueue_epilogue(bool merge, bool slide, bool increment, bool plant, bool trace, int ctrls,
                        bool merged_row = false) {
    const EpilogueArgs<R> e = epilogue_args(merge, slide, increment, plant, trace, merged_row);
    dispatch(kPhilox, [&]<int HH, class Sys, int Mode>() {
      const size_t smem = epilogue_smem_bytes<R, HH>(T, merge ? e.n_chunks : 0, merge ? e.tile_rows : 0,
                                                     partial_stride, plant);
      auto kern = epilogue_kernel<R, HH, Sys, kEpiBlock>;
      if (smem > 48 * 1024)
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      kern<<<ctrls, kEpiBlock, smem, stream>>>(e, holder<HH>());
    });
    ++launches;
    CUDA_TRY(cudaGetLastError());
  }

  void upload_x0(const double* x0) {
    const int n = state_dim();
    for (int c = 0; c < C; ++c)
      for (int i = 0; i < 8; ++i) {
        const double v = (i < n) ? x0[c * n + i] : 0.0;
        if (!std::isfinite(v)) throw_invalid("x0 must be finite");
        h_x0.p[c * 8 + i] = static_cast<R>(v);
      }
  }

  // One captured graph per iteration flavour; replayed on every call.
  void run_graph(int which, bool slide, bool plant, bool trace) {
    if (graph[which] && graph_trace[which] != trace) {
      cudaGraphExecDestroy(graph[which]);
      graph[which] = nullptr;
    }
    if (!graph[which]) {
      cudaGraph_t g = nullptr;
      CUDA_TRY(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      try {
        // step graphs (slots 0, 1): x0 host-to-device, then K1.  The status
        // is clear between steps (throw_status clears it after a failure), so
        // no memset node.  (Reading x0 from the mapped host buffer in K1
        // instead of this copy measured 17 us slower: every warp's PCIe read.)
        // (tensor-core path: a one-CTA fetch kernel instead, K1 its programmatic
        // dependent, so K1's prologue overlaps the PCIe round trip)
        n_before_capture = launches;
        k1_pdl = which < 2 && use_tc && std::is_same<R, float>::value && cfg.weight_rule != MPPI_WEIGHT_CEM;
        if (k1_pdl) {
          if constexpr (std::is_same<R, float>::value) {
            const int n4 = C * 2;  // (rows of 8 floats: two float4 each; pinned buffers are page-aligned)
            const int threads = std::min(kFetchX0Block, (n4 + 31) / 32 * 32);
            fetch_x0_kernel<><<<(n4 + threads - 1) / threads, threads, 0, stream>>>(
                reinterpret_cast<const float4*>(h_x0.p), reinterpret_cast<float4*>(d_x0.p), n4);
            ++launches;
            CUDA_TRY(cudaGetLastError());
          }
        } else if (which < 2) {
          CUDA_TRY(cudaMemcpyAsync(d_x0.p, h_x0.p, C * 8 * sizeof(R), cudaMemcpyHostToDevice, stream));
        }
        const bool prof = profile;
        profile = false;
        // step graphs on the tensor-core path: the tail writes the host status
        // mirror itself (no device-to-host copy node at the end of the graph)
        status_direct = which < 2 && use_tc && std::is_same<R, float>::value && cfg.weight_rule != MPPI_WEIGHT_CEM;
        enqueue_iteration(cfg.noise_mode, /*events=*/which == 2, slide, /*increment=*/slide, plant, trace);
        k1_pdl = false;
        profile = prof;
        const bool direct = status_direct;
        status_direct = false;
        graph_direct[which] = direct;
        if (which < 2 && !direct)
          CUDA_TRY(cudaMemcpyAsync(h_status.p, d_status.p, C * sizeof(StepStatus), cudaMemcpyDeviceToHost, stream));
      } catch (...) {
        status_direct = false;
        k1_pdl = false;
        cudaStreamEndCapture(stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      CUDA_TRY(cudaStreamEndCapture(stream, &g));
      cudaError_t e = cudaGraphInstantiate(&graph[which], g, 0);
      cudaGraphDestroy(g);
      CUDA_TRY(e);
      graph_trace[which] = trace;
      graph_kernels[which] = static_cast<int>(launches - n_before_capture);
      launches = n_before_capture;  // counted again per replay below
    }
    CUDA_TRY(cudaGraphLaunch(graph[which], stream));
    launches += graph_kernels[which];
  }

  int check_status(bool update_iters) {
    int code = MPPI_OK;
    for (int c = 0; c < C; ++c) {
      if (h_status.p[c].code != 0 && code == MPPI_OK) code = h_status.p[c].code;
      if (update_iters) h_iters[c] = h_status.p[c].iteration;
    }
    return code;
  }
  [[noreturn]] void throw_status(int code) {
    // a failed step leaves the device status sticky (K1 aborts on it); clear
    // it so the next call starts clean (the step graphs carry no memset)
    cudaMemsetAsync(d_status.p, 0, C * sizeof(StepStatus), stream);
    cudaStreamSynchronize(stream);
    if (code == MPPI_ERR_NONFINITE) throw Error(code, "it_weights: non-finite cost");
    if (code == MPPI_ERR_INVALID_ARGUMENT)
      throw Error(code, "ControlPlan: needs a finite T x m matrix, T >= 1");
    throw Error(code, "device step failed");
  }

  // Wait for a step whose tail publishes the host status itself: spin on the
  // sequence words (every field is written before them), polling the stream
  // for errors now and then; false (the caller synchronises the stream) on
  // an error, a stream that drained without publishing, or after ~2 s.
  bool wait_published(const std::vector<unsigned long long>& want) {
    auto seq_ok = [&] {
      for (int c = 0; c < C; ++c)
        if (*reinterpret_cast<volatile unsigned long long*>(&h_status.p[c].seq) != want[c]) return false;
      return true;
    };
    const auto t0 = std::chrono::steady_clock::now();
    for (long i = 1;; ++i) {
      if (seq_ok()) {
        std::atomic_thread_fence(std::memory_order_acquire);
        return true;
      }
      if ((i & 1023) == 0) {
        const cudaError_t q = cudaStreamQuery(stream);
        if (q != cudaErrorNotReady) {
          if (q == cudaSuccess && seq_ok()) {
            std::atomic_thread_fence(std::memory_order_acquire);
            return true;
          }
          return false;
        }
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) return false;
      }
    }
  }

  // mpc_step / compute_control
  void step(const double* x0, double* u0, bool slide) {
    require_ready();
    upload_x0(x0);
    const int which = slide ? 0 : 1;
    std::vector<unsigned long long>& want = seq_want;
    want.resize(C);
    for (int c = 0; c < C; ++c) want[c] = *reinterpret_cast<volatile unsigned long long*>(&h_status.p[c].seq) + 1;
    run_graph(which, slide, false, false);
    if (!(graph_direct[which] && wait_published(want))) CUDA_TRY(cudaStreamSynchronize(stream));
    const int code = check_status(true);
    if (code != MPPI_OK) {
      // a failed step leaves plan and iteration untouched (mpc_step throws
      // before assigning cs.plan, controller.cpp:137-138)
      throw_status(code);
    }
    if (!slide) {
      // compute_control does not advance the iteration; the counter is read
      // back from the device state for the host mirror
      for (int c = 0; c < C; ++c) h_iters[c] = h_status.p[c].iteration;
    }
    if (u0)
      for (int c = 0; c < C; ++c) {
        u0[c * 2] = h_status.p[c].u0[0];
        u0[c * 2 + 1] = h_status.p[c].u0[1];
      }
  }

  void slide_only() {
    const size_t smem = sizeof(R) * 2 * T;
    CUDA_TRY(cudaMemsetAsync(d_status.p, 0, C * sizeof(StepStatus), stream));
    slide_kernel<R><<<C, 256, smem, stream>>>(d_plan.p, T, d_iters.p, d_status.p);
    ++launches;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(stream));
  }

  void optimize(const double* x0, int iterations) {
    if (iterations < 1) throw_invalid("optimize_to_convergence: iterations must be >= 1");
    require_ready();
    upload_x0(x0);
    CUDA_TRY(cudaMemsetAsync(d_status.p, 0, C * sizeof(StepStatus), stream));
    CUDA_TRY(cudaMemcpyAsync(d_x0.p, h_x0.p, C * 8 * sizeof(R), cudaMemcpyHostToDevice, stream));
    for (int i = 0; i < iterations; ++i) enqueue_iteration(cfg.noise_mode, false, false, true, false, false);
    CUDA_TRY(cudaMemcpyAsync(h_status.p, d_status.p, C * sizeof(StepStatus), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    const int code = check_status(false);
    if (code != MPPI_OK) throw_status(code);
  }

  void closed_loop(const double* x_init, int iterations, double* u_trace, double* x_trace,
                   size_t flush_bytes, double* ms_out, double* iter_ms_out) {
    if (iterations < 1) throw_invalid("closed_loop: iterations must be >= 1");
    require_ready();
    upload_x0(x_init);
    const bool trace = u_trace || x_trace;
    if (trace) {
      d_utrace.alloc(static_cast<size_t>(iterations) * C * 2);
      d_xtrace.alloc(static_cast<size_t>(iterations + 1) * C * 8);
      CUDA_TRY(cudaMemcpyAsync(d_xtrace.p, h_x0.p, C * 8 * sizeof(R), cudaMemcpyHostToDevice, stream));
      // graphs hold trace pointers: re-capture if the buffers moved
      for (int w = 2; w < 4; ++w)
        if (graph[w]) {
          cudaGraphExecDestroy(graph[w]);
          graph[w] = nullptr;
        }
    }
    if (flush_bytes) d_flush.alloc(flush_bytes);
    CUDA_TRY(cudaMemsetAsync(d_status.p, 0, C * sizeof(StepStatus), stream));
    CUDA_TRY(cudaMemcpyAsync(d_x0.p, h_x0.p, C * 8 * sizeof(R), cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaMemcpyAsync(d_trace_base.p, d_iters.p, C * sizeof(uint64_t), cudaMemcpyDeviceToDevice, stream));
    double total = 0.0;
    const bool per_iter_timing = flush_bytes > 0;
    if (!per_iter_timing && ms_out) CUDA_TRY(cudaEventRecord(ev_it0, stream));
    // The iteration graph without event nodes (slot 3): an event record node
    // between K1 and the tail would cut the tail's programmatic (PDL) edge to
    // K1.  With profiling on (set_profile), the graph that brackets K1 with
    // event nodes (slot 2) runs instead and K1's own durations (the roofline's
    // denominator) accumulate for read_profile.
    const bool k1_events = profile;
    for (int i = 0; i < iterations; ++i) {
      if (per_iter_timing) {
        CUDA_TRY(cudaMemsetAsync(d_flush.p, i & 0xff, flush_bytes, stream));
        CUDA_TRY(cudaEventRecord(ev_it0, stream));
      }
      run_graph(k1_events ? 2 : 3, true, true, trace);
      if (per_iter_timing) {
        CUDA_TRY(cudaEventRecord(ev_it1, stream));
        CUDA_TRY(cudaEventSynchronize(ev_it1));
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, ev_it0, ev_it1));
        total += ms;
        if (iter_ms_out) iter_ms_out[i] = ms;
        float k1 = 0;
        if (k1_events && chunk_hi > chunk_lo && cudaEventElapsedTime(&k1, ev_a, ev_b) == cudaSuccess) {
          prof_ms += k1;
          ++prof_launches;
        } else {
          cudaGetLastError();
        }
        float xm = 0;
        if (k1_events && world > 1 && cudaEventElapsedTime(&xm, ev_x0, ev_x1) == cudaSuccess) {
          prof_x_ms += xm;
          ++prof_x_n;
        } else {
          cudaGetLastError();
        }
      }
    }
    if (!per_iter_timing && ms_out) {
      CUDA_TRY(cudaEventRecord(ev_it1, stream));
      CUDA_TRY(cudaEventSynchronize(ev_it1));
      float ms = 0;
      CUDA_TRY(cudaEventElapsedTime(&ms, ev_it0, ev_it1));
      total = ms;
    }
    CUDA_TRY(cudaMemcpyAsync(h_status.p, d_status.p, C * sizeof(StepStatus), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    if (ms_out) *ms_out = total;
    const int code = check_status(true);
    if (code != MPPI_OK) throw_status(code);
    if (trace) {
      std::vector<R> ut(static_cast<size_t>(iterations) * C * 2), xt(static_cast<size_t>(iterations + 1) * C * 8);
      CUDA_TRY(cudaMemcpy(ut.data(), d_utrace.p, ut.size() * sizeof(R), cudaMemcpyDeviceToHost));
      CUDA_TRY(cudaMemcpy(xt.data(), d_xtrace.p, xt.size() * sizeof(R), cudaMemcpyDeviceToHost));
      const int n = state_dim();
      if (u_trace)
        for (size_t i = 0; i < ut.size(); ++i) u_trace[i] = static_cast<double>(ut[i]);
      if (x_trace)
        for (int s = 0; s <= iterations; ++s)
          for (int c = 0; c < C; ++c)
            for (int i = 0; i < n; ++i)
              x_trace[(static_cast<size_t>(s) * C + c) * n + i] = static_cast<double>(xt[(static_cast<size_t>(s) * C + c) * 8 + i]);
    }
  }

  // ------------------------------------------------------------- parity ---
  int effective_mode(bool injected) const { return injected ? static_cast<int>(kInjected) : cfg.noise_mode; }

  void sample_perturbations(uint64_t iteration, double* eps_out, uint8_t* flags_out) {
    if (cfg.noise_mode == MPPI_NOISE_INJECTED && !has_noise) throw_invalid("INJECTED noise: no batch set");
    uint64_t saved = 0;
    CUDA_TRY(cudaMemcpy(&saved, d_iters.p, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(d_iters.p, &iteration, sizeof(uint64_t), cudaMemcpyHostToDevice));
    const size_t n = static_cast<size_t>(K) * 2 * T;
    DevBuf<double> out;
    out.alloc(n);
    const RolloutArgs<R> a = rollout_args();
    const int blocks = (K + 127) / 128;
    switch (cfg.noise_mode) {
      case kInjected: sample_kernel<R, kInjected><<<blocks, 128, 0, stream>>>(a, out.p); break;
      case kRefSplitmix: sample_kernel<R, kRefSplitmix><<<blocks, 128, 0, stream>>>(a, out.p); break;
      default: sample_kernel<R, kPhilox><<<blocks, 128, 0, stream>>>(a, out.p); break;
    }
    ++launches;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(eps_out, out.p, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    CUDA_TRY(cudaMemcpy(d_iters.p, &saved, sizeof(uint64_t), cudaMemcpyHostToDevice));
    if (flags_out)
      for (int k = 0; k < K; ++k) flags_out[k] = k >= zero_start ? 1 : 0;
  }

  void rollout_costs(const double* x0, const double* eps_in, double* costs_out, double* eps_stored_out) {
    if (eps_in) upload_injected(eps_in);
    else if (cfg.noise_mode == MPPI_NOISE_INJECTED && !has_noise) throw_invalid("INJECTED noise: no batch set");
    if (!has_mlp) throw_invalid("vehicle system: model (MLP weights / basis Theta) not set");
    if (!has_map) throw_invalid("vehicle system: costmap not set");
    upload_x0(x0);
    CUDA_TRY(cudaMemsetAsync(d_status.p, 0, C * sizeof(StepStatus), stream));
    CUDA_TRY(cudaMemcpyAsync(d_x0.p, h_x0.p, C * 8 * sizeof(R), cudaMemcpyHostToDevice, stream));
    const int mode = effective_mode(eps_in != nullptr);
    enqueue_rollout(mode);  // (this rank's samples only when sharded)
    CUDA_TRY(cudaMemcpyAsync(costs_out, d_costs.p, K * sizeof(Acc), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    batch_valid = true;
    batch_injected = eps_in != nullptr || cfg.noise_mode == MPPI_NOISE_INJECTED;
    CUDA_TRY(cudaMemcpy(&batch_iteration, d_iters.p, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (eps_stored_out) {
      const size_t n = static_cast<size_t>(K) * 2 * T;
      DevBuf<double> out;
      out.alloc(n);
      const RolloutArgs<R> a = rollout_args();
      const int blocks = (K + 127) / 128;
      switch (mode) {
        case kInjected: materialize_batch_kernel<R, kInjected><<<blocks, 128, 0, stream>>>(a, 1, out.p); break;
        case kRefSplitmix: materialize_batch_kernel<R, kRefSplitmix><<<blocks, 128, 0, stream>>>(a, 1, out.p); break;
        default: materialize_batch_kernel<R, kPhilox><<<blocks, 128, 0, stream>>>(a, 1, out.p); break;
      }
      ++launches;
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaMemcpyAsync(eps_stored_out, out.p, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
      CUDA_TRY(cudaStreamSynchronize(stream));
    }
  }

  // it_weights on caller costs; the softmin runs in double for every
  // precision (Acc, rollout.cuh), as in the fused path.
  int cem_elite() const { return static_cast<int>(std::lround(K * (1.0 - cfg.cem_delta))); }

  void weights(const double* costs, double* w_out, double* rho, double* eta) {
    DevBuf<Acc> d_c;
    d_c.alloc(K);
    d_w.alloc(K);
    CUDA_TRY(cudaMemcpyAsync(d_c.p, costs, K * sizeof(Acc), cudaMemcpyHostToDevice, stream));
    if (cfg.weight_rule == MPPI_WEIGHT_CEM)  // compute_weights (controller.cpp:111-116)
      cem_weights_kernel<1024><<<1, 1024, 0, stream>>>(d_c.p, K, cem_elite(), d_w.p, d_rho_eta.p, d_bad.p, nullptr);
    else
      weights_kernel<Acc, 1024><<<1, 1024, 0, stream>>>(d_c.p, K, cfg.lambda, d_w.p, d_rho_eta.p, d_bad.p);
    ++launches;
    CUDA_TRY(cudaGetLastError());
    int bad = 0;
    Acc re[2];
    CUDA_TRY(cudaMemcpyAsync(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaMemcpyAsync(re, d_rho_eta.p, 2 * sizeof(Acc), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaMemcpyAsync(w_out, d_w.p, K * sizeof(Acc), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    if (bad)
      throw Error(MPPI_ERR_NONFINITE,
                  cfg.weight_rule == MPPI_WEIGHT_CEM ? "cem_weights: non-finite cost" : "it_weights: non-finite cost");
    *rho = re[0];
    *eta = re[1];
  }

  void update_plan(const double* w) {
    if (!batch_valid) throw_invalid("update_plan: no rollout batch");
    d_w.alloc(K);
    CUDA_TRY(cudaMemcpyAsync(d_w.p, w, K * sizeof(Acc), cudaMemcpyHostToDevice, stream));
    uint64_t saved = 0;
    CUDA_TRY(cudaMemcpy(&saved, d_iters.p, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(d_iters.p, &batch_iteration, sizeof(uint64_t), cudaMemcpyHostToDevice));
    const RolloutArgs<R> a = rollout_args();
    const int mode = effective_mode(batch_injected);
    const int blocks = (T + 127) / 128;
    switch (mode) {
      case kInjected: weighted_agg_kernel<R, kInjected><<<blocks, 128, 0, stream>>>(a, d_w.p, d_agg.p); break;
      case kRefSplitmix: weighted_agg_kernel<R, kRefSplitmix><<<blocks, 128, 0, stream>>>(a, d_w.p, d_agg.p); break;
      default: weighted_agg_kernel<R, kPhilox><<<blocks, 128, 0, stream>>>(a, d_w.p, d_agg.p); break;
    }
    ++launches;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(stream));
    CUDA_TRY(cudaMemcpy(d_iters.p, &saved, sizeof(uint64_t), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemsetAsync(d_status.p, 0, C * sizeof(StepStatus), stream));
    enqueue_epilogue(false, false, false, false, false, 1);
    CUDA_TRY(cudaMemcpyAsync(h_status.p, d_status.p, C * sizeof(StepStatus), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    const int code = h_status.p[0].code;
    if (code != MPPI_OK) throw_status(code);
  }

  void rollout_states(const double* x0, int sample, double* out) {
    if (!batch_valid) throw_invalid("rollout_states: no rollout batch");
    if (sample < 0 || sample >= K) throw_invalid("bad sample index");
    upload_x0(x0);
    CUDA_TRY(cudaMemcpyAsync(d_x0.p, h_x0.p, C * 8 * sizeof(R), cudaMemcpyHostToDevice, stream));
    const int n = state_dim();
    d_states.alloc(static_cast<size_t>(T + 1) * n);
    uint64_t saved = 0;
    CUDA_TRY(cudaMemcpy(&saved, d_iters.p, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(d_iters.p, &batch_iteration, sizeof(uint64_t), cudaMemcpyHostToDevice));
    RolloutArgs<R> a = rollout_args();
    if (use_ws || use_tc) {
      // trace the production kernel itself: sample `sample`'s state per step
      a.trace_states = d_states.p;
      a.trace_k = sample;
      a.chunk0 = 0;
      a.chunk_end = n_chunks;
      CUDA_TRY(cudaMemcpyAsync(d_states.p, h_x0.p, 7 * sizeof(R), cudaMemcpyHostToDevice, stream));
      if (use_umma) {
        if constexpr (std::is_same<R, float>::value)
          CUDA_TRY((H == 32 ? launch_rollout_umma<32> : launch_rollout_umma<64>)(
              a, d_umma.p, effective_mode(batch_injected), n_chunks, 1, stream));
      } else if (use_tc) {
        if constexpr (std::is_same<R, float>::value)
          CUDA_TRY((H == 32 ? launch_rollout_tc<32> : launch_rollout_tc<64>)(a, d_tcfrag.p, effective_mode(batch_injected),
                                                                            tc_mt, n_chunks, 1, stream));
      } else {
        launch_ws(a, effective_mode(batch_injected), dim3(n_chunks, 1));
      }
    } else {
      dispatch(effective_mode(batch_injected), [&]<int HH, class Sys, int Mode>() {
        rollout_states_kernel<R, HH, Sys, Mode><<<1, 32, 0, stream>>>(a, holder<HH>(), sample, d_states.p);
      });
    }
    ++launches;
    CUDA_TRY(cudaGetLastError());
    std::vector<R> s(d_states.n);
    CUDA_TRY(cudaMemcpyAsync(s.data(), d_states.p, s.size() * sizeof(R), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    CUDA_TRY(cudaMemcpy(d_iters.p, &saved, sizeof(uint64_t), cudaMemcpyHostToDevice));
    for (size_t i = 0; i < s.size(); ++i) out[i] = static_cast<double>(s[i]);
  }

  // ----------------------------------------------------------- multi-GPU --
  // Validation first, then the commit: a rejected call leaves the handle as it was.
  void validate_shard(int r, int w) const {
    if (w < 1 || r < 0 || r >= w) throw_invalid("set_comm: bad rank/world_size");
    if (w > 1 && C != 1) throw Error(MPPI_ERR_UNSUPPORTED, "set_comm: fleets shard controllers, not samples");
    if (cfg.weight_rule == MPPI_WEIGHT_CEM && w > 1)
      throw Error(MPPI_ERR_UNSUPPORTED, "set_comm: the CEM rule needs every cost on one device");
    if (n_groups % w != 0)
      throw Error(MPPI_ERR_UNSUPPORTED, "set_comm: world_size must divide the exchange group count (" +
                                            std::to_string(n_groups) + ")");
  }
  void apply_shard(int r, int w, int mode) {
    rank = r;
    world = w;
    exchange_mode = w > 1 ? mode : static_cast<int>(kExNone);
    group_lo = r * (n_groups / w);
    group_hi = (r + 1) * (n_groups / w);
    chunk_lo = group_first_chunk(group_lo, n_chunks, n_groups);
    chunk_hi = group_first_chunk(group_hi, n_chunks, n_groups);
    invalidate_graphs();
  }
  void set_comm(int r, int w, const unsigned char id[128]) override {
    validate_shard(r, w);
    ncclComm_t fresh = nullptr;
    if (w > 1) {
      if (!id) throw_invalid("set_comm: null id");
      ncclUniqueId uid;
      static_assert(sizeof(uid) == 128, "ncclUniqueId must be 128 bytes");
      std::memcpy(&uid, id, 128);
      NCCL_TRY(nccl().CommInitRank(&fresh, w, uid, r));
    }
    if (comm) nccl().CommDestroy(comm);
    comm = fresh;
    leave_local_group();
    apply_shard(r, w, kExNccl);
  }
  // In-process sharding over `peers` (this handle is peers[r]): the exchange
  // copies the other ranks' group rows from their buffers.
  void set_comm_local_base(const std::vector<HandleBase*>& base, int r) override {
    std::vector<Handle<R>*> peers;
    for (HandleBase* b : base) {
      auto* p = dynamic_cast<Handle<R>*>(b);
      if (!p) throw_invalid("set_comm_local: every handle of a group needs the same precision");
      peers.push_back(p);
    }
    set_comm_local(peers, r);
  }
  void set_comm_local(const std::vector<Handle<R>*>& peers, int r) {
    const int w = static_cast<int>(peers.size());
    validate_shard(r, w);
    for (const Handle<R>* p : peers) {
      if (!p) throw_invalid("set_comm_local: null handle");
      if (p->K != K || p->T != T || p->H != H || p->C != C || p->n_chunks != n_chunks || p->n_groups != n_groups ||
          p->cfg.seed != cfg.seed || p->cfg.noise_mode != cfg.noise_mode || p->cfg.system != cfg.system)
        throw_invalid("set_comm_local: every handle of a group needs the same configuration");
    }
    for (const Handle<R>* p : peers)
      if (p->device != device) {
        cudaDeviceEnablePeerAccess(p->device, 0);  // best effort: the copies stage through the host otherwise
        cudaGetLastError();
      }
    if (comm) {
      nccl().CommDestroy(comm);
      comm = nullptr;
    }
    leave_local_group();
    local_peers = peers;
    apply_shard(r, w, kExLocal);
  }
  void leave_local_group() {
    for (Handle<R>* p : local_peers)
      if (p && p != this)
        for (auto& q : p->local_peers)
          if (q == this) q = nullptr;
    local_peers.clear();
  }
  // A step of a local group in phases, driven by mppi_gpu_step_local
  // (abi.cpp): every rank's front (K1 + group merge), a host sync, then every
  // rank's back (exchange + tail) — no kernel ever waits on another rank's.
  void local_front(const double* x0) override {
    require_ready();
    if (exchange_mode != kExLocal) throw_invalid("step_local: handle is not in a local group");
    upload_x0(x0);
    CUDA_TRY(cudaMemsetAsync(d_status.p, 0, C * sizeof(StepStatus), stream));
    CUDA_TRY(cudaMemcpyAsync(d_x0.p, h_x0.p, C * 8 * sizeof(R), cudaMemcpyHostToDevice, stream));
    enqueue_front(cfg.noise_mode, false);
  }
  void local_back(bool slide) override {
    enqueue_back(/*events=*/false, slide, /*increment=*/slide, false, false);
    CUDA_TRY(cudaMemcpyAsync(h_status.p, d_status.p, C * sizeof(StepStatus), cudaMemcpyDeviceToHost, stream));
  }
  void local_finish(double* u0) override {
    CUDA_TRY(cudaStreamSynchronize(stream));
    const int code = check_status(true);
    if (code != MPPI_OK) throw_status(code);
    if (u0)
      for (int c = 0; c < C; ++c) {
        u0[c * 2] = h_status.p[c].u0[0];
        u0[c * 2 + 1] = h_status.p[c].u0[1];
      }
  }
  void sync_stream() override { CUDA_TRY(cudaStreamSynchronize(stream)); }
  void shard_info(int* out) const override {
    const int v[8] = {rank, world, n_chunks, n_groups, chunk_lo, chunk_hi, group_lo, group_hi};
    for (int i = 0; i < 8; ++i) out[i] = v[i];
  }
  void read_exchange_profile(double* ms, uint64_t* n, bool reset) override {
    if (ms) *ms = prof_x_ms;
    if (n) *n = prof_x_n;
    if (reset) {
      prof_x_ms = 0;
      prof_x_n = 0;
    }
  }
};

}  // namespace mppi_host
