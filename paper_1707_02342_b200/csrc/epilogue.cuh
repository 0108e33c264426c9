// epilogue.cuh — K2: merge chunk partials, Savitzky-Golay, plan update,
// u0 = clamp(U'[0]), slide, ++iteration (+ optional device plant step).
//
// One CTA per controller.  Implements the tail of mpc_step
// (controller.cpp:137-146): it_weights' normaliser from the chunk partials
// (rho = min_c rho_c, eta = sum_c exp(-(rho_c - rho)/lambda) eta_c, merged in
// global chunk order), agg = num / eta, sg_smooth (smoothing.cpp:48-65) with
// mirror padding, U' = U + agg with the ControlPlan finiteness check
// (types.hpp:79-83), then clamp / slide.
#pragma once

#include "model.cuh"
#include "rollout.cuh"

namespace mppi_dev {

struct StepStatus {
  int code;        // MPPI_OK or an MPPI_ERR_* code (sticky until cleared)
  int pad;
  double u0[2];    // clamp(U'[0])
  double x[8];     // state after the device plant (closed loop)
  unsigned long long iteration;
  // host mirror only: bumped after every other field of a step is published
  // (the host waits on it instead of a stream synchronisation, handle.cuh)
  unsigned long long seq;
};

constexpr int kMaxSgWindow = 63;

template <class R>
struct EpilogueArgs {
  int T, n_chunks, partial_stride;
  int tile_rows;                 // partial rows staged per shared-memory tile
  long long partials_ctrl_stride;
  double lambda;
  R lo0, lo1, hi0, hi1;
  int sg_window;
  double sg[kMaxSgWindow];
  int slide, increment, plant;
  const Acc* partials;   // [C][chunks][stride] (merge mode) or nullptr
  const Acc* agg_in;     // [T][2] (caller-weights mode, controller 0) or nullptr
  R* plan;               // [C][T][2]
  R* x0;                 // [C][8] (plant mode: advanced in place)
  uint64_t* iters;       // [C]
  StepStatus* status;    // [C]
  StepStatus* status_host;  // [C] mapped pinned host mirror written directly (tensor-core tail), or nullptr
  R* u_trace;            // [iter][C][2] or nullptr
  R* x_trace;            // [iter+1][C][8] or nullptr
  const uint64_t* trace_base;  // [C] iteration at trace start
  int n_ctrl;
  SystemArgs<R> sys;
};

// reflect_index (smoothing.cpp:37-44)
__device__ __forceinline__ int reflect_index(int i, int n) {
  if (n == 1) return 0;
  while (i < 0 || i >= n) {
    if (i < 0) i = -i;
    if (i >= n) i = 2 * (n - 1) - i;
  }
  return i;
}

// Dynamic smem: agg (2T doubles) | chunk scales (n_chunks doubles) | a tile
// of tile_rows partial rows (tile_rows x partial_stride doubles) | U' (2T R) |
// MLP scratch (2H R) | the plant's MLP weights (MlpParams<R,H>, plant only).
// The partial rows are merged tile by tile: every value of a tile is loaded
// at once into shared memory (one L2 round trip per tile), then each thread
// accumulates its elements over the rows in ascending order.
template <class R, int H>
__host__ __device__ constexpr size_t epilogue_smem_bytes(int T, int n_chunks, int tile_rows, int stride, bool plant) {
  return sizeof(Acc) * (2 * T + n_chunks + static_cast<size_t>(tile_rows) * stride) + sizeof(R) * (2 * T + 2 * H) +
         (plant ? sizeof(MlpParams<R, H>) + 16 : 0);
}
// The epilogue of one controller, executed by one CTA of BLOCK threads
// (epilogue_kernel, or CTA 0 of the cooperative tensor-core K1).  `w` points
// to the model weights (the plant step), `smem_raw` to epilogue_smem_bytes of
// dynamic shared memory.
template <class R, int H, class Sys, int BLOCK>
__device__ __forceinline__ void epilogue_body(const EpilogueArgs<R>& a, const MlpParams<R, H>* w_src, int ctrl,
                                              unsigned char* smem_raw) {
  const int T = a.T;
  const int n_rows = a.partials ? a.n_chunks : 0;
  Acc* s_agg = reinterpret_cast<Acc*>(smem_raw);
  Acc* s_scale = s_agg + 2 * T;
  Acc* s_tile = s_scale + n_rows;
  R* s_new = reinterpret_cast<R*>(s_tile + (a.partials ? static_cast<size_t>(a.tile_rows) * a.partial_stride : 0));
  R* s_mlp = s_new + 2 * T;
  MlpParams<R, H>* s_w = reinterpret_cast<MlpParams<R, H>*>(
      (reinterpret_cast<uintptr_t>(s_mlp + 2 * H) + 15) & ~uintptr_t(15));
  __shared__ Acc s_red[BLOCK / 32];
  __shared__ int s_bad;
  __shared__ R s_u[2];
  __shared__ Acc s_eta;
  StepStatus* st = a.status + ctrl;
  if (st->code != 0) return;  // sticky abort: a previous stage failed
  R* plan = a.plan + static_cast<size_t>(ctrl) * 2 * T;
  if constexpr (Sys::kMlp) {
    if (a.plant) {  // stage the plant's weights (overlaps the merge)
      const float4* src = reinterpret_cast<const float4*>(w_src);
      float4* dst = reinterpret_cast<float4*>(s_w);
      for (int i = threadIdx.x; i < static_cast<int>(sizeof(MlpParams<R, H>) / 16); i += BLOCK) dst[i] = src[i];
    }
  }

  if (a.partials) {
    const Acc* P = a.partials + static_cast<size_t>(ctrl) * a.partials_ctrl_stride;
    const int stride = a.partial_stride;
    // any non-finite sample cost -> it_weights throws (weights.cpp:12)
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    Acc m = INFINITY;
    for (int c = threadIdx.x; c < n_rows; c += BLOCK) {
      const Acc* pc = P + static_cast<size_t>(c) * stride;
      if (pc[2] != 0.0) s_bad = 1;
      const Acc r = pc[0];
      m = (r < m) ? r : m;
      s_scale[c] = r;
    }
    const Acc rho = block_min<Acc, BLOCK>(m, s_red);
    if (s_bad) {
      if (threadIdx.x == 0) st->code = 2;  // MPPI_ERR_NONFINITE
      return;
    }
    for (int c = threadIdx.x; c < n_rows; c += BLOCK) s_scale[c] = exp(-(s_scale[c] - rho) / a.lambda);
    // per-thread accumulators: element 1 (eta) and the 2T numerators
    constexpr int kMaxPer = (2 * 4096 + kPartialHeader + BLOCK - 1) / BLOCK;  // T <= 4096
    Acc acc[kMaxPer];
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q) acc[q] = 0.0;
    for (int r0 = 0; r0 < n_rows; r0 += a.tile_rows) {
      const int nr = min(a.tile_rows, n_rows - r0);
      __syncthreads();  // previous tile consumed (and s_scale written)
      const Acc* src = P + static_cast<size_t>(r0) * stride;
      for (int f = threadIdx.x; f < nr * stride; f += BLOCK) s_tile[f] = src[f];
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kMaxPer; ++q) {
        const int i = threadIdx.x + q * BLOCK;
        if (i < stride && (i == 1 || i >= kPartialHeader))
          for (int r = 0; r < nr; ++r) acc[q] = fma(s_scale[r0 + r], s_tile[r * stride + i], acc[q]);
      }
    }
    if (threadIdx.x == 1) s_eta = acc[0];
    __syncthreads();
    const Acc eta = s_eta;
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q) {
      const int i = threadIdx.x + q * BLOCK;
      if (i >= kPartialHeader && i < stride) s_agg[i - kPartialHeader] = acc[q] / eta;
    }
  } else {
    for (int i = threadIdx.x; i < 2 * T; i += BLOCK) s_agg[i] = a.agg_in[i];
  }
  // SG smoothing of the aggregated perturbation, then U' = U + agg.
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  const int half = a.sg_window / 2;
  for (int i = threadIdx.x; i < 2 * T; i += BLOCK) {
    const int t = i >> 1, c = i & 1;
    Acc v;
    if (a.sg_window > 0) {
      Acc acc = 0.0;
      for (int j = -half; j <= half; ++j)
        acc = __dadd_rn(acc, __dmul_rn(a.sg[j + half], s_agg[reflect_index(t + j, T) * 2 + c]));
      v = acc;
    } else {
      v = s_agg[i];
    }
    // U' = U + SG(agg) in double, rounded once to R
    const R nv = static_cast<R>(__dadd_rn(static_cast<Acc>(plan[i]), v));
    if (!isfinite_r(nv)) s_bad = 1;
    s_new[i] = nv;
  }
  __syncthreads();
  if (s_bad) {  // ControlPlan rejects non-finite plans (types.hpp:79-83)
    if (threadIdx.x == 0) st->code = 1;  // MPPI_ERR_INVALID_ARGUMENT
    return;
  }
  if (threadIdx.x == 0) {
    s_u[0] = clamp_r(s_new[0], a.lo0, a.hi0);
    s_u[1] = clamp_r(s_new[1], a.lo1, a.hi1);
    st->u0[0] = static_cast<double>(s_u[0]);
    st->u0[1] = static_cast<double>(s_u[1]);
  }
  // slide (controller.cpp:143-145) or plain replacement
  for (int i = threadIdx.x; i < 2 * T; i += BLOCK) {
    if (a.slide) plan[i] = (i + 2 < 2 * T) ? s_new[i + 2] : R(0);
    else plan[i] = s_new[i];
  }
  __syncthreads();
  uint64_t it = a.iters[ctrl];
  if (a.increment) it += 1;
  if (a.u_trace && threadIdx.x == 0) {
    const uint64_t idx = it - 1 - a.trace_base[ctrl];
    a.u_trace[(idx * a.n_ctrl + ctrl) * 2] = s_u[0];
    a.u_trace[(idx * a.n_ctrl + ctrl) * 2 + 1] = s_u[1];
  }
  if (a.plant) {
    // Device plant: the same model stepped with the executed (clamped) input.
    R* x = a.x0 + static_cast<size_t>(ctrl) * 8;
    if constexpr (Sys::kMlp) {
      // warp-parallel MLP step: thread j owns hidden unit j
      const MlpParams<R, H>& w = *s_w;
      const R in[6] = {x[3], x[4], x[5], x[6], s_u[0], s_u[1]};
      R* h1 = s_mlp;
      R* h2 = s_mlp + H;
      __shared__ R s_d[4];
      if (threadIdx.x < H) {
        const int j = threadIdx.x;
        R acc = w.b1[j];
        for (int i = 0; i < 6; ++i) acc = fma_r(w.w1t[i][j], in[i], acc);
        h1[j] = tanh_r(acc);
      }
      __syncthreads();
      if (threadIdx.x < H) {
        const int j = threadIdx.x;
        R acc = w.b2[j];
        for (int i = 0; i < H; ++i) acc = fma_r(w.w2t[i][j], h1[i], acc);
        h2[j] = tanh_r(acc);
      }
      __syncthreads();
      if (threadIdx.x < 4) {
        const int o = threadIdx.x;
        R acc = w.b3[o];
        for (int i = 0; i < H; ++i) acc = fma_r(w.w3t[i][o], h2[i], acc);
        s_d[o] = acc;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        R xs[7];
        for (int i = 0; i < 7; ++i) xs[i] = x[i];
        advance_split<R>(xs, s_d, a.sys.dt);
        for (int i = 0; i < 7; ++i) x[i] = xs[i];
      }
    } else {
      if (threadIdx.x == 0) {  // quadratic fixture / basis-function model: one thread
        R xs[7];
        for (int i = 0; i < 7; ++i) xs[i] = (i < Sys::kStateDim) ? x[i] : R(0);
        Sys::step(xs, s_u[0], s_u[1], *w_src, a.sys);
        for (int i = 0; i < Sys::kStateDim; ++i) x[i] = xs[i];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < 8; ++i) st->x[i] = static_cast<double>(x[i]);
      if (a.x_trace) {
        const uint64_t idx = it - a.trace_base[ctrl];
        for (int i = 0; i < 8; ++i) a.x_trace[(idx * a.n_ctrl + ctrl) * 8 + i] = x[i];
      }
    }
  }
  if (threadIdx.x == 0) {
    a.iters[ctrl] = it;
    st->iteration = it;
  }
}

template <class R, int H, class Sys, int BLOCK>
__global__ void __launch_bounds__(BLOCK) epilogue_kernel(const __grid_constant__ EpilogueArgs<R> a,
                                                         const __grid_constant__ WeightHolder<R, H> wh) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  epilogue_body<R, H, Sys, BLOCK>(a, &wh.get(), blockIdx.x, smem_raw);
}

// The slide half of mpc_step on its own (controller.cpp:143-146).
template <class R>
__global__ void slide_kernel(R* plan, int T, uint64_t* iters, StepStatus* status) {
  const int ctrl = blockIdx.x;
  if (status[ctrl].code != 0) return;
  R* p = plan + static_cast<size_t>(ctrl) * 2 * T;
  // in-place shift: read everything first
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* s = reinterpret_cast<R*>(smem_raw);
  for (int i = threadIdx.x; i < 2 * T; i += blockDim.x) s[i] = p[i];
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * T; i += blockDim.x) p[i] = (i + 2 < 2 * T) ? s[i + 2] : R(0);
  if (threadIdx.x == 0) {
    iters[ctrl] += 1;
    status[ctrl].iteration = iters[ctrl];
  }
}

// it_weights (weights.cpp:8-25) on caller costs (parity entry point); the
// softmin runs in double for every precision (see Acc in rollout.cuh).
template <class R, int BLOCK>
__global__ void __launch_bounds__(BLOCK) weights_kernel(const R* __restrict__ S, int K, R lambda,
                                                        R* w, R* rho_eta, int* bad_out) {
  __shared__ R s_red[BLOCK / 32];
  int bad = 0;
  R m = R(INFINITY);
  for (int k = threadIdx.x; k < K; k += BLOCK) {
    const R c = S[k];
    if (!isfinite_r(c)) bad = 1;
    m = (c < m) ? c : m;
  }
  bad = __syncthreads_or(bad);
  if (bad) {
    if (threadIdx.x == 0) *bad_out = 1;
    return;
  }
  const R rho = block_min<R, BLOCK>(m, s_red);
  R e = R(0);
  for (int k = threadIdx.x; k < K; k += BLOCK) {
    const R v = exp_r(div_r(-sub_rn(S[k], rho), lambda));
    w[k] = v;
    e = e + v;
  }
  const R eta = block_sum<R, BLOCK>(e, s_red);
  for (int k = threadIdx.x; k < K; k += BLOCK) w[k] = div_r(w[k], eta);
  if (threadIdx.x == 0) {
    rho_eta[0] = rho;
    rho_eta[1] = eta;
    *bad_out = 0;
  }
}

// Fleet maps: map_c[cell] = clamp(base[cell] + sigma * N(0,1), -2.5, 2.5)
// with N from the reference counter stream keyed (seed, stream, c, cell).
template <class R>
__global__ void perturb_map_kernel(const R* __restrict__ base, size_t cells, int ctrl, double sigma,
                                   uint64_t seed, R* out) {
  const uint64_t prefix = ref_hash_prefix(seed, static_cast<uint64_t>(ctrl));
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cells;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    double z0, z1;
    ref_normal_pair(prefix, i, 0x6d6170ull /* "map" */, z0, z1);
    double v = static_cast<double>(base[i]) + sigma * z0;
    v = v < -2.5 ? -2.5 : (v > 2.5 ? 2.5 : v);
    out[i] = static_cast<R>(v);
  }
}

// Reference-layout batch generation for mppi_gpu_sample_perturbations.
template <class R, int Mode>
__global__ void sample_kernel(const __grid_constant__ RolloutArgs<R> a, double* eps_out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.K) return;
  NoiseStream<R, Mode> ns = make_noise<R, Mode>(a, 0, k);
  for (int t = 0; t < a.T; ++t) {
    R e0, e1;
    ns.eps(t, e0, e1);
    eps_out[(static_cast<size_t>(k) * 2 + 0) * a.T + t] = static_cast<double>(e0);
    eps_out[(static_cast<size_t>(k) * 2 + 1) * a.T + t] = static_cast<double>(e1);
  }
}

}  // namespace mppi_dev
