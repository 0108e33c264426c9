// abi.cpp — the extern "C" surface of include/mppi_gpu.h.  Every entry point
// converts exceptions to MPPI_* status codes (mppi_gpu_last_error() holds the
// message) and forwards to the precision-specific handle.
#include <cuda_runtime_api.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstring>
#include <memory>

#include "../../include/mppi_gpu.h"
#include "errors.hpp"
#include "handle_iface.hpp"
#include "nccl_api.hpp"
#include "shard.hpp"

#include <utility>
#include <vector>

using namespace mppi_host;

namespace {

template <class F>
int with_handle(mppi_gpu_handle* h, F&& f) {
  return guard([&] {
    if (!h || !h->impl) throw_invalid("null handle");
    CUDA_TRY(cudaSetDevice(h->impl->device_index()));
    f(*h->impl);
  });
}

// NVTX3 range around a hot-path entry point (SURVEY §5 tracing plan): the
// iteration itself is one graph replay, so the range brackets its launch and
// host-side wait; nsys / ncu --nvtx attribute the kernels to it.  A branch on
// a null pointer when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
template <class F>
int with_handle_traced(const char* name, mppi_gpu_handle* h, F&& f) {
  NvtxRange r(name);
  return with_handle(h, std::forward<F>(f));
}

}  // namespace

// ================================================================ C ABI =====
extern "C" {

int mppi_gpu_abi_version(void) { return MPPI_GPU_ABI_VERSION; }
size_t mppi_gpu_config_sizeof(void) { return sizeof(mppi_gpu_config); }
const char* mppi_gpu_last_error(void) { return mppi_host::last_error().c_str(); }

void mppi_gpu_config_init(mppi_gpu_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->samples = 1200;
  c->horizon_steps = 80;
  c->dt = 0.025;
  c->sigma_diag[0] = 0.0306;
  c->sigma_diag[1] = 0.0506;
  c->lambda = 12.5;
  c->gamma = 0.1;
  c->explore_fraction = 0.01;
  c->seed = 0;
  c->bounds_lower[0] = c->bounds_lower[1] = -1.0;
  c->bounds_upper[0] = c->bounds_upper[1] = 1.0;
  c->sg_window = 9;
  c->sg_degree = 3;
  c->weight_rule = MPPI_WEIGHT_IT;
  c->cem_delta = 0.8;
  c->with_terminal = 1;
  c->noise_mode = MPPI_NOISE_PHILOX;
  c->precision = MPPI_FP32;
  c->system = MPPI_SYSTEM_VEHICLE_MLP;
  c->mlp_hidden = 32;
  c->n_controllers = 1;
  c->device = 0;
  c->quad_cost_scale = 1.0;
  c->cost.alpha_track = 100.0;
  c->cost.alpha_speed = 4.25;
  c->cost.alpha_stab = 10.0;
  c->cost.v_des = 6.0;
  c->cost.impulse = 10000.0;
  c->cost.decay = 0.9;
  c->cost.boundary_threshold = 0.99;
  c->cost.slip_limit = 0.75;
  c->cost.crash_penalty = 0.0;
  c->cost.crash_threshold = 1.0;
  c->cost.roll_limit = INFINITY;
  c->controller_offset = 0;
}

int mppi_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int mppi_gpu_create(const mppi_gpu_config* cfg, mppi_gpu_handle** out) {
  return guard([&] {
    if (!cfg || !out) throw_invalid("mppi_gpu_create: null argument");
    *out = nullptr;
    auto h = std::make_unique<mppi_gpu_handle>();
    if (cfg->precision == MPPI_FP64) h->impl.reset(make_handle_f64(*cfg));
    else if (cfg->precision == MPPI_FP32) h->impl.reset(make_handle_f32(*cfg));
    else throw_invalid("precision");
    *out = h.release();
  });
}
int mppi_gpu_destroy(mppi_gpu_handle* h) {
  return guard([&] { delete h; });
}

int mppi_gpu_set_dynamics_mlp(mppi_gpu_handle* h, int hidden, const double* w1, const double* b1,
                              const double* w2, const double* b2, const double* w3, const double* b3) {
  return with_handle(h, [&](auto& x) {
    if (!w1 || !b1 || !w2 || !b2 || !w3 || !b3) throw_invalid("set_dynamics_mlp: null array");
    x.set_mlp(hidden, w1, b1, w2, b2, w3, b3);
  });
}
int mppi_gpu_set_dynamics_basis(mppi_gpu_handle* h, const double* theta) {
  return with_handle(h, [&](auto& x) {
    if (!theta) throw_invalid("set_dynamics_basis: null theta");
    x.set_basis(theta);
  });
}
int mppi_gpu_set_dynamics_bicycle(mppi_gpu_handle* h, const mppi_bicycle_params* p) {
  return with_handle(h, [&](auto& x) {
    if (!p) throw_invalid("set_dynamics_bicycle: null params");
    x.set_bicycle(*p);
  });
}
int mppi_gpu_set_costmap(mppi_gpu_handle* h, int controller, const double* values, int width,
                         int height, double x0, double y0, double resolution) {
  return with_handle(h, [&](auto& x) {
    if (!values) throw_invalid("set_costmap: null values");
    x.set_map_f64(controller, values, width, height, x0, y0, resolution);
  });
}
int mppi_gpu_set_costmap_f32(mppi_gpu_handle* h, int controller, const float* values, int width,
                             int height, double x0, double y0, double resolution) {
  return with_handle(h, [&](auto& x) {
    if (!values) throw_invalid("set_costmap: null values");
    x.set_map_f32(controller, values, width, height, x0, y0, resolution);
  });
}
int mppi_gpu_perturb_fleet_costmaps(mppi_gpu_handle* h, double sigma, uint64_t seed) {
  return with_handle(h, [&](auto& x) { x.perturb_fleet(sigma, seed); });
}
int mppi_gpu_get_costmap_f32(mppi_gpu_handle* h, int controller, float* values_out) {
  return with_handle(h, [&](auto& x) {
    if (!values_out) throw_invalid("get_costmap: null");
    x.get_map_f32(controller, values_out);
  });
}
int mppi_gpu_set_plan(mppi_gpu_handle* h, int controller, const double* U) {
  return with_handle(h, [&](auto& x) {
    if (!U) throw_invalid("set_plan: null");
    x.set_plan(controller, U);
  });
}
int mppi_gpu_get_plan(mppi_gpu_handle* h, int controller, double* U) {
  return with_handle(h, [&](auto& x) {
    if (!U) throw_invalid("get_plan: null");
    x.get_plan(controller, U);
  });
}
int mppi_gpu_set_iteration(mppi_gpu_handle* h, int controller, uint64_t iteration) {
  return with_handle(h, [&](auto& x) { x.set_iteration(controller, iteration); });
}
int mppi_gpu_get_iteration(mppi_gpu_handle* h, int controller, uint64_t* iteration) {
  return with_handle(h, [&](auto& x) {
    if (!iteration) throw_invalid("get_iteration: null");
    *iteration = x.get_iteration(controller);
  });
}
int mppi_gpu_set_seed(mppi_gpu_handle* h, int controller, uint64_t seed) {
  return with_handle(h, [&](auto& x) { x.set_seed(controller, seed); });
}
int mppi_gpu_set_noise(mppi_gpu_handle* h, const double* eps) {
  return with_handle(h, [&](auto& x) {
    if (!eps) throw_invalid("set_noise: null");
    if (x.config().noise_mode != MPPI_NOISE_INJECTED) throw_invalid("set_noise: handle is not in INJECTED mode");
    x.set_noise(eps);
  });
}
int mppi_gpu_compute_control(mppi_gpu_handle* h, const double* x0, double* u0_out) {
  return with_handle_traced("mppi_gpu_compute_control", h, [&](auto& x) {
    if (!x0) throw_invalid("compute_control: null x0");
    x.step(x0, u0_out, false);
  });
}
int mppi_gpu_slide(mppi_gpu_handle* h) {
  return with_handle(h, [&](auto& x) { x.slide_only(); });
}
int mppi_gpu_step(mppi_gpu_handle* h, const double* x0, double* u0_out) {
  return with_handle_traced("mppi_gpu_step", h, [&](auto& x) {
    if (!x0) throw_invalid("step: null x0");
    x.step(x0, u0_out, true);
  });
}
int mppi_gpu_optimize(mppi_gpu_handle* h, const double* x0, int iterations) {
  return with_handle_traced("mppi_gpu_optimize", h, [&](auto& x) {
    if (!x0) throw_invalid("optimize: null x0");
    x.optimize(x0, iterations);
  });
}
int mppi_gpu_closed_loop(mppi_gpu_handle* h, const double* x_init, int iterations, double* u_trace,
                         double* x_trace) {
  return with_handle_traced("mppi_gpu_closed_loop", h, [&](auto& x) {
    if (!x_init) throw_invalid("closed_loop: null x_init");
    x.closed_loop(x_init, iterations, u_trace, x_trace, 0, nullptr, nullptr);
  });
}
int mppi_gpu_closed_loop_timed(mppi_gpu_handle* h, const double* x_init, int iterations,
                               uint64_t flush_l2_bytes, double* device_ms_out, double* iter_ms_out) {
  return with_handle_traced("mppi_gpu_closed_loop_timed", h, [&](auto& x) {
    if (!x_init) throw_invalid("closed_loop: null x_init");
    if (iter_ms_out && flush_l2_bytes == 0) throw_invalid("closed_loop_timed: per-iteration times need flush mode");
    x.closed_loop(x_init, iterations, nullptr, nullptr, static_cast<size_t>(flush_l2_bytes), device_ms_out,
                  iter_ms_out);
  });
}
int mppi_gpu_sample_perturbations(mppi_gpu_handle* h, uint64_t iteration, double* eps_out,
                                  uint8_t* flags_out) {
  return with_handle(h, [&](auto& x) {
    if (!eps_out) throw_invalid("sample_perturbations: null");
    x.sample_perturbations(iteration, eps_out, flags_out);
  });
}
int mppi_gpu_rollout_costs(mppi_gpu_handle* h, const double* x0, const double* eps_in,
                           double* costs_out, double* eps_stored_out) {
  return with_handle_traced("mppi_gpu_rollout_costs", h, [&](auto& x) {
    if (!x0 || !costs_out) throw_invalid("rollout_costs: null");
    if (x.controllers() != 1) throw Error(MPPI_ERR_UNSUPPORTED, "parity entry points use single-controller handles");
    x.rollout_costs(x0, eps_in, costs_out, eps_stored_out);
  });
}
int mppi_gpu_weights(mppi_gpu_handle* h, const double* costs, double* w_out, double* rho, double* eta) {
  return with_handle_traced("mppi_gpu_weights", h, [&](auto& x) {
    if (!costs || !w_out || !rho || !eta) throw_invalid("weights: null");
    x.weights(costs, w_out, rho, eta);
  });
}
int mppi_gpu_update_plan(mppi_gpu_handle* h, const double* weights) {
  return with_handle_traced("mppi_gpu_update_plan", h, [&](auto& x) {
    if (!weights) throw_invalid("update_plan: null");
    x.update_plan(weights);
  });
}
int mppi_gpu_rollout_states(mppi_gpu_handle* h, const double* x0, int sample, double* states_out) {
  return with_handle(h, [&](auto& x) {
    if (!x0 || !states_out) throw_invalid("rollout_states: null");
    x.rollout_states(x0, sample, states_out);
  });
}
int mppi_gpu_nccl_unique_id(unsigned char id_out[128]) {
  return guard([&] {
    if (!id_out) throw_invalid("nccl_unique_id: null");
    ncclUniqueId uid;
    NCCL_TRY(nccl().GetUniqueId(&uid));
    std::memcpy(id_out, &uid, 128);
  });
}
int mppi_gpu_set_comm(mppi_gpu_handle* h, int rank, int world_size, const unsigned char id[128]) {
  return with_handle(h, [&](auto& x) {
    x.set_comm(rank, world_size, id);
  });
}
int mppi_gpu_set_comm_local(mppi_gpu_handle** handles, int n) {
  return guard([&] {
    if (!handles || n < 1) throw_invalid("set_comm_local: need at least one handle");
    std::vector<HandleBase*> peers;
    for (int i = 0; i < n; ++i) {
      if (!handles[i] || !handles[i]->impl) throw_invalid("set_comm_local: null handle");
      for (int j = 0; j < i; ++j)
        if (handles[j] == handles[i]) throw_invalid("set_comm_local: a handle appears twice");
      peers.push_back(handles[i]->impl.get());
    }
    // (rank 0 checks the whole group, so a mismatch is rejected before any commit)
    for (int r = 0; r < n; ++r) {
      CUDA_TRY(cudaSetDevice(peers[r]->device_index()));
      peers[r]->set_comm_local_base(peers, r);
    }
  });
}
int mppi_gpu_step_local(mppi_gpu_handle** handles, int n, const double* x0, double* u0_out) {
  return guard([&] {
    NvtxRange range("mppi_gpu_step_local");
    if (!handles || n < 1 || !x0) throw_invalid("step_local: null argument");
    for (int i = 0; i < n; ++i)
      if (!handles[i] || !handles[i]->impl) throw_invalid("step_local: null handle");
    auto on = [&](int r) -> HandleBase& {
      HandleBase& x = *handles[r]->impl;
      CUDA_TRY(cudaSetDevice(x.device_index()));
      return x;
    };
    // fronts, a host sync of every rank, then backs: no kernel of one rank
    // ever waits for another rank's
    for (int r = 0; r < n; ++r) on(r).local_front(x0);
    for (int r = 0; r < n; ++r) on(r).sync_stream();
    for (int r = 0; r < n; ++r) on(r).local_back(true);
    for (int r = 0; r < n; ++r) on(r).local_finish(u0_out ? u0_out + 2 * r : nullptr);
  });
}
int mppi_gpu_shard_info(mppi_gpu_handle* h, int32_t out[8]) {
  return with_handle(h, [&](auto& x) {
    if (!out) throw_invalid("shard_info: null");
    int v[8];
    x.shard_info(v);
    for (int i = 0; i < 8; ++i) out[i] = v[i];
  });
}
int mppi_gpu_shard_plan(int samples, int chunk_samples, int rank, int world_size, int32_t out[8]) {
  return guard([&] {
    if (!out) throw_invalid("shard_plan: null");
    if (samples < 1 || chunk_samples < 1) throw_invalid("shard_plan: samples and chunk_samples must be >= 1");
    if (world_size < 1 || rank < 0 || rank >= world_size) throw_invalid("shard_plan: bad rank/world_size");
    const int n_chunks = (samples + chunk_samples - 1) / chunk_samples;
    const int n_groups = mppi_dev::group_count(n_chunks);
    if (n_groups % world_size != 0)
      throw Error(MPPI_ERR_UNSUPPORTED, "shard_plan: world_size must divide the exchange group count");
    const int g_lo = rank * (n_groups / world_size), g_hi = (rank + 1) * (n_groups / world_size);
    const int v[8] = {rank, world_size, n_chunks, n_groups, mppi_dev::group_first_chunk(g_lo, n_chunks, n_groups),
                      mppi_dev::group_first_chunk(g_hi, n_chunks, n_groups), g_lo, g_hi};
    for (int i = 0; i < 8; ++i) out[i] = v[i];
  });
}
int mppi_gpu_profile_read_exchange(mppi_gpu_handle* h, double* exchange_ms, uint64_t* exchanges, int reset) {
  return with_handle(h, [&](auto& x) { x.read_exchange_profile(exchange_ms, exchanges, reset != 0); });
}
int mppi_gpu_get_stream(mppi_gpu_handle* h, void** stream_out) {
  return with_handle(h, [&](auto& x) {
    if (!stream_out) throw_invalid("get_stream: null");
    *stream_out = x.stream_ptr();
  });
}
int mppi_gpu_launch_count(mppi_gpu_handle* h, uint64_t* count_out) {
  return with_handle(h, [&](auto& x) {
    if (!count_out) throw_invalid("launch_count: null");
    *count_out = x.launch_count();
  });
}
int mppi_gpu_profile_enable(mppi_gpu_handle* h, int enable) {
  return with_handle(h, [&](auto& x) { x.set_profile(enable != 0); });
}
int mppi_gpu_profile_read(mppi_gpu_handle* h, double* rollout_ms, uint64_t* rollout_launches, int reset) {
  return with_handle(h, [&](auto& x) { x.read_profile(rollout_ms, rollout_launches, reset != 0); });
}
int mppi_gpu_kernel_variant(mppi_gpu_handle* h, char* name_out, int capacity) {
  return with_handle(h, [&](auto& x) {
    if (!name_out || capacity < 1) throw_invalid("kernel_variant: bad buffer");
    std::snprintf(name_out, capacity, "%s", x.variant_name().c_str());
  });
}

}  // extern "C"
