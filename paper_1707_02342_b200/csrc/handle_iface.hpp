// handle_iface.hpp — precision-erased controller handle behind the C ABI.
// One implementation per arithmetic type (handle_f32.cu / handle_f64.cu).
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/mppi_gpu.h"

namespace mppi_host {

struct HandleBase {
  virtual ~HandleBase() = default;
  virtual int device_index() const = 0;
  virtual int controllers() const = 0;
  virtual const mppi_gpu_config& config() const = 0;
  virtual void set_mlp(int hidden, const double* w1, const double* b1, const double* w2,
                       const double* b2, const double* w3, const double* b3) = 0;
  virtual void set_basis(const double* theta) = 0;
  virtual void set_bicycle(const mppi_bicycle_params& p) = 0;
  virtual void set_map_f64(int ctrl, const double* v, int w, int h, double x0, double y0, double res) = 0;
  virtual void set_map_f32(int ctrl, const float* v, int w, int h, double x0, double y0, double res) = 0;
  virtual void perturb_fleet(double sigma, uint64_t seed) = 0;
  virtual void get_map_f32(int ctrl, float* out) = 0;
  virtual void map_geometry(int* w, int* h, double* x0, double* y0, double* res) const = 0;
  virtual void set_plan(int ctrl, const double* U) = 0;
  virtual void get_plan(int ctrl, double* U) = 0;
  virtual void set_iteration(int ctrl, uint64_t it) = 0;
  virtual uint64_t get_iteration(int ctrl) = 0;
  virtual void set_seed(int ctrl, uint64_t seed) = 0;
  virtual void set_noise(const double* eps) = 0;
  virtual void step(const double* x0, double* u0, bool slide) = 0;
  virtual void slide_only() = 0;
  virtual void optimize(const double* x0, int iterations) = 0;
  virtual void closed_loop(const double* x_init, int iterations, double* u_trace, double* x_trace,
                           size_t flush_bytes, double* ms_out, double* iter_ms_out) = 0;
  virtual void sample_perturbations(uint64_t iteration, double* eps_out, uint8_t* flags_out) = 0;
  virtual void rollout_costs(const double* x0, const double* eps_in, double* costs_out,
                             double* eps_stored_out) = 0;
  virtual void weights(const double* costs, double* w_out, double* rho, double* eta) = 0;
  virtual void update_plan(const double* w) = 0;
  virtual void rollout_states(const double* x0, int sample, double* out) = 0;
  virtual void set_comm(int rank, int world, const unsigned char id[128]) = 0;
  virtual void set_comm_local_base(const std::vector<HandleBase*>& peers, int rank) = 0;
  virtual void local_front(const double* x0) = 0;
  virtual void local_back(bool slide) = 0;
  virtual void local_finish(double* u0) = 0;
  virtual void sync_stream() = 0;
  virtual void shard_info(int* out) const = 0;
  virtual void read_exchange_profile(double* ms, uint64_t* n, bool reset) = 0;
  virtual void* stream_ptr() const = 0;
  virtual uint64_t launch_count() const = 0;
  virtual void set_profile(bool on) = 0;
  virtual void read_profile(double* ms, uint64_t* launches, bool reset) = 0;
  virtual std::string variant_name() const = 0;
};

HandleBase* make_handle_f32(const mppi_gpu_config& cfg);
HandleBase* make_handle_f64(const mppi_gpu_config& cfg);

}  // namespace mppi_host

struct mppi_gpu_handle {
  std::unique_ptr<mppi_host::HandleBase> impl;
};
