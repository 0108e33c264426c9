// mppi_gpu.hpp — header-only C++ binding of the C ABI in mppi_gpu.h.
//
// This is the reference-side binding a maintainer of the reference C++
// library would add: it keeps the reference's controller
// vocabulary (proj/include/mppi/controller.hpp:18-90) and its exception types,
// so code written against `mppi::mpc_step` / `rollout_batch` / `update_plan`
// switches to the B200 path by swapping the state object:
//
//   reference                                  here
//   ---------------------------------------    -------------------------------------
//   make_controller_state(params, rule, sg,    mppi::gpu::Controller c(cfg)
//     bounds)             controller.cpp:37
//   make_vehicle_system(model, bounds, map,    c.set_dynamics_mlp(...), c.set_costmap(...)
//     cp, dt, T)          controller.cpp:7
//   mpc_step(sys, x0, cs, n)  controller.cpp:133   c.mpc_step(x0)           -> u0
//   rollout_batch(sys, x0, cs, batch, n) :55   c.rollout_batch(x0, eps, &stored)
//   compute_weights(cs, costs)           :111  c.compute_weights(costs)
//   update_plan(cs, batch, w)            :118  c.update_plan(w)
//   optimize_to_convergence(sys, x0, cs, n) :150 c.optimize_to_convergence(x0, n)
//
// Errors: MPPI_ERR_INVALID_ARGUMENT / MPPI_ERR_NONFINITE -> std::invalid_argument
// (types.hpp:105-122, weights.cpp:10-12); MPPI_ERR_DOMAIN -> std::domain_error
// (dynamics.cpp:25-27); everything else -> std::runtime_error.  Vector sizes
// are checked here, before the C ABI reads K, 2T or state_dim entries, with
// the reference's messages (controller.cpp:118-124, types.hpp:79-83).
// Header-only; link with -lmppi_gpu (paper_1707_02342_b200/lib/libmppi_gpu.so).
#ifndef MPPI_GPU_HPP_
#define MPPI_GPU_HPP_

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mppi_gpu.h"

namespace mppi {
namespace gpu {

inline void check(int code) {
  if (code == MPPI_OK) return;
  const char* msg = mppi_gpu_last_error();
  const std::string m = msg ? msg : "mppi_gpu error";
  if (code == MPPI_ERR_INVALID_ARGUMENT || code == MPPI_ERR_NONFINITE) throw std::invalid_argument(m);
  if (code == MPPI_ERR_DOMAIN) throw std::domain_error(m);
  throw std::runtime_error(m);
}

/// it_weights result (weights.hpp:9-17).
struct WeightResult {
  std::vector<double> weights;
  double normalizer = 0.0;  // eta
  double min_cost = 0.0;    // rho
};

/// One control loop (or fleet) on one device.  Owns the device state that
/// ControllerState holds in the reference; not copyable, movable.
class Controller {
 public:
  explicit Controller(const mppi_gpu_config& cfg)
      : K_(cfg.samples),
        T_(cfg.horizon_steps),
        C_(cfg.n_controllers),
        S_(cfg.system == MPPI_SYSTEM_QUADRATIC ? 2 : 7) {
    check(mppi_gpu_create(&cfg, &h_));
  }
  ~Controller() {
    if (h_) mppi_gpu_destroy(h_);
  }
  Controller(const Controller&) = delete;
  Controller& operator=(const Controller&) = delete;
  Controller(Controller&& o) noexcept
      : h_(std::exchange(o.h_, nullptr)), K_(o.K_), T_(o.T_), C_(o.C_), S_(o.S_) {}

  static mppi_gpu_config default_config() {
    mppi_gpu_config c;
    mppi_gpu_config_init(&c);
    return c;
  }

  // make_vehicle_system: the model and cost are data, copied to the device.
  void set_dynamics_mlp(int hidden, const double* w1, const double* b1, const double* w2, const double* b2,
                        const double* w3, const double* b3) {
    check(mppi_gpu_set_dynamics_mlp(h_, hidden, w1, b1, w2, b2, w3, b3));
  }
  void set_dynamics_bicycle(const mppi_bicycle_params& p) { check(mppi_gpu_set_dynamics_bicycle(h_, &p)); }
  void set_costmap(const std::vector<double>& values, int width, int height, double x0, double y0, double res) {
    if (width < 2 || height < 2 || values.size() != static_cast<size_t>(width) * static_cast<size_t>(height))
      throw std::invalid_argument("CostMap: values must hold width x height entries");
    check(mppi_gpu_set_costmap(h_, -1, values.data(), width, height, x0, y0, res));
  }

  // ControllerState accessors (plan is T x 2 row-major).
  std::vector<double> plan() const {
    std::vector<double> u(static_cast<size_t>(T_) * 2);
    check(mppi_gpu_get_plan(h_, 0, u.data()));
    return u;
  }
  void set_plan(const std::vector<double>& u) {
    if (u.size() != static_cast<size_t>(T_) * 2) throw std::invalid_argument("ControlPlan: needs a finite T x m matrix, T >= 1");
    check(mppi_gpu_set_plan(h_, 0, u.data()));
  }
  std::uint64_t iteration() const {
    std::uint64_t it = 0;
    check(mppi_gpu_get_iteration(h_, 0, &it));
    return it;
  }
  void set_iteration(std::uint64_t it) { check(mppi_gpu_set_iteration(h_, 0, it)); }

  /// mpc_step (controller.cpp:133-148): returns clamp(U'[0]) and slides.
  std::vector<double> mpc_step(const std::vector<double>& x0) {
    check_state(x0, C_);
    std::vector<double> u0(static_cast<size_t>(C_) * 2);
    check(mppi_gpu_step(h_, x0.data(), u0.data()));
    return u0;
  }
  /// rollout_batch (controller.cpp:55-109).  eps (nullable) in the reference
  /// layout K x (T x 2 column-major); `stored` receives the batch as the
  /// reference leaves it (zero-mean samples rewritten to eps - U).
  std::vector<double> rollout_batch(const std::vector<double>& x0, const double* eps = nullptr,
                                    std::vector<double>* stored = nullptr) {
    check_state(x0, 1);
    std::vector<double> costs(static_cast<size_t>(K_));
    if (stored) stored->resize(static_cast<size_t>(K_) * T_ * 2);
    check(mppi_gpu_rollout_costs(h_, x0.data(), eps, costs.data(), stored ? stored->data() : nullptr));
    return costs;
  }
  /// compute_weights / it_weights (weights.cpp:8-25).
  WeightResult compute_weights(const std::vector<double>& costs) {
    if (costs.size() != static_cast<size_t>(K_)) throw std::invalid_argument("compute_weights: cost/sample count mismatch");
    WeightResult r;
    r.weights.resize(costs.size());
    check(mppi_gpu_weights(h_, costs.data(), r.weights.data(), &r.min_cost, &r.normalizer));
    return r;
  }
  /// update_plan (controller.cpp:118-131) over the last rollout batch.
  std::vector<double> update_plan(const WeightResult& w) {
    if (w.weights.size() != static_cast<size_t>(K_)) throw std::invalid_argument("update_plan: weight/sample count mismatch");
    check(mppi_gpu_update_plan(h_, w.weights.data()));
    return plan();
  }
  /// optimize_to_convergence (controller.cpp:150-164).
  std::vector<double> optimize_to_convergence(const std::vector<double>& x0, int iterations) {
    check_state(x0, C_);
    check(mppi_gpu_optimize(h_, x0.data(), iterations));
    return plan();
  }

  mppi_gpu_handle* handle() const { return h_; }

 private:
  void check_state(const std::vector<double>& x0, int controllers) const {
    if (x0.size() != static_cast<size_t>(controllers) * static_cast<size_t>(S_))
      throw std::invalid_argument("x0: state dimension mismatch");
  }
  mppi_gpu_handle* h_ = nullptr;
  int K_ = 0, T_ = 0, C_ = 1, S_ = 7;
};

}  // namespace gpu
}  // namespace mppi

#endif  // MPPI_GPU_HPP_
