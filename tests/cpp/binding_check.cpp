// Compiles the header-only C++ binding (include/mppi_gpu.hpp) against the
// C-ABI library and checks the reference's exception mapping.  With a device
// present it also runs mpc_step / rollout_batch / compute_weights /
// update_plan through the binding on a tiny quadratic system
// (the reference fixture quadratic_system, test_controller.cpp:23-37).
// Prints one line per check; exit code 0 on success.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "mppi_gpu.hpp"

static int fails = 0;
#define EXPECT(c)                                              \
  do {                                                         \
    if (!(c)) {                                                \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);  \
      ++fails;                                                 \
    }                                                          \
  } while (0)

int main() {
  // SamplingParams::validate -> std::invalid_argument, before any device use
  {
    mppi_gpu_config c = mppi::gpu::Controller::default_config();
    c.samples = 0;
    bool threw = false;
    try {
      mppi::gpu::Controller ctl(c);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    EXPECT(threw);
    std::printf("invalid_argument mapping ok\n");
  }
  mppi_gpu_config c = mppi::gpu::Controller::default_config();
  c.samples = 64;
  c.horizon_steps = 8;
  c.system = MPPI_SYSTEM_QUADRATIC;
  c.quad_cost_scale = 1.0;
  c.lambda = 1.0;
  c.explore_fraction = 0.0;
  c.noise_mode = MPPI_NOISE_REF_SPLITMIX;
  c.precision = MPPI_FP64;
  if (mppi_gpu_device_count() == 0) {
    bool threw = false;
    try {
      mppi::gpu::Controller ctl(c);
    } catch (const std::runtime_error&) {
      threw = true;  // no CPU fallback: the B200 path fails loudly
    }
    EXPECT(threw);
    std::printf("no-device runtime_error ok\n");
    return fails ? 1 : 0;
  }
  mppi::gpu::Controller ctl(c);
  const std::vector<double> x0 = {1.0, -0.5};
  std::vector<double> stored;
  const std::vector<double> costs = ctl.rollout_batch(x0, nullptr, &stored);
  EXPECT(costs.size() == 64 && stored.size() == 64u * 8 * 2);
  const mppi::gpu::WeightResult w = ctl.compute_weights(costs);
  double s = 0;
  for (double v : w.weights) s += v;
  EXPECT(std::fabs(s - 1.0) < 1e-12);
  const std::vector<double> U = ctl.update_plan(w);
  EXPECT(U.size() == 16);
  const std::vector<double> u0 = ctl.mpc_step(x0);
  EXPECT(u0.size() == 2 && std::isfinite(u0[0]) && std::isfinite(u0[1]));
  EXPECT(ctl.iteration() == 1);
  bool threw = false;
  try {
    std::vector<double> bad(64, NAN);
    ctl.compute_weights(bad);  // it_weights rejects non-finite costs (weights.cpp:12)
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  // sizes are checked before the C ABI reads K / 2T / state_dim entries
  auto throws_invalid = [](auto&& f) {
    try {
      f();
    } catch (const std::invalid_argument&) {
      return true;
    }
    return false;
  };
  EXPECT(throws_invalid([&] { ctl.compute_weights(std::vector<double>(63, 1.0)); }));
  EXPECT(throws_invalid([&] {
    mppi::gpu::WeightResult short_w;
    short_w.weights.assign(10, 0.1);
    ctl.update_plan(short_w);
  }));
  EXPECT(throws_invalid([&] { ctl.set_plan(std::vector<double>(3, 0.0)); }));
  EXPECT(throws_invalid([&] { ctl.mpc_step(std::vector<double>(7, 0.0)); }));
  EXPECT(throws_invalid([&] { ctl.rollout_batch(std::vector<double>(1, 0.0)); }));
  EXPECT(ctl.iteration() == 1);  // none of the rejected calls touched the state
  std::printf("size checks ok\n");
  std::printf("device binding ok: u0 = (%g, %g)\n", u0[0], u0[1]);
  return fails ? 1 : 0;
}
