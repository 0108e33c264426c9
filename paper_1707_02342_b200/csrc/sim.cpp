// sim.cpp — the closed-loop driver of the device controller: simulate_episode
// (/root/reference/proj/src/simulator.cpp:102-177) with the reference's
// bicycle truth plant (dynamics.cpp:23-81) on the host.
//
// Per control period: the state estimate (exact, or + N(0, std^2) noise from
// the counter stream kStreamEstimateNoise), mpc_step on the device through the
// handle (the hot path), execution noise on the commanded input
// (kStreamExecutionNoise, the sampling covariance unless given), the clamped
// truth step, then the disturbance kicks due after this step.  Every noise
// draw is the reference's counter-addressed Box-Muller (sampler.hpp:15-60), so
// an episode is a pure function of the handle's seed.  Double precision on
// the host, compiled without FMA contraction: the truth plant rounds exactly
// as the reference's expression order.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "../../include/mppi_gpu.h"
#include "errors.hpp"
#include "handle_iface.hpp"

using namespace mppi_host;

namespace {

// sampler.hpp:15-60
inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
inline uint64_t counter_hash(uint64_t seed, uint64_t stream, uint64_t it, uint64_t k, uint64_t t, uint64_t pair) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ stream);
  h = splitmix64(h ^ it);
  h = splitmix64(h ^ k);
  h = splitmix64(h ^ t);
  return splitmix64(h ^ pair);
}
inline double counter_normal(uint64_t seed, uint64_t stream, uint64_t it, uint64_t k, uint64_t t, int component) {
  const uint64_t h = counter_hash(seed, stream, it, k, t, static_cast<uint64_t>(component / 2));
  const double u1 = static_cast<double>((h >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(splitmix64(h) >> 11) * 0x1.0p-53;
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double phi = 2.0 * M_PI * u2;
  return (component % 2 == 0) ? r * std::cos(phi) : r * std::sin(phi);
}
constexpr uint64_t kStreamExecutionNoise = 0x657865636e6f6973ull;
constexpr uint64_t kStreamEstimateNoise = 0x657374696d617465ull;

void validate_bicycle(const mppi_bicycle_params& p) {  // BicycleParams::validate (dynamics.hpp:53-61)
  const double v[9] = {p.mass, p.yaw_inertia, p.a, p.b, p.stiffness, p.mu, p.load, p.steer_scale, p.force_scale};
  for (double x : v)
    if (!(x > 0.0) || !std::isfinite(x)) throw_invalid("BicycleParams: all parameters must be positive");
}

// brush_tire_force (dynamics.cpp:23-43)
double brush_tire_force(double alpha, double u_F, const mppi_bicycle_params& p) {
  const double limit = p.mu * p.load;
  if (std::abs(u_F) > limit)
    throw Error(MPPI_ERR_DOMAIN, "brush_tire_force: |u_F| exceeds the friction circle mu*F_z");
  const double xi = std::sqrt(limit * limit - u_F * u_F) / limit;
  if (xi == 0.0) return 0.0;
  const double sign = (alpha >= 0.0) ? 1.0 : -1.0;
  const double crossover = std::atan(3.0 * xi * p.mu * p.load / p.stiffness);
  if (std::abs(alpha) >= crossover) return -p.mu * xi * p.load * sign;
  const double ta = std::tan(alpha);
  const double c = p.stiffness;
  return -c * ta + c * c / (3.0 * xi * p.mu * p.load) * ta * std::abs(ta) -
         c * c * c / (27.0 * p.mu * p.mu * xi * xi * p.load * p.load) * ta * ta * ta;
}

// step_bicycle_truth (dynamics.cpp:51-81); kSlipGuardSpeed = 0.1
void bicycle_step(const mppi_bicycle_params& p, const double x[7], double steer, double throttle, double dt,
                  double n[7]) {
  if (!(dt > 0.0)) throw_invalid("step_bicycle_truth: dt must be > 0");
  const double u_delta = p.steer_scale * steer;
  const double u_F = p.force_scale * throttle;
  const double r = x[6];
  double alpha_f, alpha_r;
  if (x[4] > 0.1) {
    const double beta = x[5] / x[4];
    alpha_f = std::atan(beta + p.a * r / x[4]) - u_delta;
    alpha_r = std::atan(beta - p.b * r / x[4]);
  } else {
    alpha_f = -u_delta;
    alpha_r = 0.0;
  }
  const double f_yf = brush_tire_force(alpha_f, u_F, p);
  const double f_yr = brush_tire_force(alpha_r, u_F, p);
  for (int i = 0; i < 7; ++i) n[i] = x[i];
  n[0] += (std::cos(x[2]) * x[4] - std::sin(x[2]) * x[5]) * dt;
  n[1] += (std::sin(x[2]) * x[4] + std::cos(x[2]) * x[5]) * dt;
  n[2] += r * dt;
  n[4] += ((u_F - f_yf * std::sin(u_delta)) / p.mass + r * x[5]) * dt;
  n[5] += ((f_yf + f_yr) / p.mass - r * x[4]) * dt;
  n[6] += ((p.a * f_yf - p.b * f_yr) / p.yaw_inertia) * dt;
}

struct HostMap {
  std::vector<float> v;
  int w = 0, h = 0;
  double x0 = 0, y0 = 0, res = 1;
  // costmap_lookup (costs.cpp:7-22)
  double lookup(double px, double py) const {
    double gx = std::clamp((px - x0) / res, 0.0, static_cast<double>(w - 1));
    double gy = std::clamp((py - y0) / res, 0.0, static_cast<double>(h - 1));
    const int ix = std::min(static_cast<int>(gx), w - 2), iy = std::min(static_cast<int>(gy), h - 2);
    const double fx = gx - ix, fy = gy - iy;
    auto at = [&](int i, int j) { return static_cast<double>(v[static_cast<size_t>(j) * w + i]); };
    return (1 - fx) * (1 - fy) * at(ix, iy) + fx * (1 - fy) * at(ix + 1, iy) + (1 - fx) * fy * at(ix, iy + 1) +
           fx * fy * at(ix + 1, iy + 1);
  }
};

// state_cost(x, 0, map, costs) (costs.cpp:29-43) + the BASELINE crash term; decay^0 = 1
double state_cost0(const double x[7], double h, const mppi_cost_params& cp) {
  double track = h;
  if (h > cp.boundary_threshold) track += std::pow(cp.decay, 0) * cp.impulse;
  const double dv = x[4] - cp.v_des;
  const double speed = dv * dv;
  const double zeta = (std::abs(x[4]) < 0.01) ? 0.0 : -std::atan(x[5] / std::abs(x[4]));  // side_slip
  double stab = zeta * zeta;
  if (std::abs(zeta) > cp.slip_limit) stab += cp.impulse;
  double c = cp.alpha_track * track + cp.alpha_speed * speed + cp.alpha_stab * stab;
  if (cp.crash_penalty != 0.0 && (h > cp.crash_threshold || std::abs(x[3]) > cp.roll_limit)) c += cp.crash_penalty;
  return c;
}

}  // namespace

extern "C" {

void mppi_bicycle_params_init(mppi_bicycle_params* p) {
  if (!p) return;
  *p = mppi_bicycle_params{22.0, 1.8, 0.45, 0.35, 180.0, 0.65, 107.9, 0.35, 35.0};
}

void mppi_sim_config_init(mppi_sim_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->episode_s = 30.0;
  c->exec_noise = 1;
  mppi_bicycle_params_init(&c->plant);
}

int mppi_brush_tire_force(double alpha, double u_F, const mppi_bicycle_params* p, double* force_out) {
  return guard([&] {
    if (!p || !force_out) throw_invalid("brush_tire_force: null");
    validate_bicycle(*p);
    *force_out = brush_tire_force(alpha, u_F, *p);
  });
}

int mppi_bicycle_step(const mppi_bicycle_params* p, const double x[7], const double v[2], double dt, double out[7]) {
  return guard([&] {
    if (!p || !x || !v || !out) throw_invalid("bicycle_step: null");
    validate_bicycle(*p);
    bicycle_step(*p, x, v[0], v[1], dt, out);
  });
}

int mppi_sim_episode(mppi_gpu_handle* h, const mppi_sim_config* cfg, mppi_sim_record* out, int capacity,
                     int* n_steps_out, int* aborted_out) {
  return guard([&] {
    if (!h || !h->impl || !cfg || !out || !n_steps_out || !aborted_out) throw_invalid("sim_episode: null argument");
    HandleBase& ctl = *h->impl;
    CUDA_TRY(cudaSetDevice(ctl.device_index()));
    const mppi_gpu_config& c = ctl.config();
    if (c.n_controllers != 1) throw Error(MPPI_ERR_UNSUPPORTED, "simulate_episode: one controller per handle");
    if (c.system == MPPI_SYSTEM_QUADRATIC) throw_invalid("simulate_episode: needs a vehicle system");
    validate_bicycle(cfg->plant);
    if (cfg->n_disturbances < 0 || (cfg->n_disturbances > 0 && !cfg->disturbances))
      throw_invalid("simulate_episode: bad disturbance list");
    const double dt = c.dt;
    const long steps = std::lround(cfg->episode_s / dt);
    if (steps < 0 || steps > capacity) throw_invalid("simulate_episode: records_out holds fewer than the episode's steps");
    HostMap map;
    ctl.map_geometry(&map.w, &map.h, &map.x0, &map.y0, &map.res);
    map.v.resize(static_cast<size_t>(map.w) * map.h);
    ctl.get_map_f32(0, map.v.data());
    const double exec_var[2] = {cfg->has_exec_noise_diag ? cfg->exec_noise_diag[0] : c.sigma_diag[0],
                                cfg->has_exec_noise_diag ? cfg->exec_noise_diag[1] : c.sigma_diag[1]};
    const uint64_t seed = c.seed;
    double x[7], xn[7];
    std::memcpy(x, cfg->start_state, sizeof(x));
    *aborted_out = 0;
    int n = 0;
    for (long i = 0; i < steps; ++i) {
      bool finite = true;
      for (double v : x) finite = finite && std::isfinite(v);
      if (!finite) {
        *aborted_out = 1;
        break;
      }
      double est[7];
      std::memcpy(est, x, sizeof(est));
      if (cfg->has_estimate_noise)
        for (int k = 0; k < 7; ++k)
          est[k] += cfg->estimate_noise_std[k] *
                    counter_normal(seed, kStreamEstimateNoise, static_cast<uint64_t>(i), 0, 0, k);
      double u0[2];
      ctl.step(est, u0, /*slide=*/true);  // mpc_step on the device
      double real[2] = {u0[0], u0[1]};
      if (cfg->exec_noise)
        for (int j = 0; j < 2; ++j)
          real[j] += std::sqrt(exec_var[j]) *
                     counter_normal(seed, kStreamExecutionNoise, static_cast<uint64_t>(i), 0, 0, j);
      mppi_sim_record& r = out[n++];
      r.time = static_cast<double>(i) * dt;
      std::memcpy(r.state, x, sizeof(x));
      r.commanded[0] = u0[0];
      r.commanded[1] = u0[1];
      r.realized[0] = real[0];
      r.realized[1] = real[1];
      r.map_h = map.lookup(x[0], x[1]);
      r.cost = state_cost0(x, r.map_h, c.cost);
      // clamp_controls (dynamics.cpp:8-21), std::clamp semantics
      const double v0 = std::clamp(real[0], c.bounds_lower[0], c.bounds_upper[0]);
      const double v1 = std::clamp(real[1], c.bounds_lower[1], c.bounds_upper[1]);
      bicycle_step(cfg->plant, x, v0, v1, dt, xn);
      std::memcpy(x, xn, sizeof(x));
      for (int d = 0; d < cfg->n_disturbances; ++d) {
        const mppi_disturbance& k = cfg->disturbances[d];
        if (std::lround(k.time_s / dt) == i + 1) {
          x[4] += k.dv_x;
          x[5] += k.dv_y;
          x[6] += k.dtheta_dot;
        }
      }
    }
    *n_steps_out = n;
  });
}

}  // extern "C"
