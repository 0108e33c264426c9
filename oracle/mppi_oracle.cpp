// ============================================================================
// mppi_oracle.cpp — CPU restatement of the reference IT-MPPI hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library, and
// only as the checker (or as the timed reference CPU arm).  The product path
// (paper_1707_02342_b200/) never links or calls it.
//
// Why a restatement: the reference (/root/reference/proj) cannot be built in
// this environment — find_package(Eigen3 REQUIRED) (proj/CMakeLists.txt:12)
// fails because Eigen3 is absent, and vendor/ (CLI11, nlohmann/json, doctest)
// is gitignored and absent.  Eigen3 is the only third-party dependency on the
// path (version unpinned: `find_package(Eigen3 3.3)` is a minimum); its
// arithmetic here is plain dense GEMV / elementwise tanh / LDLT of a tiny
// normal matrix, restated below in scalar loops.  Eigen's internal GEMV
// summation order is not reproduced, so parity with an Eigen build is "within
// rounding", never bitwise.  The oracle is pinned against the reference's own
// known-answer tests (tests/golden/reference_pins.json, tests/test_oracle_*.py).
//
// Each function cites the reference file:line it follows.  The code is
// templated on the arithmetic type R: R = double is the reference restatement;
// R = float mirrors the device fp32 path's operation order (same FMA use, same
// host-computed tables) so the fp32 kernel can be compared tightly.
//
// Threading mirrors the reference: rollouts over contiguous sample chunks with
// one std::thread per chunk spawned and joined on every call
// (proj/include/mppi/parallel.hpp:11-29); sampling, weights and the update are
// serial (sampler.cpp:19-35, weights.cpp:15-23, controller.cpp:125-128).
// ============================================================================
#include "../include/mppi_gpu.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- errors ----
struct NonFinite : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
thread_local std::string g_last_error;

// ------------------------------------------------- counter RNG (reference) --
// proj/include/mppi/sampler.hpp:15-20
inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
// sampler.hpp:22-32
inline uint64_t counter_hash(uint64_t seed, uint64_t stream, uint64_t iteration, uint64_t k,
                             uint64_t t, uint64_t pair) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ stream);
  h = splitmix64(h ^ iteration);
  h = splitmix64(h ^ k);
  h = splitmix64(h ^ t);
  h = splitmix64(h ^ pair);
  return h;
}
// sampler.hpp:35-42 (Box-Muller; u1 in (0,1], u2 in [0,1))
inline void normal_pair(uint64_t h, double& z0, double& z1) {
  const double u1 = static_cast<double>((h >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(splitmix64(h) >> 11) * 0x1.0p-53;
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double phi = 2.0 * M_PI * u2;
  z0 = r * std::cos(phi);
  z1 = r * std::sin(phi);
}
// sampler.hpp:46-54
inline double counter_normal(uint64_t seed, uint64_t stream, uint64_t iteration, uint64_t k,
                             uint64_t t, int component) {
  double z0 = 0.0, z1 = 0.0;
  normal_pair(counter_hash(seed, stream, iteration, k, t, static_cast<uint64_t>(component / 2)),
              z0, z1);
  return (component % 2 == 0) ? z0 : z1;
}
constexpr uint64_t kStreamPerturbations = 0x706572747572626full;  // sampler.hpp:57

// ------------------------------------------------------ Philox4x32-10 -------
// Production noise of the device path (not in the reference; BASELINE.json
// north_star asks for Philox).  Restated from the published Philox4x32-10
// definition (Salmon et al., SC'11): 10 rounds, multipliers 0xD2511F53 /
// 0xCD9E8D57, Weyl key increments 0x9E3779B9 / 0xBB67AE85.
inline void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}
// Counter layout of the device stream: ctr = (t/2, k, iter_lo, iter_hi),
// key = (seed_lo, seed_hi); outputs (0,1) feed even t, (2,3) odd t.
// u1 = ((a>>8)+1) 2^-24 in (0,1], u2 = (b>>8) 2^-24 in [0,1).
inline void philox_normal_pair(uint64_t seed, uint64_t iteration, uint64_t k, uint64_t t,
                               double& z0, double& z1) {
  const uint32_t ctr[4] = {static_cast<uint32_t>(t >> 1), static_cast<uint32_t>(k),
                           static_cast<uint32_t>(iteration),
                           static_cast<uint32_t>(iteration >> 32)};
  const uint32_t key[2] = {static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)};
  uint32_t r[4];
  philox4x32_10(ctr, key, r);
  const uint32_t a = (t & 1) ? r[2] : r[0];
  const uint32_t b = (t & 1) ? r[3] : r[1];
  const double u1 = static_cast<double>((a >> 8) + 1u) * 0x1.0p-24;
  const double u2 = static_cast<double>(b >> 8) * 0x1.0p-24;
  const double rr = std::sqrt(-2.0 * std::log(u1));
  z0 = rr * std::cos(2.0 * M_PI * u2);
  z1 = rr * std::sin(2.0 * M_PI * u2);
}

// -------------------------------------------------------------- types -------
// SamplingParams (types.hpp:92-123); validate() restated verbatim.
struct Sampling {
  int samples = 1200, horizon_steps = 80;
  double dt = 0.025;
  double sigma_diag[2] = {0.0306, 0.0506};
  int m = 2;  // control dimension (sigma_diag.size())
  double lambda = 12.5, gamma = 0.1, explore_fraction = 0.01;
  uint64_t seed = 0;
  void validate() const {
    if (samples < 1) throw std::invalid_argument("SamplingParams: samples must be >= 1");
    if (horizon_steps < 1) throw std::invalid_argument("SamplingParams: horizon_steps must be >= 1");
    if (!(dt > 0.0)) throw std::invalid_argument("SamplingParams: dt must be > 0");
    for (int c = 0; c < m; ++c)
      if (!(sigma_diag[c] > 0.0) || !std::isfinite(sigma_diag[c]))
        throw std::invalid_argument("SamplingParams: sigma_diag entries must be finite and > 0");
    if (!(lambda > 0.0)) throw std::invalid_argument("SamplingParams: lambda must be > 0");
    if (!(gamma >= 0.0)) throw std::invalid_argument("SamplingParams: gamma must be >= 0");
    if (!(explore_fraction >= 0.0 && explore_fraction < 1.0))
      throw std::invalid_argument("SamplingParams: explore_fraction must be in [0, 1)");
  }
  int n_zero_mean() const {  // sampler.cpp:36
    return static_cast<int>(std::lround(explore_fraction * samples));
  }
};

// PerturbationBatch (types.hpp:127-132); eps[k] stored column-major T x m.
template <class R>
struct Batch {
  int K = 0, T = 0, m = 2;
  std::vector<R> eps;            // K * m * T, eps[k][c][t]
  std::vector<uint8_t> flags;    // K
  R& at(int k, int t, int c) { return eps[(static_cast<size_t>(k) * m + c) * T + t]; }
  R at(int k, int t, int c) const { return eps[(static_cast<size_t>(k) * m + c) * T + t]; }
};

// sample_perturbations (sampler.cpp:5-39).  Noise is generated in double and
// rounded to R once (the device does the same for its fp32 path).
template <class R>
Batch<R> sample_perturbations(const Sampling& p, uint64_t iteration, int mode) {
  p.validate();
  Batch<R> b;
  b.K = p.samples; b.T = p.horizon_steps; b.m = p.m;
  b.eps.assign(static_cast<size_t>(b.K) * b.m * b.T, R(0));
  b.flags.assign(b.K, 0);
  double scale[2];
  for (int c = 0; c < p.m; ++c) scale[c] = std::sqrt(p.sigma_diag[c]);
  for (int k = 0; k < b.K; ++k) {
    for (int t = 0; t < b.T; ++t) {
      for (int pair = 0; pair * 2 < p.m; ++pair) {
        double z0 = 0.0, z1 = 0.0;
        if (mode == MPPI_NOISE_PHILOX) {
          philox_normal_pair(p.seed, iteration, static_cast<uint64_t>(k),
                             static_cast<uint64_t>(t), z0, z1);
        } else {
          normal_pair(counter_hash(p.seed, kStreamPerturbations, iteration,
                                   static_cast<uint64_t>(k), static_cast<uint64_t>(t),
                                   static_cast<uint64_t>(pair)),
                      z0, z1);
        }
        b.at(k, t, 2 * pair) = static_cast<R>(scale[2 * pair] * z0);
        if (2 * pair + 1 < p.m) b.at(k, t, 2 * pair + 1) = static_cast<R>(scale[2 * pair + 1] * z1);
      }
    }
  }
  const int n_zero = p.n_zero_mean();
  for (int k = b.K - n_zero; k < b.K; ++k) b.flags[k] = 1;
  return b;
}

// ControlBounds + clamp_controls (dynamics.hpp:12-33, dynamics.cpp:8-21).
// std::clamp semantics (NaN passes through), mirrored on the device.
template <class R>
inline R clampv(R v, R lo, R hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }

// MlpWeights (dynamics.hpp:110-119), generalised to H in {32, 64}; row-major.
template <class R>
struct Mlp {
  int H = 32;
  std::vector<R> w1, b1, w2, b2, w3, b3;
};
template <class R>
inline R mac(R acc, R w, R x) { return std::fma(w, x, acc); }

// Evaluation-order variant of mlp_forward (accuracy studies only, default 0):
// 1 sums every dot product over its inputs in DESCENDING order.  Two valid
// fp32 evaluations of the same MLP differ by rounding alone; the spread of the
// fp32 restatement between the two orders is the envelope an fp32 device
// kernel with yet another order (tensor-core split products) is held to.
inline int g_mlp_order = 0;

// mlp_forward (dynamics.cpp:197-204): h1 = tanh(W1 in + b1),
// h2 = tanh(W2 h1 + b2), out = W3 h2 + b3.  Accumulation starts from the bias
// and runs over inputs in ascending order with fused multiply-adds (the
// device kernel uses the same order).
template <class R>
void mlp_forward(const R in[6], const Mlp<R>& w, R out[4]) {
  const int H = w.H;
  R h1[64], h2[64];
  const bool rev = g_mlp_order == 1;
  for (int j = 0; j < H; ++j) {
    R a = w.b1[j];
    for (int q = 0; q < 6; ++q) {
      const int i = rev ? 5 - q : q;
      a = mac(a, w.w1[j * 6 + i], in[i]);
    }
    h1[j] = std::tanh(a);
  }
  for (int j = 0; j < H; ++j) {
    R a = w.b2[j];
    for (int q = 0; q < H; ++q) {
      const int i = rev ? H - 1 - q : q;
      a = mac(a, w.w2[j * H + i], h1[i]);
    }
    h2[j] = std::tanh(a);
  }
  for (int o = 0; o < 4; ++o) {
    R a = w.b3[o];
    for (int q = 0; q < H; ++q) {
      const int i = rev ? H - 1 - q : q;
      a = mac(a, w.w3[o * H + i], h2[i]);
    }
    out[o] = a;
  }
}

// advance_split (dynamics.cpp:137-148): explicit Euler from the OLD state.
template <class R>
void advance_split(const R x[7], const R d[4], R dt, R n[7]) {
  const R c = std::cos(x[2]), s = std::sin(x[2]);
  n[0] = x[0] + (c * x[4] - s * x[5]) * dt;
  n[1] = x[1] + (s * x[4] + c * x[5]) * dt;
  n[2] = x[2] + x[6] * dt;
  n[3] = x[3] + d[0] * dt;
  n[4] = x[4] + d[1] * dt;
  n[5] = x[5] + d[2] * dt;
  n[6] = x[6] + d[3] * dt;
}

// ----------------------------------------------- basis-function model ------
// eval_basis (dynamics.cpp:83-133); kSlipGuardSpeed = 0.1 (dynamics.cpp:47).
template <class R>
void eval_basis(R roll, R v_x, R v_y, R r, R u_delta, R u_F, R phi[25]) {
  R alpha_f, alpha_r, ratio;
  if (v_x > R(0.1)) {
    ratio = v_y / v_x;
    alpha_f = std::atan(ratio + R(0.45) * r / v_x - u_delta);
    alpha_r = std::atan(ratio - R(0.35) * r / v_x);
  } else {
    ratio = R(0);
    alpha_f = -u_delta;
    alpha_r = R(0);
  }
  const R tf = std::tan(alpha_f), tr = std::tan(alpha_r), sd = std::sin(u_delta);
  phi[0] = u_F;
  phi[1] = v_x / R(10.0);
  phi[2] = sd * tf / R(1200.0);
  phi[3] = sd * tf * std::abs(tf) / R(1200.0 * 1200.0);
  phi[4] = sd * tf * tf * tf / R(1200.0 * 1200.0 * 1200.0);
  phi[5] = r * v_y / R(25.0);
  phi[6] = r / R(10.0);
  phi[7] = v_y / R(10.0);
  phi[8] = sd;
  phi[9] = ratio / R(40.0);
  phi[10] = tf / R(1400.0);
  phi[11] = tf * std::abs(tf) / R(1400.0 * 1400.0);
  phi[12] = tf * tf * tf / R(1400.0 * 1400.0 * 1400.0);
  phi[13] = tr / R(40.0);
  phi[14] = tr * std::abs(tr) / R(40.0 * 40.0);
  phi[15] = tr * tr * tr / R(40.0 * 40.0 * 40.0);
  phi[16] = r * v_x / R(50.0);
  phi[17] = roll;
  phi[18] = roll * r;
  phi[19] = roll * v_x / R(3.0);
  phi[20] = roll * v_x * r / R(5.0);
  phi[21] = v_x * v_x / R(100.0);
  phi[22] = v_x * v_x * v_x / R(1000.0);
  phi[23] = u_F * u_F;
  phi[24] = u_F * u_F * u_F;
}
// step_basis_model (dynamics.cpp:152-157): xd_dot = coeffs^T phi, the sum over
// the 25 basis functions in ascending order (Eigen's GEMV order is not
// reproduced), then advance_split.
template <class R>
void basis_dot(const R theta[100], const R phi[25], R d[4]) {
  for (int o = 0; o < 4; ++o) {
    R acc = theta[o] * phi[0];
    for (int b = 1; b < 25; ++b) acc = acc + theta[b * 4 + o] * phi[b];
    d[o] = acc;
  }
}

// CostMap (costs.hpp:11-38)
template <class R>
struct Map {
  int width = 0, height = 0;
  R x0 = 0, y0 = 0, res = 1, inv_res = 1;
  std::vector<R> v;
};
// costmap_lookup (costs.cpp:7-22).  The fp32 restatement multiplies by the
// host-rounded reciprocal of the resolution, as the device does.
template <class R>
R costmap_lookup(const Map<R>& m, R px, R py) {
  R gx, gy;
  if constexpr (std::is_same_v<R, double>) {
    gx = (px - m.x0) / m.res;
    gy = (py - m.y0) / m.res;
  } else {
    gx = (px - m.x0) * m.inv_res;
    gy = (py - m.y0) * m.inv_res;
  }
  gx = clampv<R>(gx, R(0), static_cast<R>(m.width - 1));
  gy = clampv<R>(gy, R(0), static_cast<R>(m.height - 1));
  // static_cast<int>(NaN) is UB in C++; the device maps NaN to cell 0 and the
  // NaN still propagates through the weights below.
  const int ix = std::isnan(gx) ? 0 : std::min(static_cast<int>(gx), m.width - 2);
  const int iy = std::isnan(gy) ? 0 : std::min(static_cast<int>(gy), m.height - 2);
  const R fx = gx - static_cast<R>(ix);
  const R fy = gy - static_cast<R>(iy);
  const size_t base = static_cast<size_t>(iy) * m.width + ix;
  const R v00 = m.v[base], v10 = m.v[base + 1];
  const R v01 = m.v[base + m.width], v11 = m.v[base + m.width + 1];
  return (R(1) - fx) * (R(1) - fy) * v00 + fx * (R(1) - fy) * v10 + (R(1) - fx) * fy * v01 +
         fx * fy * v11;
}

// CostParams (costs.hpp:46-64) + the BASELINE crash term (see mppi_gpu.h).
template <class R>
struct Cost {
  R alpha_track, alpha_speed, alpha_stab, v_des, impulse, decay, boundary_threshold,
      slip_limit, crash_penalty, crash_threshold, roll_limit;
  std::vector<R> decay_pow;  // decay^t, t = 0..T (host std::pow, costs.cpp:35)
};

// side_slip (costs.cpp:24-27)
template <class R>
R side_slip(R vx, R vy) {
  if (std::abs(vx) < R(0.01)) return R(0);
  return -std::atan(vy / std::abs(vx));
}

// state_cost (costs.cpp:29-43) + crash term.
template <class R>
R state_cost(const R x[7], int t, const Map<R>& map, const Cost<R>& cp) {
  const R h = costmap_lookup(map, x[0], x[1]);
  R track = h;
  if (h > cp.boundary_threshold) track += cp.decay_pow[t] * cp.impulse;
  const R dv = x[4] - cp.v_des;
  const R speed = dv * dv;
  R c = cp.alpha_track * track + cp.alpha_speed * speed;
  if (cp.alpha_stab != R(0)) {
    const R zeta = side_slip(x[4], x[5]);
    R stab = zeta * zeta;
    if (std::abs(zeta) > cp.slip_limit) stab += cp.impulse;
    c += cp.alpha_stab * stab;
  }
  if (cp.crash_penalty != R(0) && (h > cp.crash_threshold || std::abs(x[3]) > cp.roll_limit))
    c += cp.crash_penalty;
  return c;
}

// RolloutSystem (controller.hpp:18-24): the type-erased plugin triple.
template <class R>
struct System {
  int state_dim = 0, control_dim = 0;
  std::function<void(const R* x, const R* v, int t, R* x_next)> step;
  std::function<R(const R* x, int t)> running_cost;
  std::function<R(const R* x)> terminal_cost;
};

// make_vehicle_system (controller.cpp:7-35) over an MlpModel (dynamics.hpp:164-174).
template <class R>
System<R> make_vehicle_system(const Mlp<R>& mlp, const R lo[2], const R hi[2],
                              const Map<R>& map, const Cost<R>& cp, R dt, int horizon,
                              bool with_terminal) {
  if (!(dt > R(0))) throw std::invalid_argument("step_mlp_model: dt must be > 0");
  System<R> s;
  s.state_dim = 7;
  s.control_dim = 2;
  const R l0 = lo[0], l1 = lo[1], h0 = hi[0], h1 = hi[1];
  s.step = [&mlp, l0, l1, h0, h1, dt](const R* x, const R* v, int, R* xn) {
    const R in[6] = {x[3], x[4], x[5], x[6], clampv(v[0], l0, h0), clampv(v[1], l1, h1)};
    R d[4];
    mlp_forward(in, mlp, d);          // step_mlp_model (dynamics.cpp:206-210)
    advance_split(x, d, dt, xn);
  };
  s.running_cost = [&map, &cp](const R* x, int t) { return state_cost(x, t, map, cp); };
  if (with_terminal) {
    s.terminal_cost = [&map, &cp, horizon](const R* x) { return state_cost(x, horizon, map, cp); };
  } else {
    s.terminal_cost = [](const R*) { return R(0); };
  }
  return s;
}

// make_vehicle_system (controller.cpp:7-35) over a BasisFunctionModel
// (dynamics.hpp:151-162).
template <class R>
System<R> make_basis_system(const std::vector<R>& theta, const R lo[2], const R hi[2], const Map<R>& map,
                            const Cost<R>& cp, R dt, int horizon, bool with_terminal) {
  if (!(dt > R(0))) throw std::invalid_argument("step_basis_model: dt must be > 0");
  System<R> s;
  s.state_dim = 7;
  s.control_dim = 2;
  const R l0 = lo[0], l1 = lo[1], h0 = hi[0], h1 = hi[1];
  s.step = [&theta, l0, l1, h0, h1, dt](const R* x, const R* v, int, R* xn) {
    R phi[25], d[4];
    eval_basis<R>(x[3], x[4], x[5], x[6], clampv(v[0], l0, h0), clampv(v[1], l1, h1), phi);
    basis_dot<R>(theta.data(), phi, d);
    advance_split(x, d, dt, xn);
  };
  s.running_cost = [&map, &cp](const R* x, int t) { return state_cost(x, t, map, cp); };
  if (with_terminal) {
    s.terminal_cost = [&map, &cp, horizon](const R* x) { return state_cost(x, horizon, map, cp); };
  } else {
    s.terminal_cost = [](const R*) { return R(0); };
  }
  return s;
}

// ------------------------------------------------ bicycle truth model -------
// BicycleParams (dynamics.hpp:42-62), entries in declaration order.
template <class R>
struct Bicycle {
  R mass = R(22.0), yaw_inertia = R(1.8), a = R(0.45), b = R(0.35), stiffness = R(180.0), mu = R(0.65),
    load = R(107.9), steer_scale = R(0.35), force_scale = R(35.0);
};

// brush_tire_force (dynamics.cpp:23-43)
template <class R>
R brush_tire_force(R alpha, R u_F, const Bicycle<R>& p) {
  const R limit = p.mu * p.load;
  if (std::abs(u_F) > limit)
    throw std::domain_error("brush_tire_force: |u_F| exceeds the friction circle mu*F_z");
  const R xi = std::sqrt(limit * limit - u_F * u_F) / limit;
  if (xi == R(0)) return R(0);
  const R sign = (alpha >= R(0)) ? R(1) : R(-1);
  const R crossover = std::atan(R(3) * xi * p.mu * p.load / p.stiffness);
  if (std::abs(alpha) >= crossover) return -p.mu * xi * p.load * sign;
  const R ta = std::tan(alpha);
  const R c = p.stiffness;
  return -c * ta + c * c / (R(3) * xi * p.mu * p.load) * ta * std::abs(ta) -
         c * c * c / (R(27) * p.mu * p.mu * xi * xi * p.load * p.load) * ta * ta * ta;
}

// step_bicycle_truth (dynamics.cpp:51-81), kSlipGuardSpeed = 0.1; roll unchanged
template <class R>
void step_bicycle(const R x[7], const R v[2], R dt, const Bicycle<R>& p, R n[7]) {
  if (!(dt > R(0))) throw std::invalid_argument("step_bicycle_truth: dt must be > 0");
  const R u_delta = p.steer_scale * v[0];
  const R u_F = p.force_scale * v[1];
  const R r = x[6];
  R alpha_f, alpha_r;
  if (x[4] > R(0.1)) {
    const R beta = x[5] / x[4];
    alpha_f = std::atan(beta + p.a * r / x[4]) - u_delta;
    alpha_r = std::atan(beta - p.b * r / x[4]);
  } else {
    alpha_f = -u_delta;
    alpha_r = R(0);
  }
  const R f_yf = brush_tire_force<R>(alpha_f, u_F, p);
  const R f_yr = brush_tire_force<R>(alpha_r, u_F, p);
  for (int i = 0; i < 7; ++i) n[i] = x[i];
  n[0] += (std::cos(x[2]) * x[4] - std::sin(x[2]) * x[5]) * dt;
  n[1] += (std::sin(x[2]) * x[4] + std::cos(x[2]) * x[5]) * dt;
  n[2] += r * dt;
  n[4] += ((u_F - f_yf * std::sin(u_delta)) / p.mass + r * x[5]) * dt;
  n[5] += ((f_yf + f_yr) / p.mass - r * x[4]) * dt;
  n[6] += ((p.a * f_yf - p.b * f_yr) / p.yaw_inertia) * dt;
}

// make_vehicle_system (controller.cpp:7-35) over a BicycleTruthModel
// (dynamics.hpp:176-183): clamp, then step_bicycle_truth.
template <class R>
System<R> make_bicycle_system(const Bicycle<R>& bike, const R lo[2], const R hi[2], const Map<R>& map,
                              const Cost<R>& cp, R dt, int horizon, bool with_terminal) {
  System<R> s;
  s.state_dim = 7;
  s.control_dim = 2;
  const R l0 = lo[0], l1 = lo[1], h0 = hi[0], h1 = hi[1];
  s.step = [&bike, l0, l1, h0, h1, dt](const R* x, const R* v, int, R* xn) {
    const R g[2] = {clampv(v[0], l0, h0), clampv(v[1], l1, h1)};
    step_bicycle<R>(x, g, dt, bike, xn);
  };
  s.running_cost = [&map, &cp](const R* x, int t) { return state_cost(x, t, map, cp); };
  if (with_terminal) {
    s.terminal_cost = [&map, &cp, horizon](const R* x) { return state_cost(x, horizon, map, cp); };
  } else {
    s.terminal_cost = [](const R*) { return R(0); };
  }
  return s;
}

// quadratic_system (test_controller.cpp:23-37), running cost scaled.
template <class R>
System<R> make_quadratic_system(int m, R dt, R cost_scale) {
  System<R> s;
  s.state_dim = m;
  s.control_dim = m;
  s.step = [m, dt](const R* x, const R* v, int, R* nx) {
    for (int i = 0; i < m; ++i) nx[i] = x[i] + v[i] * dt;
  };
  s.running_cost = [m, cost_scale](const R* x, int) {
    R acc = 0;
    for (int i = 0; i < m; ++i) acc += x[i] * x[i];
    return cost_scale * acc;
  };
  s.terminal_cost = [](const R*) { return R(0); };
  return s;
}

// parallel_for_chunks (parallel.hpp:11-29), verbatim semantics.
inline void parallel_for_chunks(int n, int n_threads, const std::function<void(int, int)>& fn) {
  if (n <= 0) return;
  if (n_threads <= 1 || n == 1) {
    fn(0, n);
    return;
  }
  const int workers = std::min(n_threads, n);
  std::vector<std::thread> pool;
  pool.reserve(workers);
  const int chunk = (n + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const int begin = w * chunk;
    const int end = std::min(n, begin + chunk);
    if (begin >= end) break;
    pool.emplace_back([&fn, begin, end] { fn(begin, end); });
  }
  for (auto& t : pool) t.join();
}

// SGFilter / sg_coefficients (smoothing.cpp:5-33): kernel = X (X^T X)^{-1} e0.
// The reference solves the normal equations with Eigen LDLT; restated with a
// thin QR of the (column-scaled) design matrix, in double.
inline std::vector<double> sg_coefficients(int window, int degree) {
  if (window < 3 || window % 2 == 0)
    throw std::invalid_argument("sg_coefficients: window must be odd and >= 3");
  if (degree < 0 || degree >= window)
    throw std::invalid_argument("sg_coefficients: need 0 <= degree < window");
  const int half = window / 2, n = degree + 1;
  // Scaled design matrix X[i][j] = ((i - half) / half)^j (column scaling
  // leaves the centre-point functional unchanged), thin QR by modified
  // Gram-Schmidt with one re-orthogonalisation pass, then
  // kernel = Q R^{-T} e0 — the same functional as e0^T (X^T X)^{-1} X^T
  // without squaring the condition number of X.
  std::vector<double> Q(static_cast<size_t>(window) * n), Rm(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < window; ++i) {
    double p = 1.0;
    for (int j = 0; j < n; ++j) {
      Q[i * n + j] = p;
      p *= static_cast<double>(i - half) / static_cast<double>(half);
    }
  }
  for (int j = 0; j < n; ++j) {
    for (int pass = 0; pass < 2; ++pass) {
      for (int k = 0; k < j; ++k) {
        double d = 0.0;
        for (int i = 0; i < window; ++i) d += Q[i * n + k] * Q[i * n + j];
        Rm[k * n + j] += d;
        for (int i = 0; i < window; ++i) Q[i * n + j] -= d * Q[i * n + k];
      }
    }
    double nrm = 0.0;
    for (int i = 0; i < window; ++i) nrm += Q[i * n + j] * Q[i * n + j];
    nrm = std::sqrt(nrm);
    Rm[j * n + j] = nrm;
    for (int i = 0; i < window; ++i) Q[i * n + j] /= nrm;
  }
  std::vector<double> z(n, 0.0);  // R^T z = e0 (forward substitution)
  for (int j = 0; j < n; ++j) {
    double s = (j == 0) ? 1.0 : 0.0;
    for (int k = 0; k < j; ++k) s -= Rm[k * n + j] * z[k];
    z[j] = s / Rm[j * n + j];
  }
  std::vector<double> coeffs(window);
  for (int i = 0; i < window; ++i) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += Q[i * n + j] * z[j];
    coeffs[i] = s;
  }
  return coeffs;
}

// reflect_index (smoothing.cpp:37-44)
inline int reflect_index(int i, int n) {
  if (n == 1) return 0;
  while (i < 0 || i >= n) {
    if (i < 0) i = -i;
    if (i >= n) i = 2 * (n - 1) - i;
  }
  return i;
}

// sg_smooth (smoothing.cpp:48-65); seq row-major n x m.
template <class R>
std::vector<R> sg_smooth(const std::vector<R>& seq, int n, int m, const std::vector<R>& coeffs) {
  if (n < 1) throw std::invalid_argument("sg_smooth: empty sequence");
  const int half = static_cast<int>(coeffs.size()) / 2;
  std::vector<R> out(static_cast<size_t>(n) * m);
  for (int c = 0; c < m; ++c) {
    for (int i = 0; i < n; ++i) {
      R acc = 0;
      for (int j = -half; j <= half; ++j) acc += coeffs[j + half] * seq[reflect_index(i + j, n) * m + c];
      out[i * m + c] = acc;
    }
  }
  return out;
}

// WeightResult / it_weights (weights.hpp:9-17, weights.cpp:8-25)
template <class R>
struct Weights {
  std::vector<R> w;
  R rho = 0, normalizer = 0;
};
template <class R>
Weights<R> it_weights(const std::vector<R>& costs, R lambda) {
  const int K = static_cast<int>(costs.size());
  if (K < 1) throw std::invalid_argument("it_weights: need at least one cost");
  if (!(lambda > R(0))) throw std::invalid_argument("it_weights: lambda must be > 0");
  for (R c : costs)
    if (!std::isfinite(c)) throw NonFinite("it_weights: non-finite cost");
  Weights<R> r;
  r.rho = *std::min_element(costs.begin(), costs.end());
  r.w.resize(K);
  R eta = 0;
  for (int k = 0; k < K; ++k) {
    r.w[k] = std::exp(-(costs[k] - r.rho) / lambda);
    eta += r.w[k];
  }
  r.normalizer = eta;
  for (auto& x : r.w) x /= eta;
  return r;
}

// cem_weights (weights.cpp:27-53): the lround(K (1 - delta)) lowest costs,
// ties broken by ascending sample index, each weighted 1 / elite.
template <class R>
Weights<R> cem_weights(const std::vector<R>& costs, double delta) {
  const int K = static_cast<int>(costs.size());
  if (K < 1) throw std::invalid_argument("cem_weights: need at least one cost");
  if (!(delta > 0.0 && delta < 1.0)) throw std::invalid_argument("cem_weights: delta must be in (0, 1)");
  for (R c : costs)
    if (!std::isfinite(c)) throw NonFinite("cem_weights: non-finite cost");
  const int elite = static_cast<int>(std::lround(K * (1.0 - delta)));
  if (elite < 1) throw std::invalid_argument("cem_weights: delta leaves an empty elite set");
  std::vector<int> order(K);
  for (int k = 0; k < K; ++k) order[k] = k;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    if (costs[a] != costs[b]) return costs[a] < costs[b];
    return a < b;
  });
  Weights<R> r;
  r.rho = costs[order.front()];
  r.normalizer = static_cast<R>(elite);
  r.w.assign(K, R(0));
  for (int i = 0; i < elite; ++i) r.w[order[i]] = R(1) / static_cast<R>(elite);
  return r;
}

// ControllerState (controller.hpp:40-58) + the data the device handle owns.
template <class R>
struct Controller {
  mppi_gpu_config cfg{};
  Sampling p;
  std::vector<R> plan;  // T x m row-major
  uint64_t iteration = 0;
  std::vector<double> sg;  // empty = no filter
  std::vector<R> sg_r;
  R lo[2], hi[2];
  Mlp<R> mlp;
  Map<R> map;
  Cost<R> cost;
  std::vector<R> injected;   // reference layout, INJECTED mode
  Batch<R> last_batch;       // batch of the last rollout (post-mutation)
  std::vector<R> theta;  // basis-function model coeffs, theta[b*4 + o]
  Bicycle<R> bike;       // bicycle truth model parameters
  bool has_mlp = false, has_map = false;

  int T() const { return p.horizon_steps; }

  System<R> system() const {
    if (cfg.system == MPPI_SYSTEM_QUADRATIC)
      return make_quadratic_system<R>(2, static_cast<R>(p.dt), static_cast<R>(cfg.quad_cost_scale));
    if (!has_mlp) throw std::invalid_argument("vehicle system: model (MLP weights / basis Theta) not set");
    if (!has_map) throw std::invalid_argument("vehicle system: costmap not set");
    if (cfg.system == MPPI_SYSTEM_VEHICLE_BASIS)
      return make_basis_system<R>(theta, lo, hi, map, cost, static_cast<R>(p.dt), p.horizon_steps,
                                  cfg.with_terminal != 0);
    if (cfg.system == MPPI_SYSTEM_VEHICLE_BICYCLE)
      return make_bicycle_system<R>(bike, lo, hi, map, cost, static_cast<R>(p.dt), p.horizon_steps,
                                    cfg.with_terminal != 0);
    return make_vehicle_system<R>(mlp, lo, hi, map, cost, static_cast<R>(p.dt), p.horizon_steps,
                                  cfg.with_terminal != 0);
  }

  Batch<R> sample(uint64_t it) const {
    if (cfg.noise_mode == MPPI_NOISE_INJECTED) {
      if (injected.empty()) throw std::invalid_argument("INJECTED noise: no batch set");
      Batch<R> b;
      b.K = p.samples; b.T = p.horizon_steps; b.m = 2;
      b.eps = injected;
      b.flags.assign(b.K, 0);
      const int nz = p.n_zero_mean();
      for (int k = b.K - nz; k < b.K; ++k) b.flags[k] = 1;
      return b;
    }
    return sample_perturbations<R>(p, it, cfg.noise_mode);
  }

  // rollout_batch (controller.cpp:55-109).  Mixed precision as on the
  // device: per-step terms in R, the T-term cost sum in double.
  std::vector<double> rollout_batch(const System<R>& sys, const R* x0, Batch<R>& batch,
                               int n_threads) const {
    p.validate();
    const int K = batch.K, T = p.horizon_steps, m = sys.control_dim;
    // zero-mean rewrite eps_k -= U (controller.cpp:70-72)
    for (int k = 0; k < K; ++k)
      if (batch.flags[k])
        for (int t = 0; t < T; ++t)
          for (int c = 0; c < m; ++c) batch.at(k, t, c) -= plan[t * m + c];
    const R lambda = static_cast<R>(p.lambda), gamma = static_cast<R>(p.gamma);
    const R sig[2] = {static_cast<R>(p.sigma_diag[0]), static_cast<R>(p.sigma_diag[1])};
    std::vector<double> costs(K);
    parallel_for_chunks(K, n_threads, [&](int begin, int end) {
      std::vector<R> x(sys.state_dim), xn(sys.state_dim);
      R u[2], v[2];
      for (int k = begin; k < end; ++k) {
        for (int i = 0; i < sys.state_dim; ++i) x[i] = x0[i];
        const bool zero_mean = batch.flags[k] != 0;
        double cost = 0;
        for (int t = 0; t < T; ++t) {
          R uv = 0, uu = 0;
          for (int c = 0; c < m; ++c) {
            u[c] = plan[t * m + c];
            v[c] = u[c] + batch.at(k, t, c);
            uv += u[c] * v[c] / sig[c];
            uu += u[c] * u[c] / sig[c];
          }
          sys.step(x.data(), v, t, xn.data());
          x.swap(xn);
          const R coupling =
              zero_mean ? (gamma - lambda) * uv + R(0.5) * lambda * uu : gamma * uv;
          cost += static_cast<double>(sys.running_cost(x.data(), t) + coupling);
        }
        cost += static_cast<double>(sys.terminal_cost(x.data()));
        costs[k] = cost;
      }
    });
    return costs;
  }

  // update_plan (controller.cpp:118-131): ascending k, skipping zero weights.
  // The aggregate and its smoothing are double; U' = U + agg is rounded once
  // to R (the device does the same).
  std::vector<R> update_plan(const Batch<R>& batch, const std::vector<double>& w) const {
    const int K = batch.K, T = p.horizon_steps;
    if (static_cast<int>(w.size()) != K)
      throw std::invalid_argument("update_plan: weight/sample count mismatch");
    std::vector<double> agg(static_cast<size_t>(T) * 2, 0.0);
    for (int k = 0; k < K; ++k) {
      if (w[k] == 0.0) continue;
      for (int t = 0; t < T; ++t)
        for (int c = 0; c < 2; ++c) agg[t * 2 + c] += w[k] * static_cast<double>(batch.at(k, t, c));
    }
    if (!sg.empty()) agg = sg_smooth<double>(agg, T, 2, sg);
    std::vector<R> out(plan);
    for (size_t i = 0; i < out.size(); ++i) {
      out[i] = static_cast<R>(static_cast<double>(plan[i]) + agg[i]);
      if (!std::isfinite(out[i]))
        throw std::invalid_argument("ControlPlan: needs a finite T x m matrix, T >= 1");
    }
    return out;
  }

  // compute_weights (controller.cpp:111-116): IT or CEM by the weight rule.
  Weights<double> compute_weights(const std::vector<double>& costs) const {
    if (cfg.weight_rule == MPPI_WEIGHT_CEM) return cem_weights<double>(costs, cfg.cem_delta);
    return it_weights<double>(costs, p.lambda);
  }

  // mpc_step (controller.cpp:133-148)
  void mpc_step(const R* x0, R u0[2], int n_threads) {
    const System<R> sys = system();
    Batch<R> batch = sample(iteration);
    const std::vector<double> costs = rollout_batch(sys, x0, batch, n_threads);
    const Weights<double> w = compute_weights(costs);
    plan = update_plan(batch, w.w);
    for (int c = 0; c < 2; ++c) u0[c] = clampv(plan[c], lo[c], hi[c]);
    const int T = p.horizon_steps;
    for (int t = 0; t + 1 < T; ++t)
      for (int c = 0; c < 2; ++c) plan[t * 2 + c] = plan[(t + 1) * 2 + c];
    for (int c = 0; c < 2; ++c) plan[(T - 1) * 2 + c] = R(0);
    ++iteration;
    last_batch = std::move(batch);
  }

  // optimize_to_convergence (controller.cpp:150-164)
  void optimize(const R* x0, int iterations, int n_threads) {
    if (iterations < 1)
      throw std::invalid_argument("optimize_to_convergence: iterations must be >= 1");
    const System<R> sys = system();
    for (int i = 0; i < iterations; ++i) {
      Batch<R> batch = sample(iteration);
      const std::vector<double> costs = rollout_batch(sys, x0, batch, n_threads);
      const Weights<double> w = compute_weights(costs);
      plan = update_plan(batch, w.w);
      ++iteration;
    }
  }
};

template <class R>
Cost<R> make_cost(const mppi_cost_params& c, int T) {
  Cost<R> r;
  r.alpha_track = static_cast<R>(c.alpha_track);
  r.alpha_speed = static_cast<R>(c.alpha_speed);
  r.alpha_stab = static_cast<R>(c.alpha_stab);
  r.v_des = static_cast<R>(c.v_des);
  r.impulse = static_cast<R>(c.impulse);
  r.decay = static_cast<R>(c.decay);
  r.boundary_threshold = static_cast<R>(c.boundary_threshold);
  r.slip_limit = static_cast<R>(c.slip_limit);
  r.crash_penalty = static_cast<R>(c.crash_penalty);
  r.crash_threshold = static_cast<R>(c.crash_threshold);
  r.roll_limit = static_cast<R>(c.roll_limit);
  r.decay_pow.resize(T + 1);
  for (int t = 0; t <= T; ++t) r.decay_pow[t] = static_cast<R>(std::pow(c.decay, t));
  return r;
}

struct AnyController {
  int precision = MPPI_FP64;
  std::unique_ptr<Controller<double>> d;
  std::unique_ptr<Controller<float>> f;
};

template <class R>
void configure(Controller<R>& c, const mppi_gpu_config& cfg) {
  c.cfg = cfg;
  c.p.samples = cfg.samples;
  c.p.horizon_steps = cfg.horizon_steps;
  c.p.dt = cfg.dt;
  c.p.sigma_diag[0] = cfg.sigma_diag[0];
  c.p.sigma_diag[1] = cfg.sigma_diag[1];
  c.p.lambda = cfg.lambda;
  c.p.gamma = cfg.gamma;
  c.p.explore_fraction = cfg.explore_fraction;
  c.p.seed = cfg.seed;
  c.p.validate();
  for (int i = 0; i < 2; ++i) {
    if (!(cfg.bounds_lower[i] < cfg.bounds_upper[i]))
      throw std::invalid_argument("ControlBounds: lower must be < upper");
    c.lo[i] = static_cast<R>(cfg.bounds_lower[i]);
    c.hi[i] = static_cast<R>(cfg.bounds_upper[i]);
  }
  if (cfg.sg_window != 0) {
    c.sg = sg_coefficients(cfg.sg_window, cfg.sg_degree);
    c.sg_r.assign(c.sg.begin(), c.sg.end());
  }
  c.plan.assign(static_cast<size_t>(cfg.horizon_steps) * 2, R(0));
  c.cost = make_cost<R>(cfg.cost, cfg.horizon_steps);
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return MPPI_OK;
  } catch (const NonFinite& e) {
    g_last_error = e.what();
    return MPPI_ERR_NONFINITE;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return MPPI_ERR_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    g_last_error = e.what();
    return MPPI_ERR_DOMAIN;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MPPI_ERR_RUNTIME;
  }
}

template <class F>
int dispatch(AnyController* h, F&& f) {
  if (!h) {
    g_last_error = "null oracle handle";
    return MPPI_ERR_INVALID_ARGUMENT;
  }
  return guard([&] {
    if (h->precision == MPPI_FP64) f(*h->d);
    else f(*h->f);
  });
}

}  // namespace orc

// ============================================================ C API ==========
using orc::AnyController;

extern "C" {

const char* oracle_last_error(void) { return orc::g_last_error.c_str(); }
void oracle_set_mlp_order(int order) { orc::g_mlp_order = order; }

uint64_t oracle_splitmix64(uint64_t x) { return orc::splitmix64(x); }
uint64_t oracle_counter_hash(uint64_t seed, uint64_t stream, uint64_t it, uint64_t k, uint64_t t,
                             uint64_t pair) {
  return orc::counter_hash(seed, stream, it, k, t, pair);
}
double oracle_counter_normal(uint64_t seed, uint64_t stream, uint64_t it, uint64_t k, uint64_t t,
                             int component) {
  return orc::counter_normal(seed, stream, it, k, t, component);
}
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  orc::philox4x32_10(ctr, key, out);
}

// sample_perturbations with a bare SamplingParams description; m in {1, 2}.
int oracle_sample_perturbations(int K, int T, int m, const double* sigma_diag,
                                double explore_fraction, uint64_t seed, uint64_t iteration,
                                int noise_mode, double* eps_out, uint8_t* flags_out) {
  return orc::guard([&] {
    orc::Sampling p;
    p.samples = K;
    p.horizon_steps = T;
    p.m = m;
    if (m < 1 || m > 2) throw std::invalid_argument("oracle: m must be 1 or 2");
    for (int c = 0; c < m; ++c) p.sigma_diag[c] = sigma_diag[c];
    p.explore_fraction = explore_fraction;
    p.seed = seed;
    const auto b = orc::sample_perturbations<double>(p, iteration, noise_mode);
    std::memcpy(eps_out, b.eps.data(), b.eps.size() * sizeof(double));
    if (flags_out) std::memcpy(flags_out, b.flags.data(), b.flags.size());
  });
}

int oracle_sg_coefficients(int window, int degree, double* out) {
  return orc::guard([&] {
    const auto c = orc::sg_coefficients(window, degree);
    std::copy(c.begin(), c.end(), out);
  });
}
int oracle_sg_smooth(const double* seq, int n, int m, const double* coeffs, int window,
                     double* out) {
  return orc::guard([&] {
    std::vector<double> s(seq, seq + static_cast<size_t>(n) * m);
    std::vector<double> c(coeffs, coeffs + window);
    const auto o = orc::sg_smooth<double>(s, n, m, c);
    std::copy(o.begin(), o.end(), out);
  });
}
int oracle_it_weights(const double* costs, int K, double lambda, double* w_out, double* rho,
                      double* eta) {
  return orc::guard([&] {
    std::vector<double> c(costs, costs + std::max(K, 0));
    const auto r = orc::it_weights<double>(c, lambda);
    std::copy(r.w.begin(), r.w.end(), w_out);
    *rho = r.rho;
    *eta = r.normalizer;
  });
}
int oracle_cem_weights(const double* costs, int K, double delta, double* w_out, double* rho, double* eta) {
  return orc::guard([&] {
    std::vector<double> c(costs, costs + std::max(K, 0));
    const auto r = orc::cem_weights<double>(c, delta);
    std::copy(r.w.begin(), r.w.end(), w_out);
    *rho = r.rho;
    *eta = r.normalizer;
  });
}
int oracle_it_weights_f32(const float* costs, int K, float lambda, float* w_out, float* rho,
                          float* eta) {
  return orc::guard([&] {
    std::vector<float> c(costs, costs + std::max(K, 0));
    const auto r = orc::it_weights<float>(c, lambda);
    std::copy(r.w.begin(), r.w.end(), w_out);
    *rho = r.rho;
    *eta = r.normalizer;
  });
}

// Standalone model / cost pieces (double) for the dynamics and cost pins.
int oracle_mlp_forward(int H, const double* w1, const double* b1, const double* w2,
                       const double* b2, const double* w3, const double* b3, const double in[6],
                       double out[4]) {
  return orc::guard([&] {
    if (H != 32 && H != 64) throw std::invalid_argument("mlp: hidden must be 32 or 64");
    orc::Mlp<double> m;
    m.H = H;
    m.w1.assign(w1, w1 + H * 6); m.b1.assign(b1, b1 + H);
    m.w2.assign(w2, w2 + H * H); m.b2.assign(b2, b2 + H);
    m.w3.assign(w3, w3 + 4 * H); m.b3.assign(b3, b3 + 4);
    orc::mlp_forward<double>(in, m, out);
  });
}
int oracle_advance_split(const double x[7], const double d[4], double dt, double out[7]) {
  return orc::guard([&] {
    if (!(dt > 0.0)) throw std::invalid_argument("step: dt must be > 0");
    orc::advance_split<double>(x, d, dt, out);
  });
}
int oracle_clamp_controls(const double* v, const double* lo, const double* hi, int n,
                          double* out) {
  return orc::guard([&] {
    for (int i = 0; i < n; ++i) {
      if (!(lo[i] < hi[i])) throw std::invalid_argument("ControlBounds: lower must be < upper");
      out[i] = orc::clampv(v[i], lo[i], hi[i]);
    }
  });
}
static orc::Map<double> make_map(const double* values, int W, int H, double x0, double y0,
                                 double res) {
  if (W < 2 || H < 2) throw std::invalid_argument("CostMap: width and height must be >= 2");
  if (!(res > 0.0)) throw std::invalid_argument("CostMap: resolution must be > 0");
  orc::Map<double> m;
  m.width = W; m.height = H; m.x0 = x0; m.y0 = y0; m.res = res; m.inv_res = 1.0 / res;
  m.v.assign(values, values + static_cast<size_t>(W) * H);
  for (double v : m.v)
    if (!std::isfinite(v) || std::abs(v) > 2.5)
      throw std::invalid_argument("CostMap: values must be finite and within +-2.5");
  return m;
}
int oracle_costmap_lookup(const double* values, int W, int H, double x0, double y0, double res,
                          double px, double py, double* out) {
  return orc::guard([&] { *out = orc::costmap_lookup(make_map(values, W, H, x0, y0, res), px, py); });
}
int oracle_state_cost(const double x[7], int t, const double* values, int W, int H, double x0,
                      double y0, double res, const mppi_cost_params* cp, double* out) {
  return orc::guard([&] {
    const auto m = make_map(values, W, H, x0, y0, res);
    const auto c = orc::make_cost<double>(*cp, std::max(t, 0));
    *out = orc::state_cost<double>(x, t, m, c);
  });
}
double oracle_side_slip(double vx, double vy) { return orc::side_slip<double>(vx, vy); }

// ---- controller handle ------------------------------------------------------
int oracle_create(const mppi_gpu_config* cfg, AnyController** out) {
  return orc::guard([&] {
    if (!cfg || !out) throw std::invalid_argument("oracle_create: null argument");
    auto h = std::make_unique<AnyController>();
    h->precision = cfg->precision;
    if (cfg->precision == MPPI_FP64) {
      h->d = std::make_unique<orc::Controller<double>>();
      orc::configure(*h->d, *cfg);
    } else {
      h->f = std::make_unique<orc::Controller<float>>();
      orc::configure(*h->f, *cfg);
    }
    *out = h.release();
  });
}
void oracle_destroy(AnyController* h) { delete h; }

int oracle_set_mlp(AnyController* h, int H, const double* w1, const double* b1, const double* w2,
                   const double* b2, const double* w3, const double* b3) {
  return orc::dispatch(h, [&](auto& c) {
    using R = typename std::decay_t<decltype(c.plan)>::value_type;
    if (H != 32 && H != 64) throw std::invalid_argument("mlp: hidden must be 32 or 64");
    c.mlp.H = H;
    c.mlp.w1.assign(w1, w1 + H * 6); c.mlp.b1.assign(b1, b1 + H);
    c.mlp.w2.assign(w2, w2 + H * H); c.mlp.b2.assign(b2, b2 + H);
    c.mlp.w3.assign(w3, w3 + 4 * H); c.mlp.b3.assign(b3, b3 + 4);
    (void)sizeof(R);
    c.has_mlp = true;
  });
}
int oracle_set_theta(AnyController* h, const double* theta) {
  return orc::dispatch(h, [&](auto& c) {
    using R = typename std::decay_t<decltype(c.plan)>::value_type;
    c.theta.resize(100);
    for (int i = 0; i < 100; ++i) {
      if (!std::isfinite(theta[i])) throw std::invalid_argument("load_theta: non-finite entry");
      c.theta[i] = static_cast<R>(theta[i]);
    }
    c.has_mlp = true;
  });
}
int oracle_set_bicycle(AnyController* h, const double p[9]) {
  return orc::dispatch(h, [&](auto& c) {
    using R = typename std::decay_t<decltype(c.plan)>::value_type;
    for (int i = 0; i < 9; ++i)
      if (!(p[i] > 0.0) || !std::isfinite(p[i])) throw std::invalid_argument("BicycleParams: all parameters must be positive");
    c.bike = orc::Bicycle<R>{static_cast<R>(p[0]), static_cast<R>(p[1]), static_cast<R>(p[2]), static_cast<R>(p[3]),
                             static_cast<R>(p[4]), static_cast<R>(p[5]), static_cast<R>(p[6]), static_cast<R>(p[7]),
                             static_cast<R>(p[8])};
    c.has_mlp = true;
  });
}
// brush_tire_force / step_bicycle_truth in double (the reference pins); 4 = domain_error
int oracle_brush_tire_force(double alpha, double u_F, const double p[9], double* out) {
  const orc::Bicycle<double> b{p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8]};
  try {
    *out = orc::brush_tire_force<double>(alpha, u_F, b);
  } catch (const std::domain_error& e) {
    orc::g_last_error = e.what();
    return MPPI_ERR_DOMAIN;
  }
  return 0;
}
int oracle_step_bicycle(const double x[7], const double v[2], double dt, const double p[9], double out[7]) {
  const orc::Bicycle<double> b{p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8]};
  return orc::guard([&] { orc::step_bicycle<double>(x, v, dt, b, out); });
}
// eval_basis (dynamics.cpp:83-133) in double: x_d = (roll, v_x, v_y, r), v = (steer, throttle).
int oracle_eval_basis(const double x_d[4], const double v[2], double phi[25]) {
  orc::eval_basis<double>(x_d[0], x_d[1], x_d[2], x_d[3], v[0], v[1], phi);
  return 0;
}
// step_basis_model (dynamics.cpp:152-157) in double (no clamp: the reference
// step takes the already-clamped input).
int oracle_step_basis(const double x[7], const double v[2], double dt, const double theta[100], double out[7]) {
  if (!(dt > 0.0)) return 1;
  double phi[25], d[4];
  orc::eval_basis<double>(x[3], x[4], x[5], x[6], v[0], v[1], phi);
  orc::basis_dot<double>(theta, phi, d);
  orc::advance_split<double>(x, d, dt, out);
  return 0;
}
int oracle_set_costmap(AnyController* h, const double* values, int W, int H, double x0,
                       double y0, double res) {
  return orc::dispatch(h, [&](auto& c) {
    using R = typename std::decay_t<decltype(c.plan)>::value_type;
    const auto m = make_map(values, W, H, x0, y0, res);
    c.map.width = W; c.map.height = H;
    c.map.x0 = static_cast<R>(x0); c.map.y0 = static_cast<R>(y0);
    c.map.res = static_cast<R>(res); c.map.inv_res = static_cast<R>(1.0 / res);
    c.map.v.assign(m.v.begin(), m.v.end());
    c.has_map = true;
  });
}
int oracle_set_costmap_f32(AnyController* h, const float* values, int W, int H, double x0,
                           double y0, double res) {
  std::vector<double> v(values, values + static_cast<size_t>(std::max(W, 0)) * std::max(H, 0));
  return oracle_set_costmap(h, v.data(), W, H, x0, y0, res);
}
int oracle_set_plan(AnyController* h, const double* U) {
  return orc::dispatch(h, [&](auto& c) {
    for (size_t i = 0; i < c.plan.size(); ++i) {
      if (!std::isfinite(U[i])) throw std::invalid_argument("ControlPlan: non-finite");
      c.plan[i] = static_cast<typename std::decay_t<decltype(c.plan)>::value_type>(U[i]);
    }
  });
}
int oracle_get_plan(AnyController* h, double* U) {
  return orc::dispatch(h, [&](auto& c) {
    for (size_t i = 0; i < c.plan.size(); ++i) U[i] = static_cast<double>(c.plan[i]);
  });
}
int oracle_set_iteration(AnyController* h, uint64_t it) {
  return orc::dispatch(h, [&](auto& c) { c.iteration = it; });
}
int oracle_get_iteration(AnyController* h, uint64_t* it) {
  return orc::dispatch(h, [&](auto& c) { *it = c.iteration; });
}
int oracle_set_noise(AnyController* h, const double* eps) {
  return orc::dispatch(h, [&](auto& c) {
    const size_t n = static_cast<size_t>(c.p.samples) * 2 * c.p.horizon_steps;
    c.injected.resize(n);
    for (size_t i = 0; i < n; ++i)
      c.injected[i] = static_cast<typename std::decay_t<decltype(c.plan)>::value_type>(eps[i]);
  });
}

// rollout_batch on the current plan/iteration; eps_in overrides the noise.
int oracle_rollout_costs(AnyController* h, const double* x0, const double* eps_in,
                         double* costs_out, double* eps_stored_out, int n_threads) {
  return orc::dispatch(h, [&](auto& c) {
    using R = typename std::decay_t<decltype(c.plan)>::value_type;
    const auto sys = c.system();
    orc::Batch<R> b;
    if (eps_in) {
      b.K = c.p.samples; b.T = c.p.horizon_steps; b.m = 2;
      b.eps.assign(eps_in, eps_in + static_cast<size_t>(b.K) * 2 * b.T);
      b.flags.assign(b.K, 0);
      const int nz = c.p.n_zero_mean();
      for (int k = b.K - nz; k < b.K; ++k) b.flags[k] = 1;
    } else {
      b = c.sample(c.iteration);
    }
    std::vector<R> x(sys.state_dim);
    for (int i = 0; i < sys.state_dim; ++i) x[i] = static_cast<R>(x0[i]);
    const auto costs = c.rollout_batch(sys, x.data(), b, n_threads);
    for (size_t k = 0; k < costs.size(); ++k) costs_out[k] = costs[k];
    if (eps_stored_out)
      for (size_t i = 0; i < b.eps.size(); ++i) eps_stored_out[i] = static_cast<double>(b.eps[i]);
    c.last_batch = std::move(b);
  });
}
int oracle_weights(AnyController* h, const double* costs, double* w_out, double* rho,
                   double* eta) {
  return orc::dispatch(h, [&](auto& c) {
    std::vector<double> s(costs, costs + c.p.samples);
    const auto r = c.compute_weights(s);
    for (size_t k = 0; k < r.w.size(); ++k) w_out[k] = r.w[k];
    *rho = r.rho;
    *eta = r.normalizer;
  });
}
int oracle_update_plan(AnyController* h, const double* weights) {
  return orc::dispatch(h, [&](auto& c) {
    if (c.last_batch.K == 0) throw std::invalid_argument("update_plan: no rollout batch");
    std::vector<double> w(weights, weights + c.p.samples);
    c.plan = c.update_plan(c.last_batch, w);
  });
}
int oracle_rollout_states(AnyController* h, const double* x0, int sample, double* states_out) {
  return orc::dispatch(h, [&](auto& c) {
    using R = typename std::decay_t<decltype(c.plan)>::value_type;
    if (c.last_batch.K == 0) throw std::invalid_argument("rollout_states: no rollout batch");
    if (sample < 0 || sample >= c.last_batch.K) throw std::invalid_argument("bad sample index");
    const auto sys = c.system();
    const int T = c.p.horizon_steps, n = sys.state_dim;
    std::vector<R> x(n), xn(n);
    for (int i = 0; i < n; ++i) x[i] = static_cast<R>(x0[i]);
    for (int i = 0; i < n; ++i) states_out[i] = static_cast<double>(x[i]);
    for (int t = 0; t < T; ++t) {
      R v[2];
      for (int cc = 0; cc < 2; ++cc)
        v[cc] = c.plan[t * 2 + cc] + c.last_batch.at(sample, t, cc);
      sys.step(x.data(), v, t, xn.data());
      x.swap(xn);
      for (int i = 0; i < n; ++i) states_out[(t + 1) * n + i] = static_cast<double>(x[i]);
    }
  });
}
int oracle_mpc_step(AnyController* h, const double* x0, double* u0_out, int n_threads) {
  return orc::dispatch(h, [&](auto& c) {
    using R = typename std::decay_t<decltype(c.plan)>::value_type;
    const int n = (c.cfg.system == MPPI_SYSTEM_QUADRATIC) ? 2 : 7;
    std::vector<R> x(n);
    for (int i = 0; i < n; ++i) x[i] = static_cast<R>(x0[i]);
    R u0[2];
    c.mpc_step(x.data(), u0, n_threads);
    u0_out[0] = static_cast<double>(u0[0]);
    u0_out[1] = static_cast<double>(u0[1]);
  });
}
int oracle_optimize(AnyController* h, const double* x0, int iterations, int n_threads) {
  return orc::dispatch(h, [&](auto& c) {
    using R = typename std::decay_t<decltype(c.plan)>::value_type;
    const int n = (c.cfg.system == MPPI_SYSTEM_QUADRATIC) ? 2 : 7;
    std::vector<R> x(n);
    for (int i = 0; i < n; ++i) x[i] = static_cast<R>(x0[i]);
    c.optimize(x.data(), iterations, n_threads);
  });
}
// Model step of the vehicle system (the device plant of mppi_gpu_closed_loop).
int oracle_vehicle_step(AnyController* h, const double* x, const double* u, double* x_next) {
  return orc::dispatch(h, [&](auto& c) {
    using R = typename std::decay_t<decltype(c.plan)>::value_type;
    const auto sys = c.system();
    R xr[7], ur[2], xn[7];
    for (int i = 0; i < 7; ++i) xr[i] = static_cast<R>(x[i]);
    for (int i = 0; i < 2; ++i) ur[i] = static_cast<R>(u[i]);
    sys.step(xr, ur, 0, xn);
    for (int i = 0; i < 7; ++i) x_next[i] = static_cast<double>(xn[i]);
  });
}

}  // extern "C"
