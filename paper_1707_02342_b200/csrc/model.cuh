// model.cuh — device rollout systems: the data-described replacement of the
// reference's RolloutSystem callback triple (controller.hpp:18-24).
//
//  * VehicleMlp: make_vehicle_system over MlpModel (controller.cpp:7-35):
//    clamp -> mlp_forward (dynamics.cpp:197-204) -> advance_split
//    (dynamics.cpp:137-148); running cost = state_cost (costs.cpp:29-43) on the
//    post-step state with step index t, terminal = state_cost(x_T, T).
//  * Quadratic: the reference test fixture quadratic_system
//    (test_controller.cpp:23-37), used to run the reference's controller pins
//    against the device path.
#pragma once

#include "common.cuh"

namespace mppi_dev {

// Device layout of MlpWeights (dynamics.hpp:110-119), transposed to
// input-major so that one input feeds consecutive outputs (pairwise FFMA2).
template <class R, int H>
struct alignas(16) MlpParams {
  R w1t[6][H];   // w1t[i][j] = W1[j][i]
  R b1[H];
  R w2t[H][H];   // w2t[i][j] = W2[j][i]
  R b2[H];
  R w3t[H][4];   // w3t[i][o] = W3[o][i]
  R b3[4];
};

// Kernel parameters are limited to 32 KB: fp32 H=32/64 and fp64 H=32 weights
// travel by value (served from the constant bank / uniform registers); fp64
// H=64 (39 KB) is read from global memory.
template <class R, int H>
constexpr bool kWeightsByValue = sizeof(MlpParams<R, H>) <= 24 * 1024;

template <class R, int H, bool ByValue = kWeightsByValue<R, H>>
struct WeightHolder;
template <class R, int H>
struct WeightHolder<R, H, true> {
  MlpParams<R, H> w;
  __device__ __forceinline__ const MlpParams<R, H>& get() const { return w; }
};
template <class R, int H>
struct WeightHolder<R, H, false> {
  const MlpParams<R, H>* p;
  __device__ __forceinline__ const MlpParams<R, H>& get() const { return *p; }
};

// Cost parameters in the arithmetic type (mppi_cost_params, mppi_gpu.h).
template <class R>
struct CostDev {
  R alpha_track, alpha_speed, alpha_stab, v_des, impulse, boundary_threshold, slip_limit,
      crash_penalty, crash_threshold, roll_limit;
};

// Costmap view (costs.hpp:11-38): row-major values[iy*W + ix].
template <class R>
struct MapDev {
  const R* values;
  int width, height;
  R x0, y0, res, inv_res;
};

// costmap_lookup (costs.cpp:7-22): software bilinear with clamp-to-edge.
// (The paper used texture hardware interpolation; its 8-bit
// fixed-point weights would break parity with the reference, so the four taps
// are read through the read-only path and interpolated in R.)
template <class R>
struct MapTaps {
  R v00, v10, v01, v11, fx, fy;
};
template <class R>
__device__ __forceinline__ MapTaps<R> map_fetch(const MapDev<R>& m, R px, R py) {
  R gx, gy;
  if constexpr (std::is_same<R, double>::value) {
    gx = div_r(sub_rn(px, m.x0), m.res);
    gy = div_r(sub_rn(py, m.y0), m.res);
  } else {
    gx = mul_rn(sub_rn(px, m.x0), m.inv_res);
    gy = mul_rn(sub_rn(py, m.y0), m.inv_res);
  }
  gx = clamp_r<R>(gx, R(0), static_cast<R>(m.width - 1));
  gy = clamp_r<R>(gy, R(0), static_cast<R>(m.height - 1));
  int ix = static_cast<int>(gx);  // gx >= 0 (or NaN -> 0): truncation == floor
  int iy = static_cast<int>(gy);
  ix = min(ix, m.width - 2);
  iy = min(iy, m.height - 2);
  if (gx != gx) ix = 0;
  if (gy != gy) iy = 0;
  MapTaps<R> r;
  r.fx = sub_rn(gx, static_cast<R>(ix));
  r.fy = sub_rn(gy, static_cast<R>(iy));
  const R* p = m.values + static_cast<size_t>(iy) * m.width + ix;
  r.v00 = __ldg(p);
  r.v10 = __ldg(p + 1);
  r.v01 = __ldg(p + m.width);
  r.v11 = __ldg(p + m.width + 1);
  return r;
}
template <class R>
__device__ __forceinline__ R map_interp(const MapTaps<R>& q) {
  const R ofx = sub_rn(R(1), q.fx), ofy = sub_rn(R(1), q.fy);
  R s = mul_rn(mul_rn(ofx, ofy), q.v00);
  s = add_rn(s, mul_rn(mul_rn(q.fx, ofy), q.v10));
  s = add_rn(s, mul_rn(mul_rn(ofx, q.fy), q.v01));
  s = add_rn(s, mul_rn(mul_rn(q.fx, q.fy), q.v11));
  return s;
}

// state_cost (costs.cpp:29-43) given h = costmap value at (p_x, p_y), plus the
// BASELINE crash term.  decay_t = decay^t (host std::pow table).
template <class R>
__device__ __forceinline__ R state_cost_h(R h, R roll, R vx, R vy, R decay_t,
                                          const CostDev<R>& cp) {
  R track = h;
  if (h > cp.boundary_threshold) track = add_rn(track, mul_rn(decay_t, cp.impulse));
  const R dv = sub_rn(vx, cp.v_des);
  const R speed = mul_rn(dv, dv);
  R c = add_rn(mul_rn(cp.alpha_track, track), mul_rn(cp.alpha_speed, speed));
  if (cp.alpha_stab != R(0)) {
    // side_slip (costs.cpp:24-27)
    R zeta = R(0);
    if (!(abs_r(vx) < R(0.01))) zeta = -atan_r(div_r(vy, abs_r(vx)));
    R stab = mul_rn(zeta, zeta);
    if (abs_r(zeta) > cp.slip_limit) stab = add_rn(stab, cp.impulse);
    c = add_rn(c, mul_rn(cp.alpha_stab, stab));
  }
  if (cp.crash_penalty != R(0) && (h > cp.crash_threshold || abs_r(roll) > cp.roll_limit))
    c = add_rn(c, cp.crash_penalty);
  return c;
}

// mlp_forward (dynamics.cpp:197-204).  Accumulation starts from the bias and
// runs over inputs in ascending order with FMAs (the oracle does the same).
template <class R, int H>
__device__ __forceinline__ void mlp_forward(const MlpParams<R, H>& w, const R in[6], R out[4]) {
  R h1[H], h2[H];
#pragma unroll
  for (int j = 0; j < H; ++j) h1[j] = w.b1[j];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
#pragma unroll
    for (int j = 0; j < H; ++j) h1[j] = fma_r(w.w1t[i][j], in[i], h1[j]);
  }
#pragma unroll
  for (int j = 0; j < H; ++j) h1[j] = tanh_r(h1[j]);
#pragma unroll
  for (int j = 0; j < H; ++j) h2[j] = w.b2[j];
#pragma unroll
  for (int i = 0; i < H; ++i) {
#pragma unroll
    for (int j = 0; j < H; ++j) h2[j] = fma_r(w.w2t[i][j], h1[i], h2[j]);
  }
#pragma unroll
  for (int j = 0; j < H; ++j) h2[j] = tanh_r(h2[j]);
#pragma unroll
  for (int o = 0; o < 4; ++o) out[o] = w.b3[o];
#pragma unroll
  for (int i = 0; i < H; ++i) {
#pragma unroll
    for (int o = 0; o < 4; ++o) out[o] = fma_r(w.w3t[i][o], h2[i], out[o]);
  }
}

// advance_split (dynamics.cpp:137-148): Euler from the old state.
template <class R>
__device__ __forceinline__ void advance_split(R x[7], const R d[4], R dt) {
  R s, c;
  sincos_r(x[2], &s, &c);
  const R n0 = add_rn(x[0], mul_rn(sub_rn(mul_rn(c, x[4]), mul_rn(s, x[5])), dt));
  const R n1 = add_rn(x[1], mul_rn(add_rn(mul_rn(s, x[4]), mul_rn(c, x[5])), dt));
  const R n2 = add_rn(x[2], mul_rn(x[6], dt));
  x[3] = add_rn(x[3], mul_rn(d[0], dt));
  x[4] = add_rn(x[4], mul_rn(d[1], dt));
  x[5] = add_rn(x[5], mul_rn(d[2], dt));
  x[6] = add_rn(x[6], mul_rn(d[3], dt));
  x[0] = n0;
  x[1] = n1;
  x[2] = n2;
}

// BasisFunctionModel coefficients (dynamics.hpp:75-82): c[b][o] = coeffs(b, o).
template <class R>
struct ThetaDev {
  R c[25][4];
};

// eval_basis (dynamics.cpp:83-133), kSlipGuardSpeed = 0.1 (dynamics.cpp:47).
template <class R>
__device__ __forceinline__ void eval_basis(R roll, R v_x, R v_y, R r, R u_delta, R u_F, R phi[25]) {
  R alpha_f, alpha_r, ratio;
  if (v_x > R(0.1)) {
    ratio = div_r(v_y, v_x);
    alpha_f = atan_r(sub_rn(add_rn(ratio, div_r(mul_rn(R(0.45), r), v_x)), u_delta));
    alpha_r = atan_r(sub_rn(ratio, div_r(mul_rn(R(0.35), r), v_x)));
  } else {
    ratio = R(0);
    alpha_f = -u_delta;
    alpha_r = R(0);
  }
  const R tf = tan_r(alpha_f), tr = tan_r(alpha_r), sd = sin_r(u_delta);
  phi[0] = u_F;
  phi[1] = div_r(v_x, R(10.0));
  phi[2] = div_r(mul_rn(sd, tf), R(1200.0));
  phi[3] = div_r(mul_rn(mul_rn(sd, tf), abs_r(tf)), R(1200.0 * 1200.0));
  phi[4] = div_r(mul_rn(mul_rn(mul_rn(sd, tf), tf), tf), R(1200.0 * 1200.0 * 1200.0));
  phi[5] = div_r(mul_rn(r, v_y), R(25.0));
  phi[6] = div_r(r, R(10.0));
  phi[7] = div_r(v_y, R(10.0));
  phi[8] = sd;
  phi[9] = div_r(ratio, R(40.0));
  phi[10] = div_r(tf, R(1400.0));
  phi[11] = div_r(mul_rn(tf, abs_r(tf)), R(1400.0 * 1400.0));
  phi[12] = div_r(mul_rn(mul_rn(tf, tf), tf), R(1400.0 * 1400.0 * 1400.0));
  phi[13] = div_r(tr, R(40.0));
  phi[14] = div_r(mul_rn(tr, abs_r(tr)), R(40.0 * 40.0));
  phi[15] = div_r(mul_rn(mul_rn(tr, tr), tr), R(40.0 * 40.0 * 40.0));
  phi[16] = div_r(mul_rn(r, v_x), R(50.0));
  phi[17] = roll;
  phi[18] = mul_rn(roll, r);
  phi[19] = div_r(mul_rn(roll, v_x), R(3.0));
  phi[20] = div_r(mul_rn(mul_rn(roll, v_x), r), R(5.0));
  phi[21] = div_r(mul_rn(v_x, v_x), R(100.0));
  phi[22] = div_r(mul_rn(mul_rn(v_x, v_x), v_x), R(1000.0));
  phi[23] = mul_rn(u_F, u_F);
  phi[24] = mul_rn(mul_rn(u_F, u_F), u_F);
}

// BicycleParams (dynamics.hpp:42-62).
template <class R>
struct BicycleDev {
  R mass, yaw_inertia, a, b, stiffness, mu, load, steer_scale, force_scale;
};

// brush_tire_force (dynamics.cpp:23-43), the reference's expression order.
// The |u_F| > mu F_z domain error is excluded once on the host (the throttle
// is clamped to its bounds before the model, mppi_gpu_set_dynamics_bicycle);
// a NaN here would surface as a non-finite cost.
template <class R>
__device__ __forceinline__ R brush_tire_force(R alpha, R u_F, const BicycleDev<R>& p) {
  const R limit = mul_rn(p.mu, p.load);
  if (abs_r(u_F) > limit) return R(NAN);
  const R xi = div_r(sqrt_r(sub_rn(mul_rn(limit, limit), mul_rn(u_F, u_F))), limit);
  if (xi == R(0)) return R(0);
  const R sign = (alpha >= R(0)) ? R(1) : R(-1);
  const R crossover = atan_r(div_r(mul_rn(mul_rn(mul_rn(R(3), xi), p.mu), p.load), p.stiffness));
  if (abs_r(alpha) >= crossover) return mul_rn(mul_rn(mul_rn(-p.mu, xi), p.load), sign);
  const R ta = tan_r(alpha);
  const R c = p.stiffness;
  const R t1 = mul_rn(-c, ta);
  const R t2 = mul_rn(mul_rn(div_r(mul_rn(c, c), mul_rn(mul_rn(mul_rn(R(3), xi), p.mu), p.load)), ta), abs_r(ta));
  // 27 mu mu xi xi load load, multiplied left to right as in the reference
  const R den3 = mul_rn(mul_rn(mul_rn(mul_rn(mul_rn(mul_rn(R(27), p.mu), p.mu), xi), xi), p.load), p.load);
  const R t3 = mul_rn(mul_rn(mul_rn(div_r(mul_rn(mul_rn(c, c), c), den3), ta), ta), ta);
  return sub_rn(add_rn(t1, t2), t3);
}

// step_bicycle_truth (dynamics.cpp:51-81) on the 7-state (roll unchanged),
// kSlipGuardSpeed = 0.1 (dynamics.cpp:47); v is the applied (clamped) input.
template <class R>
__device__ __forceinline__ void step_bicycle(R x[7], R steer, R throttle, R dt, const BicycleDev<R>& p) {
  const R u_delta = mul_rn(p.steer_scale, steer);
  const R u_F = mul_rn(p.force_scale, throttle);
  const R r = x[6];
  R alpha_f, alpha_r;
  if (x[4] > R(0.1)) {
    const R beta = div_r(x[5], x[4]);
    alpha_f = sub_rn(atan_r(add_rn(beta, div_r(mul_rn(p.a, r), x[4]))), u_delta);
    alpha_r = atan_r(sub_rn(beta, div_r(mul_rn(p.b, r), x[4])));
  } else {
    alpha_f = -u_delta;
    alpha_r = R(0);
  }
  const R f_yf = brush_tire_force<R>(alpha_f, u_F, p);
  const R f_yr = brush_tire_force<R>(alpha_r, u_F, p);
  R s, c;
  sincos_r(x[2], &s, &c);
  const R n0 = add_rn(x[0], mul_rn(sub_rn(mul_rn(c, x[4]), mul_rn(s, x[5])), dt));
  const R n1 = add_rn(x[1], mul_rn(add_rn(mul_rn(s, x[4]), mul_rn(c, x[5])), dt));
  const R n2 = add_rn(x[2], mul_rn(r, dt));
  const R n4 = add_rn(x[4], mul_rn(add_rn(div_r(sub_rn(u_F, mul_rn(f_yf, sin_r(u_delta))), p.mass), mul_rn(r, x[5])), dt));
  const R n5 = add_rn(x[5], mul_rn(sub_rn(div_r(add_rn(f_yf, f_yr), p.mass), mul_rn(r, x[4])), dt));
  const R n6 = add_rn(x[6], mul_rn(div_r(sub_rn(mul_rn(p.a, f_yf), mul_rn(p.b, f_yr)), p.yaw_inertia), dt));
  x[0] = n0;
  x[1] = n1;
  x[2] = n2;
  x[4] = n4;
  x[5] = n5;
  x[6] = n6;
}

// Everything a rollout system needs besides the weights.
template <class R>
struct SystemArgs {
  R dt;
  R lo0, lo1, hi0, hi1;  // ControlBounds
  CostDev<R> cost;
  const R* decay_pow;    // T+1 entries
  int with_terminal;
  R quad_cost_scale;
  ThetaDev<R> theta;     // VEHICLE_BASIS coefficients
  BicycleDev<R> bike;    // VEHICLE_BICYCLE parameters
};

template <class R, int H>
struct VehicleMlp {
  static constexpr int kStateDim = 7;
  static constexpr bool kHasMap = true;
  static constexpr bool kMlp = true;
  // step (controller.cpp:13-20): clamp then MlpModel::step
  __device__ __forceinline__ static void step(R x[7], R v0, R v1, const MlpParams<R, H>& w,
                                              const SystemArgs<R>& a) {
    const R in[6] = {x[3], x[4], x[5], x[6], clamp_r(v0, a.lo0, a.hi0), clamp_r(v1, a.lo1, a.hi1)};
    R d[4];
    mlp_forward<R, H>(w, in, d);
    advance_split<R>(x, d, a.dt);
  }
};

// make_vehicle_system over BasisFunctionModel: clamp -> step_basis_model
// (dynamics.cpp:152-157): xd_dot = Theta^T phi summed over the basis functions
// in ascending order (the oracle does the same; Eigen's GEMV order is not
// reproduced, see oracle/mppi_oracle.cpp), then advance_split.
template <class R, int H>
struct VehicleBasis {
  static constexpr int kStateDim = 7;
  static constexpr bool kHasMap = true;
  static constexpr bool kMlp = false;
  __device__ __forceinline__ static void step(R x[7], R v0, R v1, const MlpParams<R, H>&, const SystemArgs<R>& a) {
    R phi[25];
    eval_basis<R>(x[3], x[4], x[5], x[6], clamp_r(v0, a.lo0, a.hi0), clamp_r(v1, a.lo1, a.hi1), phi);
    R d[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      R acc = mul_rn(a.theta.c[0][o], phi[0]);
#pragma unroll
      for (int b = 1; b < 25; ++b) acc = add_rn(acc, mul_rn(a.theta.c[b][o], phi[b]));
      d[o] = acc;
    }
    advance_split<R>(x, d, a.dt);
  }
};

// make_vehicle_system over BicycleTruthModel: clamp -> step_bicycle_truth.
template <class R, int H>
struct VehicleBicycle {
  static constexpr int kStateDim = 7;
  static constexpr bool kHasMap = true;
  static constexpr bool kMlp = false;
  __device__ __forceinline__ static void step(R x[7], R v0, R v1, const MlpParams<R, H>&, const SystemArgs<R>& a) {
    step_bicycle<R>(x, clamp_r(v0, a.lo0, a.hi0), clamp_r(v1, a.lo1, a.hi1), a.dt, a.bike);
  }
};

template <class R, int H>
struct Quadratic {
  static constexpr int kStateDim = 2;
  static constexpr bool kHasMap = false;
  static constexpr bool kMlp = false;
  __device__ __forceinline__ static void step(R x[7], R v0, R v1, const MlpParams<R, H>&,
                                              const SystemArgs<R>& a) {
    x[0] = add_rn(x[0], mul_rn(v0, a.dt));
    x[1] = add_rn(x[1], mul_rn(v1, a.dt));
  }
  __device__ __forceinline__ static R cost(const R x[7], const SystemArgs<R>& a) {
    R acc = R(0);
    acc = add_rn(acc, mul_rn(x[0], x[0]));
    acc = add_rn(acc, mul_rn(x[1], x[1]));
    return mul_rn(a.quad_cost_scale, acc);
  }
};

}  // namespace mppi_dev
