// workload.cpp — host-side generators of the BASELINE.json synthetic inputs
// (no GPU needed): seeded Xavier MLP weights, the elliptical-track costmap,
// initial states on the centreline, and the SG kernel export.
//
// All randomness is a pure function of the seed through the reference's
// counter hash (sampler.hpp:15-54) on private stream ids, so every artefact is
// reproducible and independent of thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <thread>
#include <vector>

#include "../../include/mppi_gpu.h"
#include "host_util.hpp"

namespace {

inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
inline uint64_t hash4(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ stream);
  h = splitmix64(h ^ a);
  return splitmix64(h ^ b);
}
inline double uniform01(uint64_t h) { return static_cast<double>(h >> 11) * 0x1.0p-53; }
inline double normal(uint64_t h) {
  const double u1 = static_cast<double>((h >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(splitmix64(h) >> 11) * 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

constexpr uint64_t kStreamXavier = 0x7861766965720000ull;   // "xavier"
constexpr uint64_t kStreamInit = 0x696e697473746174ull;     // "initstat"

template <class F>
int guard(F&& f) {
  try {
    f();
    return MPPI_OK;
  } catch (const std::invalid_argument& e) {
    mppi_host::last_error() = e.what();
    return MPPI_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    mppi_host::last_error() = e.what();
    return MPPI_ERR_RUNTIME;
  }
}

// Robust point-to-ellipse distance (bisection on the root of the
// orthogonality condition; e0 >= e1 > 0, query in the first quadrant).
double ellipse_root(double r0, double z0, double z1, double g) {
  const double n0 = r0 * z0;
  double s0 = z1 - 1.0;
  double s1 = (g < 0.0) ? 0.0 : std::hypot(n0, z1) - 1.0;
  double s = 0.0;
  for (int i = 0; i < 1100; ++i) {
    s = 0.5 * (s0 + s1);
    if (s == s0 || s == s1) break;
    const double ratio0 = n0 / (s + r0), ratio1 = z1 / (s + 1.0);
    g = ratio0 * ratio0 + ratio1 * ratio1 - 1.0;
    if (g > 0.0) s0 = s;
    else if (g < 0.0) s1 = s;
    else break;
  }
  return s;
}
double ellipse_distance(double e0, double e1, double y0, double y1) {
  y0 = std::abs(y0);
  y1 = std::abs(y1);
  if (y1 > 0.0) {
    if (y0 > 0.0) {
      const double z0 = y0 / e0, z1 = y1 / e1;
      const double g = z0 * z0 + z1 * z1 - 1.0;
      if (g == 0.0) return 0.0;
      const double r0 = (e0 / e1) * (e0 / e1);
      const double sbar = ellipse_root(r0, z0, z1, g);
      const double x0 = r0 * y0 / (sbar + r0), x1 = y1 / (sbar + 1.0);
      return std::hypot(x0 - y0, x1 - y1);
    }
    return std::abs(y1 - e1);
  }
  const double numer0 = e0 * y0, denom0 = e0 * e0 - e1 * e1;
  if (numer0 < denom0) {
    const double xde0 = numer0 / denom0;
    const double x0 = e0 * xde0, x1 = e1 * std::sqrt(1.0 - xde0 * xde0);
    return std::hypot(x0 - y0, x1);
  }
  return std::abs(y0 - e0);
}

}  // namespace

extern "C" {

int mppi_workload_mlp_xavier(int hidden, uint64_t seed, double out_scale, double* w1, double* b1,
                             double* w2, double* b2, double* w3, double* b3) {
  return guard([&] {
    if (hidden < 1) throw std::invalid_argument("hidden must be >= 1");
    if (!w1 || !b1 || !w2 || !b2 || !w3 || !b3) throw std::invalid_argument("null array");
    const int H = hidden;
    auto fill = [&](double* w, int rows, int cols, uint64_t layer, double scale) {
      const double a = std::sqrt(6.0 / static_cast<double>(rows + cols));
      for (int i = 0; i < rows * cols; ++i)
        w[i] = scale * (2.0 * uniform01(hash4(seed, kStreamXavier, layer, static_cast<uint64_t>(i))) - 1.0) * a;
    };
    fill(w1, H, 6, 1, 1.0);
    fill(w2, H, H, 2, 1.0);
    fill(w3, 4, H, 3, out_scale);
    std::fill(b1, b1 + H, 0.0);
    std::fill(b2, b2 + H, 0.0);
    std::fill(b3, b3 + 4, 0.0);
  });
}

int mppi_workload_ellipse_costmap(int width, int height, double x0, double y0, double res,
                                  double semi_a, double semi_b, double half_width, float* values) {
  return guard([&] {
    if (width < 2 || height < 2 || !(res > 0.0) || !values)
      throw std::invalid_argument("ellipse_costmap: bad grid");
    if (!(semi_a > 0.0 && semi_b > 0.0 && half_width > 0.0))
      throw std::invalid_argument("ellipse_costmap: bad ellipse");
    const double e0 = std::max(semi_a, semi_b), e1 = std::min(semi_a, semi_b);
    const bool swap = semi_b > semi_a;
    const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < hw; ++w) {
      pool.emplace_back([&, w] {
        for (int iy = static_cast<int>(w); iy < height; iy += static_cast<int>(hw)) {
          const double py = y0 + iy * res;
          for (int ix = 0; ix < width; ++ix) {
            const double px = x0 + ix * res;
            const double d = swap ? ellipse_distance(e0, e1, py, px) : ellipse_distance(e0, e1, px, py);
            values[static_cast<size_t>(iy) * width + ix] = static_cast<float>(std::min(d / half_width, 2.5));
          }
        }
      });
    }
    for (auto& t : pool) t.join();
  });
}

int mppi_workload_initial_states(int n, uint64_t seed, double semi_a, double semi_b, int uniform_arc,
                                 double vx_lo, double vx_hi, double noise_std, double* states_out) {
  return guard([&] {
    if (n < 1 || !states_out) throw std::invalid_argument("initial_states: bad arguments");
    // cumulative arc length of (a cos phi, b sin phi)
    const int N = 1 << 16;
    std::vector<double> cum(N + 1, 0.0);
    for (int i = 0; i < N; ++i) {
      const double p0 = 2.0 * M_PI * i / N, p1 = 2.0 * M_PI * (i + 1) / N;
      cum[i + 1] = cum[i] + std::hypot(semi_a * (std::cos(p1) - std::cos(p0)), semi_b * (std::sin(p1) - std::sin(p0)));
    }
    const double L = cum[N];
    for (int c = 0; c < n; ++c) {
      const double s = uniform_arc ? uniform01(hash4(seed, kStreamInit, static_cast<uint64_t>(c), 0))
                                   : static_cast<double>(c) / n;
      const double target = s * L;
      const size_t j = std::min<size_t>(N - 1, std::upper_bound(cum.begin(), cum.end(), target) - cum.begin() - 1);
      const double frac = (cum[j + 1] > cum[j]) ? (target - cum[j]) / (cum[j + 1] - cum[j]) : 0.0;
      const double phi = 2.0 * M_PI * (static_cast<double>(j) + frac) / N;
      double* x = states_out + static_cast<size_t>(c) * 7;
      x[0] = semi_a * std::cos(phi);
      x[1] = semi_b * std::sin(phi);
      x[2] = std::atan2(semi_b * std::cos(phi), -semi_a * std::sin(phi));  // CCW tangent
      x[3] = noise_std * normal(hash4(seed, kStreamInit, static_cast<uint64_t>(c), 1));
      x[4] = vx_lo + (vx_hi - vx_lo) * uniform01(hash4(seed, kStreamInit, static_cast<uint64_t>(c), 2));
      x[5] = noise_std * normal(hash4(seed, kStreamInit, static_cast<uint64_t>(c), 3));
      x[6] = noise_std * normal(hash4(seed, kStreamInit, static_cast<uint64_t>(c), 4));
    }
  });
}

int mppi_sg_coefficients(int window, int degree, double* coeffs_out) {
  return guard([&] {
    if (!coeffs_out) throw std::invalid_argument("null output");
    const auto c = mppi_host::sg_coefficients(window, degree);
    std::copy(c.begin(), c.end(), coeffs_out);
  });
}

}  // extern "C"
