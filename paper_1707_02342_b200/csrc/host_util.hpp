// host_util.hpp — host-side helpers shared by the handle and the workload
// generators.
#pragma once

#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

namespace mppi_host {

// Thread-local message behind mppi_gpu_last_error (one instance per process:
// inline function with a function-local thread_local).
inline std::string& last_error() {
  thread_local std::string msg;
  return msg;
}

// sg_coefficients (smoothing.cpp:5-33): kernel = X (X^T X)^{-1} e0 over the
// window design matrix X[i][j] = (i - half)^j (the reference uses Eigen's LDLT
// on the normal equations; this QR restatement agrees to rounding).
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

}  // namespace mppi_host
