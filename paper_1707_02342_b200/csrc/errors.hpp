// errors.hpp — status-code error plumbing for the C ABI.  No exception ever
// crosses extern "C"; guard() converts to MPPI_* codes + last_error().
#pragma once

#include <cuda_runtime_api.h>

#include <stdexcept>
#include <string>

#include "../../include/mppi_gpu.h"
#include "host_util.hpp"

namespace mppi_host {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void throw_invalid(const std::string& m) { throw Error(MPPI_ERR_INVALID_ARGUMENT, m); }

template <class F>
int guard(F&& f) {
  try {
    f();
    return MPPI_OK;
  } catch (const Error& e) {
    last_error() = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    last_error() = e.what();
    return MPPI_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return MPPI_ERR_RUNTIME;
  }
}

}  // namespace mppi_host

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e__ = (expr);                                                              \
    if (e__ != cudaSuccess)                                                                \
      throw ::mppi_host::Error(MPPI_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)
