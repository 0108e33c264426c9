// handle_f64.cu — fp64 instantiation of the controller handle (strict parity
// against the double-precision reference restatement).
#include "handle.cuh"

namespace mppi_host {
HandleBase* make_handle_f64(const mppi_gpu_config& cfg) { return new Handle<double>(cfg); }
}  // namespace mppi_host
