// handle_f32.cu — fp32 instantiation of the controller handle (production path).
#include "handle.cuh"

namespace mppi_host {
HandleBase* make_handle_f32(const mppi_gpu_config& cfg) { return new Handle<float>(cfg); }
}  // namespace mppi_host
