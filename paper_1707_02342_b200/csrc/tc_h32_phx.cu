// tc_h32_phx.cu — tensor-core rollout instantiations, H = 32, noise mode kPhilox (+ the tail kernel).
#define TC_H 32
#define TC_MODE mppi_dev::kPhilox
#define TC_TAIL
#include "tc_launch.cuh"
