// tc_h64_phx.cu — tensor-core rollout instantiations, H = 64, noise mode kPhilox (+ the tail kernel).
#define TC_H 64
#define TC_MODE mppi_dev::kPhilox
#define TC_TAIL
#include "tc_launch.cuh"
