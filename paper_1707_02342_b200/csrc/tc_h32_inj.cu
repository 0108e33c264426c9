// tc_h32_inj.cu — tensor-core rollout instantiations, H = 32, noise mode kInjected.
#define TC_H 32
#define TC_MODE mppi_dev::kInjected

#include "tc_launch.cuh"
