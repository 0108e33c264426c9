// tc_h64_inj.cu — tensor-core rollout instantiations, H = 64, noise mode kInjected.
#define TC_H 64
#define TC_MODE mppi_dev::kInjected

#include "tc_launch.cuh"
