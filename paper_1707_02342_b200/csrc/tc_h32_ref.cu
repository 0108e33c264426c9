// tc_h32_ref.cu — tensor-core rollout instantiations, H = 32, noise mode kRefSplitmix.
#define TC_H 32
#define TC_MODE mppi_dev::kRefSplitmix

#include "tc_launch.cuh"
