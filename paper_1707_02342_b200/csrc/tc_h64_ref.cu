// tc_h64_ref.cu — tensor-core rollout instantiations, H = 64, noise mode kRefSplitmix.
#define TC_H 64
#define TC_MODE mppi_dev::kRefSplitmix

#include "tc_launch.cuh"
