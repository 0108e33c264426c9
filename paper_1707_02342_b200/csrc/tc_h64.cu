// tc_h64.cu — the tensor-core rollout kernel and tail for H = 64 (fp32 path;
// layer-2 weight fragments in shared memory, one m16 tile per warp).
#define TC_H 64
#include "tc_launch.cuh"
