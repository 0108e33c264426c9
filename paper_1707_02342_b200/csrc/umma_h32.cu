// tcgen05 / TMEM K1 launcher, H = 32 (umma_launch.cuh)
#define UMMA_H 32
#include "umma_launch.cuh"
