// tcgen05 / TMEM K1 launcher, H = 64 (umma_launch.cuh)
#define UMMA_H 64
#include "umma_launch.cuh"
