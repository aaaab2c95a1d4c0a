// assembly kernels
#include "common.cuh"
