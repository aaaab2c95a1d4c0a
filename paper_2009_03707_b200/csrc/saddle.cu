// saddle-graph kernels (filled in below)
#include "common.cuh"
