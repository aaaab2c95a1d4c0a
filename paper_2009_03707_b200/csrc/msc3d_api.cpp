// C++ drop-in API
#include "msc3d_cuda.h"
