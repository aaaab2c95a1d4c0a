// Forwards to the B200 drop-in API (same declarations as the reference's msc3d/gradient.hpp).
#pragma once
#include "msc3d/api.hpp"
