// Forwards to the B200 drop-in API (same declarations as the reference's msc3d/saddle_graph.hpp).
#pragma once
#include "msc3d/api.hpp"
