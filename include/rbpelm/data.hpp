// Forwarding header: reference callers' #include "rbpelm/data.hpp" resolves to the B200 drop-in
// surface, which declares Dataset, loaders, normalize, synth (reference data.hpp).
#pragma once
#include "../rbpelm_b200.hpp"
