// Forwarding header: reference callers' #include "rbpelm/bench.hpp" resolves to the B200 drop-in
// surface, which declares trial protocol, sweeps and report formats (reference bench.hpp).
#pragma once
#include "../rbpelm_b200.hpp"
