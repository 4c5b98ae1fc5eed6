// Forwarding header: reference callers' #include "rbpelm/checks.hpp" resolves to the B200 drop-in
// surface, which declares test-scale algebra cross-checks and the property suite (reference checks.hpp).
#pragma once
#include "../rbpelm_b200.hpp"
