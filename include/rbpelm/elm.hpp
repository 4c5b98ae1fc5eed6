// Forwarding header: reference callers' #include "rbpelm/elm.hpp" resolves to the B200 drop-in
// surface, which declares ElmParams ... train / predict / accuracy (reference elm.hpp).
#pragma once
#include "../rbpelm_b200.hpp"
