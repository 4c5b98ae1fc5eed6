// Forwarding header: reference callers' #include "rbpelm/linalg.hpp" resolves to the B200 drop-in
// surface, which declares SingularMatrix, permutations, SpdFactor, pinv_svd, rank-revealing factorisation (reference linalg.hpp).
#pragma once
#include "../rbpelm_b200.hpp"
