// Forwarding header: reference callers' #include "rbpelm/matrix.hpp" resolves to the B200 drop-in
// surface, which declares DenseMatrix, ShapeError and the dense helpers (reference proj/include/rbpelm/matrix.hpp).
#pragma once
#include "../rbpelm_b200.hpp"
