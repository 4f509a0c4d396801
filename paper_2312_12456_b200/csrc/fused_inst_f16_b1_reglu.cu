// k_layer for f16 weights, batch 1, reglu (one instantiation unit; see fused.cuh)
#include "fused.cuh"

namespace pi {
PI_FUSED_INSTANTIATE(__half, 1, true)
}  // namespace pi
