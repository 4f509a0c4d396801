// k_layer for bf16 weights, batch 1, relu (one instantiation unit; see fused.cuh)
#include "fused.cuh"

namespace pi {
PI_FUSED_INSTANTIATE(__nv_bfloat16, 1, false)
}  // namespace pi
