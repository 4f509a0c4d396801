// k_layer for bf16 weights, batch 2, reglu (one instantiation unit; see fused.cuh)
#include "fused.cuh"

namespace pi {
PI_FUSED_INSTANTIATE(__nv_bfloat16, 2, true)
}  // namespace pi
