// per-step kernels for bf16 weights (one instantiation unit; see kernels.cuh)
#include "kernels.cuh"

namespace pi {
PI_STEPS_INSTANTIATE(__nv_bfloat16)
}  // namespace pi
