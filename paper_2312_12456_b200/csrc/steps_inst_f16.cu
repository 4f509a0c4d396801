// per-step kernels for f16 weights (one instantiation unit; see kernels.cuh)
#include "kernels.cuh"

namespace pi {
PI_STEPS_INSTANTIATE(__half)
}  // namespace pi
