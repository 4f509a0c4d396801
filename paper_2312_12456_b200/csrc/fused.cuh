// fused.cuh -- single-launch persistent layer kernel (placeholder: disabled).
#pragma once
#include "common.cuh"

namespace pi {
struct FusedWork {
  bool enabled = false;
};
struct FusedArgs {
  const void *w_up, *w_down, *b_up, *b_down, *p_w1, *p_b1, *p_w2, *p_b2;
  const float *x;
  float *y;
  int d, m, r, words, B;
  float threshold;
  bool rmsnorm, pred_relu, reglu;
  uint32_t *mask_out;
  int32_t *ids_out, *n_out;
};
template <class Alloc>
inline bool fused_alloc(FusedWork &, int, int, int, int, int, Alloc &&) { return true; }
inline void fused_init(FusedWork &, cudaStream_t) {}
inline bool fused_supported(const FusedWork &w) { return w.enabled; }
template <typename T>
inline cudaError_t fused_launch(FusedWork &, const FusedArgs &, int, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace pi
