// launch.h -- host-side entry points into libpi's kernels, one declaration per instantiation
// unit, so the ABI layer (pi_api.cu) and the kernel units compile independently and in parallel.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace pi {

// operands of the per-step kernels (library-owned device pointers of one layer handle)
struct StepArgs {
  const void *p_w1, *p_b1, *p_w2, *p_b2, *w_up, *b_up, *w_down, *b_down;
  float *g, *h, *partial;
  float *upart;       // [ceil(d/256)][m][2][B] slice partials of k_up_xs (6 <= B <= 8), or NULL
  unsigned *tickets;
  int d, m, r, kt, words, S, tiles, num_sms;
  float t;
  bool pred_relu, reglu;
  bool q4;            // PI_FFN_Q4: w_up / w_down are INT4 neuron records of rec_q4 bytes
  int64_t rec_q4;
  // batched tensor-core path (B = 9..32, tc.cuh); x3 == NULL when the layer does not support it
  uint16_t *x3, *h3;
  float *partial_tc;
  unsigned *tickets_tc;
  int S_tc;
};

// kernels.cuh, instantiated per weight type in steps_inst_<T>.cu
template <typename T>
cudaError_t steps_predict(const StepArgs &a, const float *x, int B, const float *scale, uint32_t *mask,
                          float *logits, cudaStream_t s);
template <typename T>
cudaError_t steps_ffn(const StepArgs &a, const float *x, int B, const float *scale, const int32_t *ids,
                      const int32_t *n_active, const uint32_t *mask, float *y, cudaStream_t s);

// misc.cu
cudaError_t launch_rms_scale(const float *x, int B, int d, float *scale, cudaStream_t s);
cudaError_t launch_compact(const uint32_t *mask, int B, int words, int32_t *ids, int32_t *n_active, cudaStream_t s);
cudaError_t launch_gather_rows(const void *src, const int32_t *nid, int rows, int cols, int64_t dst_stride,
                               int dst_off, void *dst, cudaStream_t s);
cudaError_t launch_pack_q4(const void *codes, const void *scales, const int32_t *nid, int rows, int d, int64_t rec,
                           int64_t dst_stride, int64_t dst_off, void *dst, cudaStream_t s);
cudaError_t launch_tile_p2(const void *src, const int32_t *nid, int rows, int cols, void *dst, cudaStream_t s);
cudaError_t launch_transpose_gather(const void *src, const int32_t *nid, int d, int m_total, int m_local,
                                    void *dst, cudaStream_t s);

}  // namespace pi
