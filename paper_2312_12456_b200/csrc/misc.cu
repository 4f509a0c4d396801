// misc.cu -- libpi's non-templated kernels: the RMS input scale, the single-CTA compaction used
// by pi_compact and the per-step path, and the create-time repacking kernels.
#include <algorithm>

#include "launch.h"

namespace pi {

constexpr float kRmsEps = 1e-6f;  // reading R19

// ---------------------------------------------------------------------------
// per-token input scale: s_b = rsqrt(mean(x_b^2) + eps)   (PI_FLAG_INPUT_RMSNORM)
// grid = B blocks, 256 threads.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_rms_scale(const float *__restrict__ x, int d,
                                                    float *__restrict__ scale) {
  const int b = blockIdx.x;
  const float *xb = x + (int64_t)b * d;
  float s = 0.f;
  // 16-byte loads, several in flight per thread (d % 8 == 0)
#pragma unroll 4
  for (int j = threadIdx.x * 4; j < d; j += blockDim.x * 4) {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(xb + j));
    s = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, s))));
  }
  __shared__ float red[8];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    scale[b] = rsqrtf(t / (float)d + kRmsEps);
  }
}

// ---------------------------------------------------------------------------
// a3: compaction of the union mask into ascending ids (single CTA, 1024 threads).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_compact(const uint32_t *__restrict__ mask, int B, int words,
                                                   int32_t *__restrict__ ids,
                                                   int32_t *__restrict__ n_active) {
  __shared__ int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (words + blockDim.x - 1) / blockDim.x;
  const int w0 = min(words, tid * per), w1 = min(words, w0 + per);
  int cnt = 0;
  for (int w = w0; w < w1; ++w) {
    uint32_t u = 0;
    for (int b = 0; b < B; ++b) u |= mask[(int64_t)b * words + w];
    cnt += __popc(u);
  }
  // block exclusive scan of cnt
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int v = (lane < (int)(blockDim.x >> 5)) ? wsum[lane] : 0;
    int iv = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, iv, o);
      if (lane >= o) iv += t;
    }
    wsum[lane] = iv - v;                  // exclusive warp offsets
  }
  __syncthreads();
  int off = wsum[warp] + incl - cnt;
  for (int w = w0; w < w1; ++w) {
    uint32_t u = 0;
    for (int b = 0; b < B; ++b) u |= mask[(int64_t)b * words + w];
    while (u) {
      const int bit = __ffs(u) - 1;
      ids[off++] = w * 32 + bit;
      u &= u - 1;
    }
  }
  if (tid == blockDim.x - 1) *n_active = off;
}

// ---------------------------------------------------------------------------
// create-time repacking (not on the hot path)
// ---------------------------------------------------------------------------
// dst[k, dst_off + j] = src[nid[k], j] for j < cols  (rows of 16-bit elements)
__global__ void k_gather_rows(const uint16_t *__restrict__ src, const int32_t *__restrict__ nid,
                              int rows, int cols, int64_t dst_stride, int dst_off,
                              uint16_t *__restrict__ dst) {
  for (int k = blockIdx.y; k < rows; k += gridDim.y) {
    const int64_t sr = nid ? nid[k] : k;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += gridDim.x * blockDim.x)
      dst[(int64_t)k * dst_stride + dst_off + j] = src[sr * cols + j];
  }
}

// dst[k, j] = src[j, nid[k]]: transpose-gather of nn.Linear W_down [d, m_total] into [m_local, d].
__global__ void k_transpose_gather(const uint16_t *__restrict__ src, const int32_t *__restrict__ nid,
                                   int d, int m_total, int m_local, uint16_t *__restrict__ dst) {
  __shared__ uint16_t tileb[32][33];
  const int k0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  for (int jj = threadIdx.y; jj < 32; jj += blockDim.y) {
    const int j = j0 + jj, k = k0 + threadIdx.x;
    if (j < d && k < m_local) {
      const int64_t col = nid ? nid[k] : k;
      tileb[jj][threadIdx.x] = src[(int64_t)j * m_total + col];
    }
  }
  __syncthreads();
  for (int kk = threadIdx.y; kk < 32; kk += blockDim.y) {
    const int k = k0 + kk, j = j0 + threadIdx.x;
    if (k < m_local && j < d) dst[(int64_t)k * d + j] = tileb[threadIdx.x][kk];
  }
}

// Fragment-major P2 (common.cuh): dst[p2_tiled_index(k, j, kt)] = src[nid[k], j] for k < rows,
// j < cols; rows padded to a multiple of 32 and columns to kt * 16 with zeros.
__global__ void k_tile_p2(const uint16_t *__restrict__ src, const int32_t *__restrict__ nid, int rows, int cols,
                          int rows_pad, int kt, uint16_t *__restrict__ dst) {
  const int64_t n = (int64_t)rows_pad * kt * 16;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = o >> 8;
    const int within = (int)(o & 255), lane = within >> 3, e = within & 7;
    const int R = (int)(blk / kt), K = (int)(blk % kt);
    const int g = lane >> 2, t = lane & 3;
    const int row = 16 * R + g + ((e >> 1) & 1) * 8;
    const int col = 16 * K + 2 * t + (e & 1) + (e >> 2) * 8;
    uint16_t v = 0;
    if (row < rows && col < cols) v = src[(int64_t)(nid ? nid[row] : row) * cols + col];
    dst[o] = v;
  }
}

cudaError_t launch_tile_p2(const void *src, const int32_t *nid, int rows, int cols, void *dst, cudaStream_t s) {
  const int rows_pad = (rows + 31) / 32 * 32, kt = (cols + 15) / 16;
  const int64_t n = (int64_t)rows_pad * kt * 16;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_tile_p2<<<grid, 256, 0, s>>>((const uint16_t *)src, nid, rows, cols, rows_pad, kt, (uint16_t *)dst);
  return cudaGetLastError();
}

// INT4 neuron records: dst[k * dst_stride + dst_off + (0 .. rec)] = codes row nid[k] (d/2 bytes)
// followed by its d/32 fp16 scales (d/16 bytes), zero padding to rec.
__global__ void k_pack_q4(const uint8_t *__restrict__ codes, const uint8_t *__restrict__ scales,
                          const int32_t *__restrict__ nid, int rows, int d, int64_t rec, int64_t dst_stride,
                          int64_t dst_off, uint8_t *__restrict__ dst) {
  const int cb = d / 2, sb = d / 16;
  for (int k = blockIdx.y; k < rows; k += gridDim.y) {
    const int64_t sr = nid ? nid[k] : k;
    uint8_t *out = dst + (int64_t)k * dst_stride + dst_off;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < rec; j += (int64_t)gridDim.x * blockDim.x)
      out[j] = j < cb ? codes[sr * cb + j] : (j < cb + sb ? scales[sr * sb + (j - cb)] : (uint8_t)0);
  }
}

cudaError_t launch_pack_q4(const void *codes, const void *scales, const int32_t *nid, int rows, int d, int64_t rec,
                           int64_t dst_stride, int64_t dst_off, void *dst, cudaStream_t s) {
  dim3 grid((unsigned)std::min<int64_t>((rec + 255) / 256, 64), rows < 65535 ? rows : 65535);
  k_pack_q4<<<grid, 256, 0, s>>>((const uint8_t *)codes, (const uint8_t *)scales, nid, rows, d, rec, dst_stride,
                                 dst_off, (uint8_t *)dst);
  return cudaGetLastError();
}

cudaError_t launch_rms_scale(const float *x, int B, int d, float *scale, cudaStream_t s) {
  k_rms_scale<<<B, 256, 0, s>>>(x, d, scale);
  return cudaGetLastError();
}

cudaError_t launch_compact(const uint32_t *mask, int B, int words, int32_t *ids, int32_t *n_active, cudaStream_t s) {
  k_compact<<<1, 1024, 0, s>>>(mask, B, words, ids, n_active);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const void *src, const int32_t *nid, int rows, int cols, int64_t dst_stride,
                               int dst_off, void *dst, cudaStream_t s) {
  dim3 grid((cols + 255) / 256 < 64 ? (cols + 255) / 256 : 64, rows < 65535 ? rows : 65535);
  k_gather_rows<<<grid, 256, 0, s>>>((const uint16_t *)src, nid, rows, cols, dst_stride, dst_off, (uint16_t *)dst);
  return cudaGetLastError();
}

cudaError_t launch_transpose_gather(const void *src, const int32_t *nid, int d, int m_total, int m_local,
                                    void *dst, cudaStream_t s) {
  dim3 grid((m_local + 31) / 32, (d + 31) / 32), block(32, 8);
  if (grid.y > 65535) return cudaErrorInvalidConfiguration;
  k_transpose_gather<<<grid, block, 0, s>>>((const uint16_t *)src, nid, d, m_total, m_local, (uint16_t *)dst);
  return cudaGetLastError();
}

}  // namespace pi
