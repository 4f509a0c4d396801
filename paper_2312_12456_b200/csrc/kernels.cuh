// kernels.cuh -- libpi's per-call sm_100a kernels (pi_predict, pi_compact, pi_sparse_ffn).
//
// Each kernel is one step of SURVEY.md 8(a); pi_layer_forward fuses them in
// fused.cuh.  All activations are fp32; weights fp16/bf16 streamed with 128-bit
// non-allocating loads; every reduction has a fixed order (no float atomics),
// so results are bitwise reproducible run to run.
#pragma once

#include <algorithm>
#include <type_traits>

#include "launch.h"
#include "tc.cuh"

namespace pi {

// ---------------------------------------------------------------------------
// a1: g[b, j] = act_p(s_b * (P1[j] . x_b) + b1[j])
// 256 threads = 8 warps; 4 warps split the d-axis of one row; 2 rows per block.
// ---------------------------------------------------------------------------
template <typename T, int B, bool PRED_RELU>
__global__ void __launch_bounds__(256) k_predict1(const T *__restrict__ p1, const T *__restrict__ b1,
                                                   const float *__restrict__ x,
                                                   const float *__restrict__ scale, int r, int d,
                                                   float *__restrict__ g, int nb) {
  constexpr int KS = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 2 + warp / KS;
  const int part = warp % KS;
  float acc[B];
#pragma unroll
  for (int b = 0; b < B; ++b) acc[b] = 0.f;
  if (row < r) {
    const int chunks = d >> 3;
    const T *w = p1 + (int64_t)row * d;
    int c = part * 32 + lane;
#pragma unroll 4
    for (; c < chunks; c += 32 * KS) {
      const Pack8 pw = ld_stream(w + (int64_t)c * 8);
      float wf[8];
      WT<T>::unpack(pw, wf);
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (B > 8 && b >= nb) break;
        float xv[8];
        ld_x8(x + (int64_t)b * d + c * 8, xv);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[b] = fmaf(wf[k], xv[k], acc[b]);
      }
    }
  }
  __shared__ float red[8][B];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const float v = warp_sum(acc[b]);
    if (lane == 0) red[warp][b] = v;
  }
  __syncthreads();
  if (threadIdx.x < 2 * B) {
    const int rr = threadIdx.x / B, b = threadIdx.x % B;
    const int orow = blockIdx.x * 2 + rr;
    if (orow < r && b < nb) {
      float u = 0.f;
#pragma unroll
      for (int p = 0; p < KS; ++p) u += red[rr * KS + p][b];
      if (scale) u *= scale[b];
      if (b1) u += WT<T>::to_float(b1, orow);
      if (PRED_RELU) u = fmaxf(u, 0.f);
      g[(int64_t)b * r + orow] = u;
    }
  }
}

// ---------------------------------------------------------------------------
// a2: z = P2 g + b2; bit = z > t, on the tensor cores (mma.m16n8k16 over the fragment-major P2,
// g split into three 16-bit parts; common.cuh).  256 threads = 8 warps = 8 row tiles of 16 =
// 4 mask words per block; g's B fragments are built once per block in shared memory; each
// warp streams its tile row of P2 straight from HBM (one 128-bit load per lane and K tile).
// ---------------------------------------------------------------------------
template <typename T, int B>
__global__ void __launch_bounds__(256) k_predict2(const T *__restrict__ p2t, const T *__restrict__ b2,
                                                   const float *__restrict__ g, float t, int m, int r, int kt,
                                                   int words, uint32_t *__restrict__ mask,
                                                   float *__restrict__ logits, int nb) {
  constexpr int NT = (3 * B + 7) / 8;
  constexpr int NC = NT >= 7 ? 1 : (NT >= 2 ? 2 : 4);   // independent accumulator chains
  extern __shared__ __align__(16) float p2smem[];
  const int ldg = kt * 16;
  float *gs = p2smem;                                          // [B][ldg]
  uint2 *gfrag = reinterpret_cast<uint2 *>(gs + B * ldg);       // [kt][NT][32]
  float *zb = reinterpret_cast<float *>(gfrag + kt * NT * 32);  // [B][128]
  __shared__ float gscale[B];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < B * ldg; i += blockDim.x) {
    const int b = i / ldg, k = i - b * ldg;
    gs[i] = (k < r && b < nb) ? g[(int64_t)b * r + k] : 0.f;
  }
  __syncthreads();
  for (int b = warp; b < B; b += 8) {   // per-token range scale (8 warps, up to 32 tokens)
    float mx = 0.f;
    for (int k = lane; k < r; k += 32) mx = fmaxf(mx, fabsf(gs[b * ldg + k]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) gscale[b] = g_scale<T>(mx);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kt * NT * 32; e += blockDim.x)
    gfrag[e] = g_fragment<T, B>(gs, ldg, gscale, e / (NT * 32), (e / 32) % NT, e & 31);
  __syncthreads();
  const int R = blockIdx.x * 8 + warp;   // global row tile
  if (R * 16 < words * 32) {
    const uint8_t *a_base = reinterpret_cast<const uint8_t *>(p2t) + (size_t)R * kt * kP2Tile + lane * 16;
    float acc[NC][NT][4];
#pragma unroll
    for (int q = 0; q < NC; ++q)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[q][nt][v] = 0.f;
    int K = 0;
    for (; K + NC <= kt; K += NC) {
      Pack8 a[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) a[q] = ld_stream(a_base + (size_t)(K + q) * kP2Tile);
#pragma unroll
      for (int q = 0; q < NC; ++q)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          mma16816<T>(acc[q][nt], make_uint4(a[q].u[0], a[q].u[1], a[q].u[2], a[q].u[3]),
                      gfrag[((K + q) * NT + nt) * 32 + lane]);
    }
    for (; K < kt; ++K) {
      const Pack8 a = ld_stream(a_base + (size_t)K * kP2Tile);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        mma16816<T>(acc[0][nt], make_uint4(a.u[0], a.u[1], a.u[2], a.u[3]), gfrag[(K * NT + nt) * 32 + lane]);
    }
    float c[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        float s = acc[0][nt][v];
#pragma unroll
        for (int q = 1; q < NC; ++q) s += acc[q][nt][v];
        c[nt][v] = s;
      }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      float z0, z1;
      tile_logits<B, NT>(c, b, z0, z1);
      if ((lane & 3) == 0) {
        const float inv = 1.f / gscale[b];
        zb[b * 128 + warp * 16 + (lane >> 2)] = z0 * inv;
        zb[b * 128 + warp * 16 + (lane >> 2) + 8] = z1 * inv;
      }
    }
  }
  __syncthreads();
  if (warp < 4) {
    const int word = blockIdx.x * 4 + warp;
    if (word >= words) return;
    const int i = word * 32 + lane;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (b >= nb) break;
      float z = __int_as_float(0x7fc00000);          // NaN: never active
      if (i < m) z = zb[b * 128 + warp * 32 + lane] + (b2 ? WT<T>::to_float(b2, i) : 0.f);
      const uint32_t bits = __ballot_sync(0xffffffffu, z > t);
      if (lane == 0) mask[(int64_t)b * words + word] = bits;
      if (logits && i < m) logits[(int64_t)b * m + i] = z;
    }
  }
}

// ---------------------------------------------------------------------------
// a4: row-sparse up(/gate) GEMV.  One warp per active neuron (grid-stride over
// the device-side count).  ReGLU rows are interleaved [gate | up] (2d elements).
// h[b, k] = masked activation, fp32.
// ---------------------------------------------------------------------------
template <typename T, int B, bool REGLU>
__global__ void __launch_bounds__(256) k_up(const T *__restrict__ wup, const T *__restrict__ bup,
                                             const float *__restrict__ x,
                                             const float *__restrict__ scale,
                                             const int32_t *__restrict__ ids,
                                             const int32_t *__restrict__ n_active,
                                             const uint32_t *__restrict__ mask, int words, int d,
                                             float *__restrict__ h, int hstride) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int tw = (gridDim.x * blockDim.x) >> 5;
  const int n = *n_active;
  const int chunks = d >> 3;
  const int64_t rowlen = REGLU ? 2 * (int64_t)d : (int64_t)d;
  for (int k = gw; k < n; k += tw) {
    const int i = ids[k];
    const T *row = wup + (int64_t)i * rowlen;
    float au[B], ag[B];
#pragma unroll
    for (int b = 0; b < B; ++b) au[b] = ag[b] = 0.f;
#pragma unroll 8
    for (int c = lane; c < chunks; c += 32) {
      float wu[8], wg[8];
      if (REGLU) {
        WT<T>::unpack(ld_stream(row + c * 8), wg);
        WT<T>::unpack(ld_stream(row + d + c * 8), wu);
      } else {
        WT<T>::unpack(ld_stream(row + c * 8), wu);
      }
#pragma unroll
      for (int b = 0; b < B; ++b) {
        float xv[8];
        ld_x8(x + (int64_t)b * d + c * 8, xv);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          au[b] = fmaf(wu[q], xv[q], au[b]);
          if (REGLU) ag[b] = fmaf(wg[q], xv[q], ag[b]);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      au[b] = warp_sum(au[b]);
      if (REGLU) ag[b] = warp_sum(ag[b]);
    }
    if (lane < B) {
      float a = 0.f, gt = 0.f;
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (b == lane) { a = au[b]; gt = ag[b]; }
      const float s = scale ? scale[lane] : 1.f;
      a = a * s + (bup ? WT<T>::to_float(bup, i) : 0.f);
      float hv = REGLU ? fmaxf(gt * s, 0.f) * a : fmaxf(a, 0.f);
      if (mask && !((mask[(int64_t)lane * words + (i >> 5)] >> (i & 31)) & 1u)) hv = 0.f;
      h[(int64_t)lane * hstride + k] = hv;
    }
  }
}

// ---------------------------------------------------------------------------
// a4 for 6 <= B <= 8 (x-stationary): a warp owns one 256-column slice of d and keeps those
// columns of x in registers for all B tokens (8 per lane); it walks a range of compacted rows,
// 4 rows' (gate and) up loads in flight, and writes each row's per-slice dot products (transpose
// reduction, one 64-byte store) to upart[slice][k][2][B].  k_up_fin then sums the slices in
// ascending order and applies the scale, b_up, the activation and the token's bit.  Replaces the
// warp-per-row k_up for these batches, which re-read all of x (B x d x 4 bytes) for every row.
// ---------------------------------------------------------------------------
template <typename T, int B, bool REGLU>
__global__ void __launch_bounds__(256) k_up_xs(const T *__restrict__ wup, const float *__restrict__ x,
                                                const int32_t *__restrict__ ids,
                                                const int32_t *__restrict__ n_active, int d, int m,
                                                float *__restrict__ upart) {
  constexpr int NV = (REGLU ? 2 : 1) * B;      // values per row: [gate | up] x tokens
  constexpr int NP = Pow2Ceil<NV>::v;
  constexpr int RU = 4;                        // rows in flight per warp
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int KW = (d + 255) / 256;              // 256-column slices
  const int R = max(1, nw / KW);               // row ranges per slice
  const int kt = gw % KW, rp = gw / KW;
  if (rp >= R) return;
  const int n = *n_active;
  const int r0 = (int)(((int64_t)rp * n) / R), r1 = (int)(((int64_t)(rp + 1) * n) / R);
  const int col = kt * 256 + lane * 8;
  const bool valid = col < d;
  const int64_t rowlen = REGLU ? 2 * (int64_t)d : (int64_t)d;
  float xr[B][8];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    if (valid) ld_x8(x + (int64_t)b * d + col, xr[b]);
    else
#pragma unroll
      for (int e = 0; e < 8; ++e) xr[b][e] = 0.f;
  }
  for (int r = r0; r < r1; r += RU) {
    Pack8 wu[RU], wg[RU];
#pragma unroll
    for (int j = 0; j < RU; ++j) {
      const bool ok = valid && r + j < r1;
      const T *row = wup + (int64_t)(ok ? ids[r + j] : 0) * rowlen;
      if (ok) {
        wu[j] = ld_stream(row + (REGLU ? d : 0) + col);
        if (REGLU) wg[j] = ld_stream(row + col);
      } else {
        wu[j].u[0] = wu[j].u[1] = wu[j].u[2] = wu[j].u[3] = 0u;
        wg[j] = wu[j];
      }
    }
#pragma unroll
    for (int j = 0; j < RU; ++j) {
      if (r + j >= r1) break;
      float acc[NP];
#pragma unroll
      for (int v = 0; v < NP; ++v) acc[v] = 0.f;
      float fu[8], fg[8];
      WT<T>::unpack(wu[j], fu);
      if (REGLU) WT<T>::unpack(wg[j], fg);
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (REGLU) acc[b] = fmaf(fg[e], xr[b][e], acc[b]);
          acc[(REGLU ? B : 0) + b] = fmaf(fu[e], xr[b][e], acc[(REGLU ? B : 0) + b]);
        }
      const float tot = warp_reduce_multi<NP>(acc);   // lane l: total of value l & (NP - 1)
      if (lane < NV) upart[((int64_t)kt * m + r + j) * (2 * B) + (REGLU ? 0 : B) + lane] = tot;
    }
  }
}

// h[b, k] = masked act(s_b * up + b_up) from the slice partials (ascending slice order)
template <typename T, int B, bool REGLU>
__global__ void __launch_bounds__(256) k_up_fin(const float *__restrict__ upart, const T *__restrict__ bup,
                                                 const float *__restrict__ scale, const int32_t *__restrict__ ids,
                                                 const int32_t *__restrict__ n_active,
                                                 const uint32_t *__restrict__ mask, int words, int d, int m,
                                                 float *__restrict__ h, int hstride) {
  const int n = *n_active;
  const int KW = (d + 255) / 256;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n * B; t += gridDim.x * blockDim.x) {
    const int k = t / B, b = t - k * B;
    float a = 0.f, g = 0.f;
    for (int kt = 0; kt < KW; ++kt) {
      const float *pp = upart + ((int64_t)kt * m + k) * (2 * B);
      a += __ldcg(pp + B + b);
      if (REGLU) g += __ldcg(pp + b);
    }
    const int i = ids[k];
    const float s = scale ? scale[b] : 1.f;
    a = a * s + (bup ? WT<T>::to_float(bup, i) : 0.f);
    float hv = REGLU ? fmaxf(g * s, 0.f) * a : fmaxf(a, 0.f);
    if (mask && !((mask[(int64_t)b * words + (i >> 5)] >> (i & 31)) & 1u)) hv = 0.f;
    h[(int64_t)b * hstride + k] = hv;
  }
}

// ---------------------------------------------------------------------------
// a5: column-sparse down GEMV, y_b = b_down + sum_k h[b,k] Wd_T[ids[k], :].
// Block (tile, split): 8 warps own a 256-column tile; split s walks compacted
// positions [s n / S, (s+1) n / S).  Warps reduce in fixed order through shared
// memory into partial[s]; the last block of each tile (integer ticket) sums the
// S partials in order s = 0..S-1 and adds b_down.  Deterministic, no float atomics.
// ---------------------------------------------------------------------------
template <typename T, int B>
__global__ void __launch_bounds__(256) k_down(const T *__restrict__ wdt, const T *__restrict__ bdown,
                                               const float *__restrict__ h, int hstride,
                                               const int32_t *__restrict__ ids,
                                               const int32_t *__restrict__ n_active, int d, int S,
                                               int tiles, float *__restrict__ partial,
                                               unsigned *__restrict__ tickets,
                                               float *__restrict__ y) {
  extern __shared__ float red[];           // [8 warps][B][256]
  __shared__ int last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x % tiles, s = blockIdx.x / tiles;
  const int n = *n_active;
  const int k0 = (int)(((int64_t)s * n) / S), k1 = (int)(((int64_t)(s + 1) * n) / S);
  const int col = tile * 256 + lane * 8;
  const bool valid = col < d;
  float acc[B][8];
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[b][q] = 0.f;
  // The split's ids and h are staged through shared memory 256 rows at a time (one coalesced
  // round trip), so each warp's weight loads -- 8 rows in flight -- depend on nothing global.
  // Warp w still walks rows k0 + w, k0 + w + 8, ... in ascending order (same sums as before).
  int *s_id = reinterpret_cast<int *>(red);   // [256]      (aliases red until the reduction)
  float *s_h = red + 256;                     // [B][256]
  for (int base = k0; base < k1; base += 256) {
    const int nc = min(256, k1 - base);
    __syncthreads();                          // the previous chunk has been consumed
    if ((int)threadIdx.x < nc) {
      s_id[threadIdx.x] = ids[base + threadIdx.x];
#pragma unroll
      for (int b = 0; b < B; ++b) s_h[b * 256 + threadIdx.x] = h[(int64_t)b * hstride + base + threadIdx.x];
    }
    __syncthreads();
    if (valid) {
      for (int r0 = warp; r0 < nc; r0 += 64) {
        Pack8 wv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = r0 + 8 * j;
          if (r < nc) wv[j] = ld_stream(wdt + (int64_t)s_id[r] * d + col);
          else wv[j].u[0] = wv[j].u[1] = wv[j].u[2] = wv[j].u[3] = 0u;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = r0 + 8 * j;
          if (r < nc) {
            float wf[8];
            WT<T>::unpack(wv[j], wf);
#pragma unroll
            for (int b = 0; b < B; ++b) {
              const float hb = s_h[b * 256 + r];
#pragma unroll
              for (int q = 0; q < 8; ++q) acc[b][q] = fmaf(hb, wf[q], acc[b][q]);
            }
          }
        }
      }
    }
  }
  __syncthreads();                            // staging done before red is written
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int q = 0; q < 8; ++q) red[(warp * B + b) * 256 + lane * 8 + q] = acc[b][q];
  __syncthreads();
  const int c = tile * 256 + threadIdx.x;
  if (c < d) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) v += red[(w * B + b) * 256 + threadIdx.x];
      partial[((int64_t)s * B + b) * d + c] = v;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&tickets[tile], 1u) == (unsigned)(S - 1));
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (c < d) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      float v = 0.f;
      for (int ss = 0; ss < S; ++ss) v += __ldcg(partial + ((int64_t)ss * B + b) * d + c);
      if (bdown) v += WT<T>::to_float(bdown, c);
      y[(int64_t)b * d + c] = v;
    }
  }
  if (threadIdx.x == 0) tickets[tile] = 0u;   // re-arm for the next launch / graph replay
}

// ---------------------------------------------------------------------------
// INT4 neuron rows (PI_FFN_Q4; format DESIGN.md reading R21, oracle/quant.py O9).  Library
// layout: one record per neuron (and per matrix) = d/2 code bytes then d/32 fp16 scales, padded
// to 16 bytes; ReGLU up records are [gate record | up record].  w = s_g * (q - 8).
// ---------------------------------------------------------------------------

// a4 over INT4 rows: one warp per active neuron; lane walks 32-element groups (16 code bytes +
// one fp16 scale per matrix); per group the integer-code dot product is scaled once.
template <typename T, int B, bool REGLU>
__global__ void __launch_bounds__(256) k_up_q4(const uint8_t *__restrict__ wup, int64_t rec,
                                                const T *__restrict__ bup, const float *__restrict__ x,
                                                const float *__restrict__ scale,
                                                const int32_t *__restrict__ ids,
                                                const int32_t *__restrict__ n_active,
                                                const uint32_t *__restrict__ mask, int words, int d,
                                                float *__restrict__ h, int hstride) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int tw = (gridDim.x * blockDim.x) >> 5;
  const int n = *n_active;
  const int groups = d >> 5;
  for (int k = gw; k < n; k += tw) {
    const int i = ids[k];
    const uint8_t *rg = wup + (int64_t)i * (REGLU ? 2 * rec : rec);   // gate record (REGLU)
    const uint8_t *ru = REGLU ? rg + rec : rg;                          // up record
    float au[B], ag[B];
#pragma unroll
    for (int b = 0; b < B; ++b) au[b] = ag[b] = 0.f;
    for (int g = lane; g < groups; g += 32) {
      const Pack8 cu = ld_stream(ru + g * 16);
      const float su = __half2float(__ushort_as_half(__ldg(reinterpret_cast<const unsigned short *>(ru + (d >> 1)) + g)));
      Pack8 cg;
      float sg = 0.f;
      if (REGLU) {
        cg = ld_stream(rg + g * 16);
        sg = __half2float(__ushort_as_half(__ldg(reinterpret_cast<const unsigned short *>(rg + (d >> 1)) + g)));
      }
      float pu[B], pg[B];
#pragma unroll
      for (int b = 0; b < B; ++b) pu[b] = pg[b] = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float fu[8], fg[8];
        q4_unpack8(cu.u[q], fu);
        if (REGLU) q4_unpack8(cg.u[q], fg);
#pragma unroll
        for (int b = 0; b < B; ++b) {
          float xv[8];
          ld_x8(x + (int64_t)b * d + g * 32 + q * 8, xv);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            pu[b] = fmaf(fu[e], xv[e], pu[b]);
            if (REGLU) pg[b] = fmaf(fg[e], xv[e], pg[b]);
          }
        }
      }
#pragma unroll
      for (int b = 0; b < B; ++b) {
        au[b] = fmaf(su, pu[b], au[b]);
        if (REGLU) ag[b] = fmaf(sg, pg[b], ag[b]);
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      au[b] = warp_sum(au[b]);
      if (REGLU) ag[b] = warp_sum(ag[b]);
    }
    if (lane < B) {
      float a = 0.f, gt = 0.f;
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (b == lane) { a = au[b]; gt = ag[b]; }
      const float s = scale ? scale[lane] : 1.f;
      a = a * s + (bup ? WT<T>::to_float(bup, i) : 0.f);
      float hv = REGLU ? fmaxf(gt * s, 0.f) * a : fmaxf(a, 0.f);
      if (mask && !((mask[(int64_t)lane * words + (i >> 5)] >> (i & 31)) & 1u)) hv = 0.f;
      h[(int64_t)lane * hstride + k] = hv;
    }
  }
}

// a5 over INT4 down records: as k_down (256-column tiles x S neuron splits, fixed-order
// reduction, integer tickets); a lane's 8 columns are one 32-bit word of codes and one scale.
template <typename T, int B>
__global__ void __launch_bounds__(256) k_down_q4(const uint8_t *__restrict__ wdn, int64_t rec,
                                                  const T *__restrict__ bdown, const float *__restrict__ h,
                                                  int hstride, const int32_t *__restrict__ ids,
                                                  const int32_t *__restrict__ n_active, int d, int S, int tiles,
                                                  float *__restrict__ partial, unsigned *__restrict__ tickets,
                                                  float *__restrict__ y) {
  extern __shared__ float red[];           // [8 warps][B][256]
  __shared__ int last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x % tiles, s = blockIdx.x / tiles;
  const int n = *n_active;
  const int k0 = (int)(((int64_t)s * n) / S), k1 = (int)(((int64_t)(s + 1) * n) / S);
  const int col = tile * 256 + lane * 8;
  const bool valid = col < d;
  float acc[B][8];
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[b][q] = 0.f;
  if (valid) {
#pragma unroll 4
    for (int k = k0 + warp; k < k1; k += 8) {
      const uint8_t *row = wdn + (int64_t)ids[k] * rec;
      uint32_t cw;
      asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(cw) : "l"(row + (col >> 1)));
      const float sc = __half2float(__ushort_as_half(__ldg(reinterpret_cast<const unsigned short *>(row + (d >> 1)) + (col >> 5))));
      float wf[8];
      q4_unpack8(cw, wf);
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const float hb = h[(int64_t)b * hstride + k] * sc;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[b][q] = fmaf(hb, wf[q], acc[b][q]);
      }
    }
  }
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int q = 0; q < 8; ++q) red[(warp * B + b) * 256 + lane * 8 + q] = acc[b][q];
  __syncthreads();
  const int c = tile * 256 + threadIdx.x;
  if (c < d) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) v += red[(w * B + b) * 256 + threadIdx.x];
      partial[((int64_t)s * B + b) * d + c] = v;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&tickets[tile], 1u) == (unsigned)(S - 1));
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (c < d) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      float v = 0.f;
      for (int ss = 0; ss < S; ++ss) v += __ldcg(partial + ((int64_t)ss * B + b) * d + c);
      if (bdown) v += WT<T>::to_float(bdown, c);
      y[(int64_t)b * d + c] = v;
    }
  }
  if (threadIdx.x == 0) tickets[tile] = 0u;   // re-arm for the next launch / graph replay
}

// ---------------------------------------------------------------------------
// launchers of the per-step kernels for one weight type (instantiated in steps_inst_<T>.cu)
// ---------------------------------------------------------------------------
template <class F>
static cudaError_t dispatch_small(int B, F &&f) {
  switch (B) {
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    case 3: return f(std::integral_constant<int, 3>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 5: return f(std::integral_constant<int, 5>{});
    case 6: return f(std::integral_constant<int, 6>{});
    case 7: return f(std::integral_constant<int, 7>{});
    case 8: return f(std::integral_constant<int, 8>{});
  }
  return cudaErrorInvalidValue;
}
template <class F>
static cudaError_t dispatch_batch(int B, F &&f) {
  if (B > 8 && B <= 16) return f(std::integral_constant<int, 16>{});   // batched (f2): tokens padded
  if (B > 16 && B <= 32) return f(std::integral_constant<int, 32>{});
  return dispatch_small(B, f);
}

template <typename T>
cudaError_t steps_predict(const StepArgs &a, const float *x, int B, const float *scale, uint32_t *mask,
                          float *logits, cudaStream_t s) {
  return dispatch_batch(B, [&](auto bb) {
    constexpr int NB = decltype(bb)::value;
    const int g1 = (a.r + 1) / 2;
    if constexpr (NB > 8) {
      // B = 9..32: the hidden layer g = act_p(s P1 x + b1) is a real GEMM -- the batched
      // tensor-core kernel with identity row ids and no mask (tc.cuh)
      if (a.x3) {
        k_split_x<T, NB><<<a.num_sms * 4, 256, 0, s>>>(x, B, a.d, a.x3);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        constexpr int N = 3 * NB;
        const int st = 128 * kTcKB * 2 + N * 128;
        const int smem = tc_stages(st) * st + 256;
        e = cudaFuncSetAttribute(k_up_tc<T, NB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        k_up_tc<T, NB, false><<<a.num_sms, kTcThreads, smem, s>>>(
            (const uint8_t *)a.p_w1, (const T *)a.p_b1, a.x3, scale, nullptr, nullptr, nullptr, 0, a.d, B, a.g, a.r,
            nullptr, a.r, a.pred_relu);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        goto predict2;
      }
    }
    if (a.pred_relu)
      k_predict1<T, NB, true><<<g1, 256, 0, s>>>((const T *)a.p_w1, (const T *)a.p_b1, x, scale, a.r, a.d, a.g, B);
    else
      k_predict1<T, NB, false><<<g1, 256, 0, s>>>((const T *)a.p_w1, (const T *)a.p_b1, x, scale, a.r, a.d, a.g, B);
    {
      cudaError_t e0 = cudaGetLastError();
      if (e0 != cudaSuccess) return e0;
    }
  predict2:
    cudaError_t e = cudaSuccess;
    constexpr int NT = (3 * NB + 7) / 8;
    const size_t smem = (size_t)NB * a.kt * 16 * 4 + (size_t)a.kt * NT * 32 * 8 + (size_t)NB * 128 * 4;
    if (smem > 32 * 1024) {   // (the kernel's static shared memory counts against the 48 KB default too)
      e = cudaFuncSetAttribute(k_predict2<T, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    k_predict2<T, NB><<<(a.words + 3) / 4, 256, smem, s>>>((const T *)a.p_w2, (const T *)a.p_b2, a.g, a.t, a.m,
                                                           a.r, a.kt, a.words, mask, logits, B);
    return cudaGetLastError();
  });
}

// batched decode on the tensor cores (B = 9..32, row f2): x splits -> k_up_tc -> k_down_tc
template <typename T, int BMAX>
cudaError_t steps_ffn_tc(const StepArgs &a, const float *x, int B, const float *scale, const int32_t *ids,
                         const int32_t *n_active, const uint32_t *mask, float *y, cudaStream_t s) {
  constexpr int N = 3 * BMAX;
  k_split_x<T, BMAX><<<a.num_sms * 4, 256, 0, s>>>(x, B, a.d, a.x3);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int up_stage = (a.reglu ? 2 : 1) * 128 * kTcKB * 2 + N * 128, dn_stage = 128 * kTcKB * 2 + N * 128;
  const int up_smem = tc_stages(up_stage) * up_stage + 256;
  const int dn_smem = tc_stages(dn_stage) * dn_stage + 256;
  if (a.reglu) {
    e = cudaFuncSetAttribute(k_up_tc<T, BMAX, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, up_smem);
    if (e != cudaSuccess) return e;
    k_up_tc<T, BMAX, true><<<a.num_sms, kTcThreads, up_smem, s>>>((const uint8_t *)a.w_up, (const T *)a.b_up, a.x3,
                                                                  scale, ids, n_active, mask, a.words, a.d, B, a.h,
                                                                  a.m, a.h3);
  } else {
    e = cudaFuncSetAttribute(k_up_tc<T, BMAX, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, up_smem);
    if (e != cudaSuccess) return e;
    k_up_tc<T, BMAX, false><<<a.num_sms, kTcThreads, up_smem, s>>>((const uint8_t *)a.w_up, (const T *)a.b_up, a.x3,
                                                                   scale, ids, n_active, mask, a.words, a.d, B, a.h,
                                                                   a.m, a.h3);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_down_tc<T, BMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, dn_smem);
  if (e != cudaSuccess) return e;
  const int tiles = a.d / 128;
  k_down_tc<T, BMAX><<<std::min(a.num_sms, tiles * a.S_tc), kTcThreads, dn_smem, s>>>(
      (const uint8_t *)a.w_down, (const T *)a.b_down, a.h3, ids, n_active, a.d, B, a.S_tc, a.partial_tc,
      a.tickets_tc, y);
  return cudaGetLastError();
}

template <typename T>
cudaError_t steps_ffn(const StepArgs &a, const float *x, int B, const float *scale, const int32_t *ids,
                      const int32_t *n_active, const uint32_t *mask, float *y, cudaStream_t s) {
  if (B > 8 && !a.q4) {
    if (!a.x3) return cudaErrorNotSupported;
    return B <= 16 ? steps_ffn_tc<T, 16>(a, x, B, scale, ids, n_active, mask, y, s)
                   : steps_ffn_tc<T, 32>(a, x, B, scale, ids, n_active, mask, y, s);
  }
  return dispatch_small(B, [&](auto bb) {
    constexpr int NB = decltype(bb)::value;
    const int gup = std::max(1, std::min((a.m + 7) / 8, a.num_sms * 8));
    if (a.q4) {
      if (a.reglu)
        k_up_q4<T, NB, true><<<gup, 256, 0, s>>>((const uint8_t *)a.w_up, a.rec_q4, (const T *)a.b_up, x, scale, ids,
                                                 n_active, mask, a.words, a.d, a.h, a.m);
      else
        k_up_q4<T, NB, false><<<gup, 256, 0, s>>>((const uint8_t *)a.w_up, a.rec_q4, (const T *)a.b_up, x, scale,
                                                  ids, n_active, mask, a.words, a.d, a.h, a.m);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      const size_t smem = (size_t)8 * NB * 256 * 4;
      if (smem > 32 * 1024) cudaFuncSetAttribute(k_down_q4<T, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_down_q4<T, NB><<<a.tiles * a.S, 256, smem, s>>>((const uint8_t *)a.w_down, a.rec_q4, (const T *)a.b_down,
                                                         a.h, a.m, ids, n_active, a.d, a.S, a.tiles, a.partial,
                                                         a.tickets, y);
      return cudaGetLastError();
    }
    bool xs = false;
    if constexpr (NB >= 6) {   // measured (c3): B = 8 5.73 -> 5.06 ms/token; B = 4 3.49 -> 3.66 (k_up kept)
      if (a.upart) {   // x-stationary up projection + slice reduction
        xs = true;
        const int gxs = a.num_sms * 8;   // 64 warps per SM
        const int gfin = std::max(1, std::min((a.m * NB + 255) / 256, a.num_sms * 4));
        if (a.reglu) {
          k_up_xs<T, NB, true><<<gxs, 256, 0, s>>>((const T *)a.w_up, x, ids, n_active, a.d, a.m, a.upart);
          k_up_fin<T, NB, true><<<gfin, 256, 0, s>>>(a.upart, (const T *)a.b_up, scale, ids, n_active, mask,
                                                     a.words, a.d, a.m, a.h, a.m);
        } else {
          k_up_xs<T, NB, false><<<gxs, 256, 0, s>>>((const T *)a.w_up, x, ids, n_active, a.d, a.m, a.upart);
          k_up_fin<T, NB, false><<<gfin, 256, 0, s>>>(a.upart, (const T *)a.b_up, scale, ids, n_active, mask,
                                                      a.words, a.d, a.m, a.h, a.m);
        }
      }
    }
    if (!xs) {
      if (a.reglu)
        k_up<T, NB, true><<<gup, 256, 0, s>>>((const T *)a.w_up, (const T *)a.b_up, x, scale, ids, n_active, mask,
                                              a.words, a.d, a.h, a.m);
      else
        k_up<T, NB, false><<<gup, 256, 0, s>>>((const T *)a.w_up, (const T *)a.b_up, x, scale, ids, n_active, mask,
                                               a.words, a.d, a.h, a.m);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)8 * NB * 256 * 4;
    if (smem > 32 * 1024) cudaFuncSetAttribute(k_down<T, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_down<T, NB><<<a.tiles * a.S, 256, smem, s>>>((const T *)a.w_down, (const T *)a.b_down, a.h, a.m, ids,
                                                    n_active, a.d, a.S, a.tiles, a.partial, a.tickets, y);
    return cudaGetLastError();
  });
}

#define PI_STEPS_INSTANTIATE(T)                                                                              \
  template cudaError_t steps_predict<T>(const StepArgs &, const float *, int, const float *, uint32_t *, float *, \
                                        cudaStream_t);                                                        \
  template cudaError_t steps_ffn<T>(const StepArgs &, const float *, int, const float *, const int32_t *,         \
                                    const int32_t *, const uint32_t *, float *, cudaStream_t);

}  // namespace pi
