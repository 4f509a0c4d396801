// common.cuh -- device helpers shared by libpi's sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace pi {

constexpr int kWarp = 32;

// 16 bytes = 8 weight elements (fp16 or bf16): the unit every weight stream moves.
struct alignas(16) Pack8 {
  uint32_t u[4];
};

// Streaming 128-bit load of weights: read-only path, do not allocate in L1
// (each weight byte is used once per token).
__device__ __forceinline__ Pack8 ld_stream(const void *p) {
  Pack8 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.u[0]), "=r"(r.u[1]), "=r"(r.u[2]), "=r"(r.u[3])
               : "l"(p));
  return r;
}

// Weight element traits: unpack 8 packed elements to fp32 (exact conversions).
template <typename T>
struct WT;

template <>
struct WT<__nv_bfloat16> {
  static __device__ __forceinline__ void unpack(const Pack8 &w, float (&f)[8]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      f[2 * k] = __uint_as_float(w.u[k] << 16);
      f[2 * k + 1] = __uint_as_float(w.u[k] & 0xffff0000u);
    }
  }
  static __device__ __forceinline__ float to_float(const void *p, int64_t i) {
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(p)[i]);
  }
};

template <>
struct WT<__half> {
  static __device__ __forceinline__ void unpack(const Pack8 &w, float (&f)[8]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      __half2 h = *reinterpret_cast<const __half2 *>(&w.u[k]);
      float2 v = __half22float2(h);
      f[2 * k] = v.x;
      f[2 * k + 1] = v.y;
    }
  }
  static __device__ __forceinline__ float to_float(const void *p, int64_t i) {
    return __half2float(reinterpret_cast<const __half *>(p)[i]);
  }
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// Tensor-core GEMV helpers for the predictor's output layer (a2).
//
// P2 is stored "fragment-major" (repacked at pi_layer_create): rows padded to a multiple of 32,
// columns to a multiple of 16, cut into 16x16 tiles; tile (R, K) is 512 contiguous bytes at
// ((R * KT) + K) * 512 (KT = ceil(r / 16)), and inside it lane L = 4 g + t owns 16 bytes holding
// exactly its A fragment of mma.m16n8k16 (row-major A):
//   A[16R+g][16K+2t], A[16R+g][16K+2t+1], A[16R+g+8][16K+2t], A[16R+g+8][16K+2t+1],
//   A[16R+g][16K+2t+8], A[16R+g][16K+2t+9], A[16R+g+8][16K+2t+8], A[16R+g+8][16K+2t+9]
// so one 128-bit load per lane fetches a whole tile, conflict-free.  A 32-row mask word is
// 32 * Kp * 2 contiguous bytes, as in a row-major layout.
//
// The fp32 hidden vector g is the B operand: each value is split into three 16-bit parts
// (hi + mid + lo, each the RN rounding of the remainder; 3 x 8 (bf16) or 3 x 11 (fp16) mantissa
// bits >= fp32's 24), so P2 . g is accumulated by the tensor core to fp32 accuracy (products of
// 16-bit values are exact in fp32).  Column n = 3 b + s of the B tile is split s of token b.
// ---------------------------------------------------------------------------
constexpr int kP2Tile = 512;   // bytes of one 16x16 16-bit tile

__device__ __forceinline__ int p2_tiled_index(int row, int col, int kt) {
  // element offset of A[row][col] in the fragment-major layout (see above)
  const int R = row >> 4, K = col >> 4, rr = row & 15, cc = col & 15;
  const int g = rr & 7, hi_row = rr >> 3, t = (cc & 7) >> 1, hi_col = cc >> 3;
  const int lane = g * 4 + t, e = (cc & 1) | (hi_row << 1) | (hi_col << 2);
  return (R * kt + K) * 256 + lane * 8 + e;
}

template <typename T>
struct Split3;
template <>
struct Split3<__nv_bfloat16> {
  static __device__ __forceinline__ void split(float v, uint16_t (&o)[3]) {
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      o[s] = __bfloat16_as_ushort(h);
      v -= __bfloat162float(h);
    }
  }
};
template <>
struct Split3<__half> {
  static __device__ __forceinline__ void split(float v, uint16_t (&o)[3]) {
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const __half h = __float2half_rn(v);
      o[s] = __half_as_ushort(h);
      v -= __half2float(h);
    }
  }
};

// D += A(16x16, row) * B(16x8, col), fp32 accumulate; a: 4 regs, b: 2 regs, d: 4 regs
template <typename T>
__device__ __forceinline__ void mma16816(float (&d)[4], const uint4 &a, const uint2 &b);
template <>
__device__ __forceinline__ void mma16816<__nv_bfloat16>(float (&d)[4], const uint4 &a, const uint2 &b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y));
}
template <>
__device__ __forceinline__ void mma16816<__half>(float (&d)[4], const uint4 &a, const uint2 &b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y));
}

// Power-of-two scale that keeps max|g| * scale within the 16-bit type's range with headroom
// (fp16 saturates at 65504); exact, undone on the fp32 result.  bf16 shares fp32's range: 1.
template <typename T>
__device__ __forceinline__ float g_scale(float maxabs) {
  if (std::is_same<T, __nv_bfloat16>::value || !(maxabs > 0.f) || !isfinite(maxabs)) return 1.f;
  int e;
  frexpf(maxabs, &e);               // maxabs in [2^(e-1), 2^e)
  return ldexpf(1.f, 14 - e);       // max |g * scale| < 2^14
}

// The B fragment (2 regs) of lane (g = lane >> 2, t = lane & 3) for K-tile K and n-tile nt:
// rows k = 16 K + {2t, 2t+1, 2t+8, 2t+9}, column n = 8 nt + g -> (token n / 3, split n % 3).
// gs: shared [B][ldg] fp32 g (zero past r), scale: per-token power-of-two scale.
template <typename T, int B>
__device__ __forceinline__ uint2 g_fragment(const float *gs, int ldg, const float *scale, int K, int nt, int lane) {
  const int n = nt * 8 + (lane >> 2), t = lane & 3;
  uint32_t r[2] = {0u, 0u};
  if (n < 3 * B) {
    const int b = n / 3, s = n % 3;
    const float *gb = gs + (size_t)b * ldg + K * 16 + 2 * t;
    const float sc = scale[b];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint16_t p0[3], p1[3];
      Split3<T>::split(gb[8 * h] * sc, p0);
      Split3<T>::split(gb[8 * h + 1] * sc, p1);
      const uint16_t a = s == 0 ? p0[0] : (s == 1 ? p0[1] : p0[2]);   // no dynamic register-array index
      const uint16_t c = s == 0 ? p1[0] : (s == 1 ? p1[1] : p1[2]);
      r[h] = (uint32_t)a | ((uint32_t)c << 16);
    }
  }
  return make_uint2(r[0], r[1]);
}

// The fp32 logits of a 16-row tile for token b from the summed accumulators c[nt][4]: column
// 3b + s of row g (regs 0,1) and row g + 8 (regs 2,3) live in lane (g, col/2); gather the three
// splits with quad shuffles and add them in split order (hi, mid, lo).
template <int B, int NT>
__device__ __forceinline__ void tile_logits(const float (&c)[NT][4], int b, float &z0, float &z1) {
  const int lane = threadIdx.x & 31;
  z0 = 0.f;
  z1 = 0.f;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const int col = 3 * b + s, nt = col >> 3, cc = col & 7;
    const int src = (lane & ~3) | (cc >> 1);
    const float v0 = __shfl_sync(0xffffffffu, (cc & 1) ? c[nt][1] : c[nt][0], src);
    const float v1 = __shfl_sync(0xffffffffu, (cc & 1) ? c[nt][3] : c[nt][2], src);
    z0 += v0;
    z1 += v1;
  }
}

// INT4 neuron rows (PI_FFN_Q4, reading R21): element k of a 32-bit code word is nibble k (byte b:
// element 2b low, 2b + 1 high); (2^23 + q) - (2^23 + 8) = q - 8 exactly
__device__ __forceinline__ void q4_unpack8(uint32_t v, float (&f)[8]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) f[e] = __int_as_float(0x4B000000 | ((v >> (4 * e)) & 15u)) - 8388616.0f;
}

// Load 8 consecutive fp32 activations (32-B aligned chunk) through the cached path.
__device__ __forceinline__ void ld_x8(const float *p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
  const float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// Transpose reduction of NV per-lane partials (NV a power of two <= 32): afterwards every
// lane l holds the warp-wide total of value (l & (NV - 1)).  NV - 1 + log2(32 / NV) shuffles
// instead of 5 NV.  Fixed order.
template <int NV>
__device__ __forceinline__ float warp_reduce_multi(float (&v)[NV]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = NV / 2; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = up ? v[i] : v[i + s];
      const float keep = up ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  float r = v[0];
#pragma unroll
  for (int o = NV; o < 32; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

template <int N>
struct Pow2Ceil {
  static constexpr int v = N <= 1 ? 1 : N <= 2 ? 2 : N <= 4 ? 4 : N <= 8 ? 8 : N <= 16 ? 16 : 32;
};

}  // namespace pi
