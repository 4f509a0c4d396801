// common.cuh -- device helpers shared by libpi's sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

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

// Load 8 consecutive fp32 activations (32-B aligned chunk) through the cached path.
__device__ __forceinline__ void ld_x8(const float *p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
  const float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

}  // namespace pi
