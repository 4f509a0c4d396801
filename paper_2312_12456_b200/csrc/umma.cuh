// umma.cuh -- thin PTX wrappers for the 5th-generation tensor cores (tcgen05) on sm_100a:
// TMEM allocation, shared-memory matrix descriptors (no-swizzle canonical layouts),
// instruction descriptors for kind::f16 (bf16/fp16 in, fp32 accumulate), the MMA itself, its
// mbarrier commit, and TMEM -> register loads for the epilogue.
//
// Canonical no-swizzle ("interleave") layouts, in 16-byte units (CUTLASS cute/atom/mma_traits_sm100.hpp):
//   K-major  : ((8, n), 2) : ((1, SBO), LBO)   -- a core matrix is 8 rows x 16 bytes of K,
//              contiguous (128 B); SBO = byte stride between 8-row groups, LBO = byte stride
//              between the two 16-byte K chunks one MMA (K = 16 elements) reads.
//   MN-major : ((1, n), (8, k)) : ((-, SBO), (1, LBO)) -- a core matrix is 8 K-rows x 16 bytes of
//              M/N (8 elements), contiguous; SBO = stride between 16-byte M chunks, LBO = stride
//              between 8-row K groups.
#pragma once

#include <stdint.h>

namespace pi {

__device__ __forceinline__ uint32_t u_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// --- TMEM allocation (one full warp executes these) ---
template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem) {
  static_assert(kCols >= 32 && kCols <= 512 && (kCols & (kCols - 1)) == 0, "TMEM columns: power of 2 in [32, 512]");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(u_smem(dst_smem)), "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// --- descriptors ---
// Shared-memory matrix descriptor, SWIZZLE_NONE, sm_100 version 1.
__device__ __forceinline__ uint64_t umma_desc(const void *smem_ptr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  const uint32_t a = u_smem(smem_ptr);
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version (Blackwell)
  // base_offset 0, lbo_mode 0, layout type SWIZZLE_NONE (0)
  return d;
}

// Instruction descriptor for kind::f16: A, B 16-bit (bf16 if kBF16 else fp16), D fp32, M x N,
// A / B major-ness (0 = K-major, 1 = MN-major).
template <bool kBF16>
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                                   // D format: F32
         | ((kBF16 ? 1u : 0u) << 7)                  // A format
         | ((kBF16 ? 1u : 0u) << 10)                 // B format
         | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]; issued by ONE thread.
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         bool accumulate) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"((uint32_t)accumulate)
      : "memory");
}

// Arrive on an mbarrier once every MMA issued so far by this thread has completed (implies
// tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void umma_commit(uint64_t *mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(u_smem(mbar))
               : "memory");
}

// --- TMEM -> registers: warp w (quarter q = w % 4) reads TMEM lanes 32q..32q+31, one lane per
// thread, 8 consecutive 32-bit columns starting at `col`.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr_lane_col, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr_lane_col));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// Generic-proxy shared-memory writes (cp.async / st.shared) must be made visible to the tensor
// core's async proxy before an MMA reads them.
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace pi
