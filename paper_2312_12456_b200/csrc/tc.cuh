// tc.cuh -- batched decode (B = 9..32 tokens) on the 5th-generation tensor cores (SURVEY.md 8(f)
// row f2; "Batching Inference").  With B tokens the union of their active neurons
// grows (49-66% of m at B = 16-32) and the gathered-row products become real
// contractions:
//
//   up   : A_up[n x B] = W_up[ids] . X^T      (gathered weight rows x tokens)   -> k_up_tc
//   down : Y[B x d]    = H . Wd_T[ids]          (tokens x gathered down rows)   -> k_down_tc
//
// Both are tcgen05.mma kind::f16 GEMMs (bf16 or fp16 operands, fp32 accumulators in TMEM).  The
// fp32 activations (x, h) enter as the B operand split into three 16-bit parts (hi + mid + lo,
// common.cuh), so the products and sums keep fp32 accuracy: column n = 3 b + s of B is split s
// of token b, N = 3 * BMAX (48 or 96).  Every weight row is read once per step.
//
// Operand staging (no TMA tensor maps): gathered rows are scattered into the no-swizzle
// canonical layouts (umma.cuh) with 16-byte cp.async by 128 producer threads; the activation
// splits are pre-laid-out in global memory in the per-K-block canonical layout so each stage's B
// tile is one contiguous bulk copy.  Producer threads fence their generic-proxy writes
// (fence.proxy.async) before arriving on the stage's mbarrier; one thread issues the MMAs;
// tcgen05.commit frees stages and hands the accumulator to the epilogue warps.
#pragma once

#include "common.cuh"
#include "umma.cuh"

namespace pi {

constexpr int kTcKB = 64;        // K elements per stage (128 bytes of each 16-bit row)
constexpr int kTcSmemBudget = 200 * 1024;   // pipeline shared memory per CTA
constexpr int kTcMaxStages = 8;
// pipeline depth for a stage of `stage_bytes`: as many stages as the budget holds (<= 8)
__host__ __device__ constexpr int tc_stages(int stage_bytes) {
  return kTcSmemBudget / stage_bytes < kTcMaxStages ? kTcSmemBudget / stage_bytes : kTcMaxStages;
}
constexpr int kTcThreads = 160;  // warps 0-3: producers + epilogue (TMEM lanes 0-127), warp 4: MMA issue

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(u_smem(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void tc_mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(u_smem(bar)), "r"(count));
}
__device__ __forceinline__ void tc_mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(u_smem(bar)) : "memory");
}
__device__ __forceinline__ void tc_mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(u_smem(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = u_smem(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tc_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   u_smem(dst)),
               "l"(src), "r"(bytes), "r"(u_smem(bar))
               : "memory");
}

// Activation splits in the K-major canonical B layout of one K block of 64 (kTcKB) elements:
// element (n, k) of block kb at  kb * N * 128 + (k / 8) * N * 16 + n * 16 + (k % 8) * 2  bytes
// (core matrices of 8 n-rows x 16 bytes; SBO = 128, LBO = N * 16).
__device__ __forceinline__ size_t tc_b_offset(int n, int k, int N) {
  return (size_t)(k / kTcKB) * N * 128 + (size_t)((k % kTcKB) / 8) * N * 16 + (size_t)n * 16 + (size_t)(k % 8) * 2;
}

}  // namespace pi

namespace pi {

// ---------------------------------------------------------------------------
// x [nb, d] fp32 -> its three 16-bit splits in the B layout of every K block (tc_b_offset), rows
// n = 3 b + s; tokens b >= nb and rows >= 3 nb are zero.  One small launch per step.
// ---------------------------------------------------------------------------
template <typename T, int BMAX>
__global__ void k_split_x(const float *__restrict__ x, int nb, int d, uint16_t *__restrict__ x3) {
  constexpr int N = 3 * BMAX;
  const int64_t total = (int64_t)BMAX * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / d), k = (int)(i % d);
    uint16_t p[3] = {0, 0, 0};
    if (b < nb) Split3<T>::split(x[(int64_t)b * d + k], p);
#pragma unroll
    for (int s = 0; s < 3; ++s) x3[tc_b_offset(3 * b + s, k, N) / 2] = p[s];
  }
}

template <int kLag, int kStages>
struct TcArrive {   // producer-side bookkeeping: arrive on full[] once a stage's cp.async copies landed
  uint32_t it = 0, arrived = 0;
  __device__ __forceinline__ void after_issue(uint64_t *full) {
    cp_async_wait<kLag>();
    fence_proxy_async_smem();
    while ((int)arrived <= (int)it - kLag) {
      tc_mbar_arrive(&full[arrived % kStages]);
      ++arrived;
    }
    ++it;
  }
  __device__ __forceinline__ void drain(uint64_t *full) {
    cp_async_wait<0>();
    fence_proxy_async_smem();
    while (arrived < it) {
      tc_mbar_arrive(&full[arrived % kStages]);
      ++arrived;
    }
  }
};

__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// ---------------------------------------------------------------------------
// a4 for B = 9..32: per CTA a chunk of <= 128 compacted positions (TMEM lane = position).
// D_up[pos, n] (and D_gate) += W[ids[pos], k-block] . X3[n, k-block] over d / 64 K blocks; the
// epilogue sums the splits per token, applies the RMS scale, b_up, the activation and the token's
// own mask bit, writes h [nb, hstride] and the down GEMM's B operand h3 (tc_b_offset over
// positions; positions [n, 64 ceil(n / 64)) zero).
// ---------------------------------------------------------------------------
// Also the predictor's hidden layer (a1) for B = 9..32: ids = NULL (row k = position k, n = the
// row count), mask = NULL (no per-token bits), relu = the act_p choice, h3 = NULL.
template <typename T, int BMAX, bool REGLU>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_up_tc(const uint8_t *__restrict__ wup, const T *__restrict__ bup, const uint16_t *__restrict__ x3,
            const float *__restrict__ scale, const int32_t *__restrict__ ids, const int32_t *__restrict__ n_active,
            const uint32_t *__restrict__ mask, int words, int d, int nb, float *__restrict__ h, int hstride,
            uint16_t *__restrict__ h3, int n_rows = 0, bool relu = true) {
  constexpr int N = 3 * BMAX;
  constexpr int NPL = REGLU ? 2 : 1;         // plane 0: up, plane 1: gate
  constexpr int A_BYTES = 128 * kTcKB * 2;   // 16 KB per plane
  constexpr int B_BYTES = N * 128;
  constexpr int STAGE = NPL * A_BYTES + B_BYTES;
  constexpr int kTcStages = tc_stages(STAGE);
  constexpr int kLag = kTcStages - 2;   // cp.async groups kept in flight per producer thread
  extern __shared__ __align__(128) uint8_t tsm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(tsm + kTcStages * STAGE);
  uint64_t *empty = full + kTcStages;
  uint64_t *acc_full = empty + kTcStages;   // [2]
  uint64_t *acc_empty = acc_full + 2;       // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int n = ids ? *n_active : n_rows;
  const int G = gridDim.x;
  const int Tn = max(G, (n + 127) / 128);
  const int KB = d / kTcKB;
  const int64_t rowb = (int64_t)NPL * d * 2;   // bytes of one library up row (ReGLU: gate | up)
  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      tc_mbar_init(&full[s], 128 + 1);
      tc_mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc_mbar_init(&acc_full[b], 1);
      tc_mbar_init(&acc_empty[b], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ---------------- MMA issuer ----------------
    if ((tid & 31) == 0) {
      constexpr uint32_t idesc = umma_idesc<std::is_same<T, __nv_bfloat16>::value>(128, N, 0, 0);
      uint32_t it = 0;
      int ci = 0;
      for (int t = blockIdx.x; t < Tn; t += G, ++ci) {
        const int ab = ci & 1;
        if (ci >= 2) tc_mbar_wait(&acc_empty[ab], ((ci >> 1) - 1) & 1);
        tc_fence_after();
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % kTcStages;
          tc_mbar_wait(&full[s], (it / kTcStages) & 1);
          tc_fence_after();
          const uint8_t *st = tsm + (size_t)s * STAGE;
#pragma unroll
          for (int kk = 0; kk < kTcKB / 16; ++kk) {
            const uint64_t bdesc = umma_desc(st + NPL * A_BYTES + kk * 2 * N * 16, N * 16, 128);
#pragma unroll
            for (int pl = 0; pl < NPL; ++pl) {
              const uint64_t adesc = umma_desc(st + pl * A_BYTES + kk * 2 * 2048, 2048, 128);
              umma_f16(tmem + ab * 256 + pl * N, adesc, bdesc, idesc, (kb | kk) != 0);
            }
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[ab]);
      }
    }
  } else {
    // ---------------- producers, then the epilogue of each chunk (thread = TMEM lane = row) ----------------
    TcArrive<kLag, kTcStages> arr;
    const int row = tid;
    int ci = 0;
    for (int t = blockIdx.x; t < Tn; t += G, ++ci) {
      const int p0 = (int)(((int64_t)t * n) / Tn), p1 = (int)(((int64_t)(t + 1) * n) / Tn), R = p1 - p0;
      const int i = row < R ? (ids ? ids[p0 + row] : p0 + row) : 0;
      const uint8_t *src = wup + (int64_t)i * rowb;
      for (int kb = 0; kb < KB; ++kb) {
        const uint32_t it = arr.it;
        const int s = it % kTcStages;
        const uint32_t use = it / kTcStages;
        if (use > 0) tc_mbar_wait(&empty[s], (use - 1) & 1);
        uint8_t *st = tsm + (size_t)s * STAGE;
        if (row < R) {
#pragma unroll
          for (int pl = 0; pl < NPL; ++pl) {
            const uint8_t *sp = src + (REGLU ? (pl == 0 ? (int64_t)d * 2 : 0) : 0) + (int64_t)kb * kTcKB * 2;
#pragma unroll
            for (int kc = 0; kc < 8; ++kc)
              cp_async16(st + pl * A_BYTES + kc * 2048 + (row >> 3) * 128 + (row & 7) * 16, sp + kc * 16);
          }
        }
        cp_async_commit();
        if (tid == 0) {
          tc_mbar_expect_tx(&full[s], B_BYTES);
          tc_bulk_g2s(st + NPL * A_BYTES, reinterpret_cast<const uint8_t *>(x3) + (size_t)kb * B_BYTES, B_BYTES,
                      &full[s]);
        }
        arr.after_issue(full);
      }
      arr.drain(full);
      // epilogue
      const int ab = ci & 1;
      tc_mbar_wait(&acc_full[ab], (ci >> 1) & 1);
      tc_fence_after();
      const uint32_t tq = tmem + ab * 256 + ((uint32_t)(warp * 32) << 16);
      const int pos = p0 + row;
      const float bu = (row < R && bup) ? WT<T>::to_float(bup, i) : 0.f;
#pragma unroll
      for (int g8 = 0; g8 < BMAX / 8; ++g8) {   // 8 tokens = 24 accumulator columns at a time
        float vu[24], vg[24];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          float tmp[8];
          tmem_ld8(tq + g8 * 24 + q * 8, tmp);
#pragma unroll
          for (int e = 0; e < 8; ++e) vu[q * 8 + e] = tmp[e];
          if (REGLU) {
            tmem_ld8(tq + N + g8 * 24 + q * 8, tmp);
#pragma unroll
            for (int e = 0; e < 8; ++e) vg[q * 8 + e] = tmp[e];
          }
        }
        if (row < R) {
#pragma unroll
          for (int bb = 0; bb < 8; ++bb) {
            const int b = g8 * 8 + bb;
            float hv = 0.f;
            if (b < nb) {
              const float s_b = scale ? scale[b] : 1.f;
              const float a = ((vu[3 * bb] + vu[3 * bb + 1]) + vu[3 * bb + 2]) * s_b + bu;
              hv = REGLU ? fmaxf(((vg[3 * bb] + vg[3 * bb + 1]) + vg[3 * bb + 2]) * s_b, 0.f) * a
                         : (relu ? fmaxf(a, 0.f) : a);
              if (mask && !((mask[(int64_t)b * words + (i >> 5)] >> (i & 31)) & 1u)) hv = 0.f;
              h[(int64_t)b * hstride + pos] = hv;
            }
            if (h3) {
              uint16_t p[3];
              Split3<T>::split(hv, p);
#pragma unroll
              for (int s = 0; s < 3; ++s) h3[tc_b_offset(3 * b + s, pos, N) / 2] = p[s];
            }
          }
        }
      }
      tc_fence_before();
      tc_mbar_arrive(&acc_empty[ab]);
    }
    // positions [n, 64 ceil(n / 64)) of the down GEMM's B operand are zero
    if (h3 && blockIdx.x == 0) {
      const int pend = (n + kTcKB - 1) / kTcKB * kTcKB;
      for (int e = tid; e < (pend - n) * N; e += 128) h3[tc_b_offset(e % N, n + e / N, N) / 2] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------
// a5 for B = 9..32: output tile of 128 columns of d (TMEM lane = column) x K split s of the
// compacted positions (whole 64-position blocks).  A = Wd_T[ids[k], tile]^T (MN-major: each
// neuron's 256 bytes scatter into 16 core-matrix columns), B = h3.  The epilogue sums the splits
// per token into partial[s][b][col]; the last split of a tile (integer ticket) adds the S
// partials in order s = 0..S-1 and b_down: deterministic, no float atomics.
// ---------------------------------------------------------------------------
template <typename T, int BMAX>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_down_tc(const uint8_t *__restrict__ wdn, const T *__restrict__ bdown, const uint16_t *__restrict__ h3,
              const int32_t *__restrict__ ids, const int32_t *__restrict__ n_active, int d, int nb, int S,
              float *__restrict__ partial, unsigned *__restrict__ tickets, float *__restrict__ y) {
  constexpr int N = 3 * BMAX;
  constexpr int A_BYTES = 128 * kTcKB * 2;   // 128 columns x 64 neurons
  constexpr int B_BYTES = N * 128;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int kTcStages = tc_stages(STAGE);
  constexpr int kLag = kTcStages - 2;
  extern __shared__ __align__(128) uint8_t tsm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(tsm + kTcStages * STAGE);
  uint64_t *empty = full + kTcStages;
  uint64_t *acc_full = empty + kTcStages;
  uint64_t *acc_empty = acc_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int n = *n_active;
  const int nkb = (n + kTcKB - 1) / kTcKB;
  const int tiles = d / 128;
  const int items = tiles * S;
  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      tc_mbar_init(&full[s], 128 + 1);
      tc_mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc_mbar_init(&acc_full[b], 1);
      tc_mbar_init(&acc_empty[b], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    if ((tid & 31) == 0) {
      constexpr uint32_t idesc = umma_idesc<std::is_same<T, __nv_bfloat16>::value>(128, N, 1, 0);
      uint32_t it = 0;
      int ci = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++ci) {
        const int s_id = item / tiles;
        const int kb0 = (int)(((int64_t)s_id * nkb) / S), kb1 = (int)(((int64_t)(s_id + 1) * nkb) / S);
        const int ab = ci & 1;
        if (ci >= 2) tc_mbar_wait(&acc_empty[ab], ((ci >> 1) - 1) & 1);
        tc_fence_after();
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % kTcStages;
          tc_mbar_wait(&full[s], (it / kTcStages) & 1);
          tc_fence_after();
          const uint8_t *st = tsm + (size_t)s * STAGE;
#pragma unroll
          for (int kk = 0; kk < kTcKB / 16; ++kk) {
            const uint64_t adesc = umma_desc(st + kk * 256, 128, 1024);   // MN-major: LBO = K-group, SBO = M-chunk
            const uint64_t bdesc = umma_desc(st + A_BYTES + kk * 2 * N * 16, N * 16, 128);
            umma_f16(tmem + ab * 128, adesc, bdesc, idesc, (kb != kb0) || kk);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[ab]);
      }
    }
  } else {
    TcArrive<kLag, kTcStages> arr;
    int ci = 0;
    const int kr = tid >> 1, half = tid & 1;   // neuron (row of the K block) and which 8 of its 16 chunks
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++ci) {
      const int tile = item % tiles, s_id = item / tiles;
      const int kb0 = (int)(((int64_t)s_id * nkb) / S), kb1 = (int)(((int64_t)(s_id + 1) * nkb) / S);
      const int c0 = tile * 128;
      for (int kb = kb0; kb < kb1; ++kb) {
        const uint32_t it = arr.it;
        const int s = it % kTcStages;
        const uint32_t use = it / kTcStages;
        if (use > 0) tc_mbar_wait(&empty[s], (use - 1) & 1);
        uint8_t *st = tsm + (size_t)s * STAGE;
        const int k = kb * kTcKB + kr;
        uint8_t *dst = st + (kr >> 3) * 128 + (kr & 7) * 16;
        if (k < n) {
          const uint8_t *src = wdn + ((int64_t)ids[k] * d + c0) * 2;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int mc = half * 8 + q;
            cp_async16(dst + mc * 1024, src + mc * 16);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) *reinterpret_cast<uint4 *>(dst + (half * 8 + q) * 1024) = make_uint4(0, 0, 0, 0);
        }
        cp_async_commit();
        if (tid == 0) {
          tc_mbar_expect_tx(&full[s], B_BYTES);
          tc_bulk_g2s(st + A_BYTES, reinterpret_cast<const uint8_t *>(h3) + (size_t)kb * B_BYTES, B_BYTES, &full[s]);
        }
        arr.after_issue(full);
      }
      arr.drain(full);
      const int ab = ci & 1;
      const int col = c0 + tid;
      if (kb1 > kb0) {
        tc_mbar_wait(&acc_full[ab], (ci >> 1) & 1);
        tc_fence_after();
      }
      const uint32_t tq = tmem + ab * 128 + ((uint32_t)(warp * 32) << 16);
#pragma unroll
      for (int g8 = 0; g8 < BMAX / 8; ++g8) {
        float v[24];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          float tmp[8];
          tmem_ld8(tq + g8 * 24 + q * 8, tmp);
#pragma unroll
          for (int e = 0; e < 8; ++e) v[q * 8 + e] = tmp[e];
        }
#pragma unroll
        for (int bb = 0; bb < 8; ++bb) {
          const int b = g8 * 8 + bb;
          if (b < nb)
            partial[((int64_t)s_id * BMAX + b) * d + col] = (kb1 > kb0) ? (v[3 * bb] + v[3 * bb + 1]) + v[3 * bb + 2] : 0.f;
        }
      }
      tc_fence_before();
      tc_mbar_arrive(&acc_empty[ab]);
      // the last split of this tile reduces the S partials in order
      __threadfence();
      epi_sync();
      if (tid == 0) s_last = (atomicAdd(&tickets[tile], 1u) == (unsigned)(S - 1));
      epi_sync();
      if (s_last) {
        __threadfence();
        for (int b = 0; b < nb; ++b) {
          float acc = 0.f;
          for (int ss = 0; ss < S; ++ss) acc += __ldcg(partial + ((int64_t)ss * BMAX + b) * d + col);
          if (bdown) acc += WT<T>::to_float(bdown, col);
          y[(int64_t)b * d + col] = acc;
        }
        if (tid == 0) tickets[tile] = 0u;   // re-arm for the next launch / graph replay
      }
      epi_sync();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc<256>(tmem);
}

}  // namespace pi
