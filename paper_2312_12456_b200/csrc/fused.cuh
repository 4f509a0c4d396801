// fused.cuh -- the k_layer kernel (see fused_host.h for the design notes, parameters and the
// host-side sizing).  Included only by the fused_inst_*.cu instantiation units.
#pragma once

#include "fused_host.h"

namespace pi {

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier, bulk copy, named barriers, grid barrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t a = smem_addr(bar);
  while (true) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) break;
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
// L2 prefetch of a global range (no shared memory, fire and forget), kept with evict_last
__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src), "r"(bytes), "l"(policy)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 128-bit shared-memory load (LDS.128) from a ring stage.  A plain (non-volatile) load, so the
// compiler can batch the loads of several rows; the mbarrier wait before it carries a "memory"
// clobber, which keeps every such load after the wait.
__device__ __forceinline__ Pack8 lds128(const void *p) {
  const uint4 v = *reinterpret_cast<const uint4 *>(p);
  Pack8 r;
  r.u[0] = v.x;
  r.u[1] = v.y;
  r.u[2] = v.z;
  r.u[3] = v.w;
  return r;
}
// Branch-free guarded load: reads base + off if ok, else base (always valid), and returns zeros
// when !ok.  Keeps the per-stage loops free of branches so the loads of a whole stage issue
// back to back.
__device__ __forceinline__ Pack8 lds128z(const uint8_t *base, size_t off, bool ok) {
  Pack8 w = lds128(base + (ok ? off : 0));
#pragma unroll
  for (int k = 0; k < 4; ++k) w.u[k] = ok ? w.u[k] : 0u;
  return w;
}
__device__ __forceinline__ uint32_t lds32(const uint8_t *p) { return *reinterpret_cast<const uint32_t *>(p); }
__device__ __forceinline__ float lds_half(const uint8_t *p) {
  return __half2float(__ushort_as_half(*reinterpret_cast<const unsigned short *>(p)));
}
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}
__device__ __forceinline__ void up_sync() { asm volatile("bar.sync 2, %0;" ::"n"(kGroup) : "memory"); }
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grid barrier over the P co-resident CTAs (cooperative launch).  bar[0] is a monotonic 64-bit
// arrival counter: an arrival that returns `old` belongs to episode e = old / P + 1, and every
// CTA polls the counter until it reaches e * P -- one round trip shorter than a flag release by
// the last arrival (scripts/microbench_barrier.cu: 1.39 vs 1.87 us per barrier on an idle GPU).
// A 4-second watchdog traps instead of hanging.  dbg (tracing only): cycles to the atomic's
// return and to the release, and the release time.
__device__ __forceinline__ void grid_sync(unsigned long long *bar, int P, unsigned long long *dbg = nullptr) {
  consumers_sync();  // every consumer thread of this CTA has issued its global writes
  if (threadIdx.x == 0) {
    const long long c0 = clock64();
    unsigned long long old;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
    if (dbg) dbg[1] = clock64() - c0;
    const unsigned long long target = (old / (unsigned long long)P + 1ull) * (unsigned long long)P;
    const unsigned long long t0 = globaltimer();
    while (true) {
      unsigned long long cur;
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(bar) : "memory");
      if (cur >= target) break;
      __nanosleep(32);
      if (globaltimer() - t0 > 4000000000ull) __trap();
    }
    if (dbg) {
      dbg[2] = clock64() - c0;
      dbg[3] = globaltimer();
    }
  }
  consumers_sync();
}

// Up-group reduction of NV values (NV <= 32): per-warp transpose reduction, lanes < NV write
// red[warp][l]; after the 256-thread barrier, red holds 8 partials per value.
template <int NV>
__device__ __forceinline__ void up_partials(float (&v)[NV], float *red) {
  constexpr int NP = Pow2Ceil<NV>::v;
  float w[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) w[i] = (i < NV) ? v[i] : 0.f;
  const float r = warp_reduce_multi<NP>(w);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane < NV) red[warp * kRedStride + lane] = r;
  up_sync();
}
__device__ __forceinline__ float up_total(const float *red, int i) {
  float s = 0.f;
#pragma unroll
  for (int w = 0; w < kGroupWarps; ++w) s += red[w * kRedStride + i];
  return s;
}

// ---------------------------------------------------------------------------
// phase 2: z = P2 g + b2 ; bit = z > t ; ballot -- on the tensor cores.
// g (fp32, every CTA reads all of it) is fetched once per CTA into shared memory and turned into
// the B fragments of mma.m16n8k16: three 16-bit splits per value, power-of-two scaled (common.cuh).
// The ring stages hold this CTA's block of P2 mask words in the fragment-major tile layout; every
// 16-row tile of a stage is one warp job: KT (= r/16) mma steps over 4 independent accumulators,
// one 128-bit shared load of A and one 64-bit load of B per step.  The splits are summed per row
// (hi + mid + lo), the logits go to zbuf, and after a consumer barrier one warp per mask word
// ballots, writes the per-token words, the union word and its popcount.
// ---------------------------------------------------------------------------
struct P2Ctx {
  uint8_t *stages;
  uint64_t *full, *empty, *hready;
  volatile uint32_t *slot_pos;   // [NS] ring position the producer last acquired each slot for
  float *zbuf, *s_b2;
  int *s_count, *s_count_full;   // union counts without / with the speculative neurons (SPEC)
  const uint32_t *spec_words;    // speculative-neuron bitmap (SPEC); cleared from the union words
  uint2 *gfrag;                  // [kt][NT][32] shared B fragments
  unsigned *gmax;                // [B] shared max |g| bits (fp16 scaling), zeroed at layer start
  unsigned long long *trace;
  int NS, SB, st_p1, st_p2, w0, w1, m, r, kt, words, words_p2, zst;
  uint32_t ring0;
  float t;
  const float *g;
  uint32_t *mask, *uni;
};

template <typename T, int B, bool SPEC>
__device__ __forceinline__ void p2_phase(const P2Ctx &x) {
  constexpr int NT = (3 * B + 7) / 8;
  static_assert(NT == 1, "fused phase 2 handles B <= 2 (one n tile)");
  constexpr bool kScaled = std::is_same<T, __half>::value;   // fp16 needs the range scale (common.cuh)
  constexpr int kUL = 12 * B;    // lanes of a K tile whose column n = lane / 4 < 3 B (the rest stay zero)
  constexpr int kMaxE = 3;       // useful B fragment entries per consumer thread (fused_alloc: kt * 12 B <= 1536)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kt = x.kt, ne = kt * kUL;
  unsigned long long *dt = (x.trace && lane == 0) ? x.trace + 128 : nullptr;   // phase-2 detail (tracing)
  if (dt && warp == 0) dt[0] = globaltimer();
  // (1) B fragments straight from g in global memory (one L2 round trip): useful entry u =
  // (K tile, lane L < 12 B) needs g[b][16K + 2t + {0,1,8,9}] of token b = (L / 4) / 3
  float gv[kMaxE][4];
#pragma unroll
  for (int q = 0; q < kMaxE; ++q) {
    const int u = tid + q * kConsumers;
    const int K = u / kUL, L = u % kUL, n = L >> 2, t = L & 3;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int kk = K * 16 + 2 * t + (v & 1) + (v >> 1) * 8;
      gv[q][v] = (u < ne && kk < x.r) ? __ldcg(x.g + (size_t)(n / 3) * x.r + kk) : 0.f;
    }
  }
  float sc[B];
#pragma unroll
  for (int b = 0; b < B; ++b) sc[b] = 1.f;
  if (kScaled) {
    // per-token max |g| (split-0 entries cover every value once): shared atomicMax on the bits
#pragma unroll
    for (int q = 0; q < kMaxE; ++q) {
      const int u = tid + q * kConsumers, n = (u % kUL) >> 2;
      if (u < ne && n % 3 == 0) {
        float mx = 0.f;
#pragma unroll
        for (int v = 0; v < 4; ++v) mx = fmaxf(mx, fabsf(gv[q][v]));
        atomicMax(x.gmax + n / 3, __float_as_uint(mx));
      }
    }
    consumers_sync();
#pragma unroll
    for (int b = 0; b < B; ++b) sc[b] = g_scale<T>(__uint_as_float(x.gmax[b]));
  }
#pragma unroll
  for (int q = 0; q < kMaxE; ++q) {
    const int u = tid + q * kConsumers;
    if (u < ne) {
      const int K = u / kUL, L = u % kUL, n = L >> 2, b = n / 3, s = n % 3;
      const float s_b = (B == 1 || b == 0) ? sc[0] : sc[B - 1];
      uint32_t r2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint16_t p0[3], p1[3];
        Split3<T>::split(gv[q][2 * h] * s_b, p0);
        Split3<T>::split(gv[q][2 * h + 1] * s_b, p1);
        r2[h] = (uint32_t)p0[s] | ((uint32_t)p1[s] << 16);
      }
      x.gfrag[K * 32 + L] = make_uint2(r2[0], r2[1]);
    }
  }
  consumers_sync();
  if (dt && warp == 0) dt[2] = globaltimer();
  bool first_job = true;
  float inv[B];
#pragma unroll
  for (int b = 0; b < B; ++b) inv[b] = 1.f / sc[b];
  // (2) jobs in ring order: job q -> stage q / J, 16-row tile and K half within it (J = 4 words_p2
  // jobs per stage), round-robin over the 16 warps, so the first stages are worked on by many
  // warps at once and their slots recycle quickly (the predictor does not fit the ring: the last
  // P2 stages load into slots freed by the first).  A warp may reach a ring position whose slot
  // still holds an older stage: it first waits until the producer has acquired the slot for this
  // position (slot_pos), after which the full barrier's parity is unambiguous.
  const int wpp = x.words_p2, nwords = x.w1 - x.w0;
  const int J = 4 * wpp;                                 // jobs per full stage: 2 tiles x 2 K halves per word
  for (int job = warp; job < x.st_p2 * J; job += kConsumerWarps) {
    const int st = job / J, jj = job - st * J;
    const int wl = st * wpp + (jj >> 2);                 // CTA-local word
    if (wl >= nwords) continue;
    const int rt = (jj >> 1) & 1, half = jj & 1;         // row tile of the word, K half
    const int k0 = half * kt / 2, k1 = (half + 1) * kt / 2;
    const uint32_t it = x.st_p1 + st;
    const int slot = it % x.NS;
    while (x.slot_pos[slot] != it) __nanosleep(20);
    mbar_wait(&x.full[slot], (it / x.NS) & 1);
    if (x.trace && jj == 0 && lane == 0 && it - x.ring0 < 56) x.trace[16 + it - x.ring0] = globaltimer();
    long long c_job = 0;
    if (dt && first_job) {
      dt[16 + warp] = globaltimer();
      c_job = clock64();
    }
    float acc[2][4];   // two accumulator chains
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[q][v] = 0.f;
    const uint8_t *a_base = x.stages + (size_t)slot * x.SB + (size_t)(2 * (jj >> 2) + rt) * kt * kP2Tile + lane * 16;
    const uint2 *b_base = x.gfrag + lane;
    int K = k0;
#pragma unroll 4
    for (; K + 1 < k1; K += 2) {
      const uint4 a0 = *reinterpret_cast<const uint4 *>(a_base + (size_t)K * kP2Tile);
      const uint4 a1 = *reinterpret_cast<const uint4 *>(a_base + (size_t)(K + 1) * kP2Tile);
      mma16816<T>(acc[0], a0, b_base[K * 32]);
      mma16816<T>(acc[1], a1, b_base[(K + 1) * 32]);
    }
    if (K < k1) mma16816<T>(acc[0], *reinterpret_cast<const uint4 *>(a_base + (size_t)K * kP2Tile), b_base[K * 32]);
    if (dt && first_job) dt[32 + warp] = (unsigned long long)(clock64() - c_job) + (acc[0][0] == 1.2345e-30f ? 1 : 0);
    float c[1][4];
#pragma unroll
    for (int v = 0; v < 4; ++v) c[0][v] = acc[0][v] + acc[1][v];
    const int zrow = wl * 32 + rt * 16 + (lane >> 2);   // CTA-local row of (g)
#pragma unroll
    for (int b = 0; b < B; ++b) {
      float z0, z1;
      tile_logits<B, 1>(c, b, z0, z1);
      if ((lane & 3) == 0) {
        float *zb = x.zbuf + (half * B + b) * x.zst;     // [K half][token][row]
        zb[zrow] = z0 * inv[b];
        zb[zrow + 8] = z1 * inv[b];
      }
    }
    __syncwarp();
    if (lane == 0) {
      // every ring use gets kConsumerWarps arrivals on `empty` and one on `hready` (phase bookkeeping).
      // Jobs are dealt round-robin, so the stage's jobs_here jobs touch nw = min(16, jobs_here) warps;
      // each of them arrives once, after its last job on the stage (jj + 16 >= jobs_here), and the warp
      // holding the jobs jj = 0 mod 16 also arrives for the 16 - nw warps with no job here.
      const int jobs_here = 4 * (min(nwords, (st + 1) * wpp) - st * wpp);
      const int nw = min(kConsumerWarps, jobs_here);
      if (jj == 0) mbar_arrive_cnt(&x.hready[slot], 32);
      if (jj + kConsumerWarps >= jobs_here)
        mbar_arrive_cnt(&x.empty[slot], 1 + ((jj % kConsumerWarps == 0) ? kConsumerWarps - nw : 0));
    }
    if (dt && first_job) dt[48 + warp] = globaltimer();
    first_job = false;
  }
  consumers_sync();   // every logit of this CTA's words is in zbuf
  if (dt && warp == 0) dt[3] = globaltimer();
  // ballots: one warp per mask word -> per-token words, union word, popcount
  int my_count = 0, my_full = 0;
  for (int wl = warp; wl < x.w1 - x.w0; wl += kConsumerWarps) {
    const int rl = wl * 32 + lane;
    const bool valid = (x.w0 * 32 + rl) < x.m;
    uint32_t u = 0;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const float z = valid ? (x.zbuf[b * x.zst + rl] + x.zbuf[(B + b) * x.zst + rl]) + x.s_b2[rl]
                            : __int_as_float(0x7fc00000);
      const uint32_t bits = __ballot_sync(0xffffffffu, z > x.t);
      u |= bits;
      if (lane == 0) x.mask[(size_t)b * x.words + x.w0 + wl] = bits;
    }
    if (lane == 0) {
      const uint32_t uc = (SPEC && x.spec_words) ? (u & ~x.spec_words[x.w0 + wl]) : u;
      x.uni[x.w0 + wl] = uc;
      my_count += __popc(uc);
      if (SPEC) my_full += __popc(u);
    }
  }
  if (lane == 0 && my_count) atomicAdd(x.s_count, my_count);
  if (SPEC && lane == 0 && my_full) atomicAdd(x.s_count_full, my_full);
  if (x.trace && tid == 0) x.trace[3] = globaltimer();
}

// ---------------------------------------------------------------------------
// the kernel
//   CH : 16-byte chunks of d per group thread (chunk = t + 256 q, q < CH)
//   NA : max neurons per ring stage (also bounds P1 rows per stage: NA == 1 -> 2, else 8)
// ---------------------------------------------------------------------------
// the first argument if S, else the second (references to arrays of the same type)
template <bool S, class A, class Bb>
__device__ __forceinline__ auto &pick(A &a, Bb &b) {
  if constexpr (S) return a;
  else return b;
}

// x chunk ch (8 consecutive columns) of all B tokens from the shared-memory copy (zeros past d)
template <int B>
__device__ __forceinline__ void load_x8(const float *s_x, int d, int ch, bool ok, float (&xq)[8][B]) {
#pragma unroll
  for (int b = 0; b < B; ++b) {
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
    if (ok) {
      a0 = reinterpret_cast<const float4 *>(s_x + (size_t)b * d + ch * 8)[0];
      a1 = reinterpret_cast<const float4 *>(s_x + (size_t)b * d + ch * 8)[1];
    }
    xq[0][b] = a0.x; xq[1][b] = a0.y; xq[2][b] = a0.z; xq[3][b] = a0.w;
    xq[4][b] = a1.x; xq[5][b] = a1.y; xq[6][b] = a1.z; xq[7][b] = a1.w;
  }
}

// this CTA's partial y (register-resident, down group) -> global [B][d]
template <int B, int CH>
__device__ __forceinline__ void store_partial(const float (&yr)[CH][8][B], float *dst0, int d, int gt, int chunks) {
#pragma unroll
  for (int q = 0; q < CH; ++q) {
    const int ch = gt + q * kGroup;
    if (ch < chunks) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        float4 *dst = reinterpret_cast<float4 *>(dst0 + (size_t)b * d + ch * 8);
        __stcg(dst, make_float4(yr[q][0][b], yr[q][1][b], yr[q][2][b], yr[q][3][b]));
        __stcg(dst + 1, make_float4(yr[q][4][b], yr[q][5][b], yr[q][6][b], yr[q][7][b]));
      }
    }
  }
}

// SPEC: one down-group FFN stage: y_part += h * down row for the stage's kn neurons
template <typename T, int B, int CH, int NA>
__device__ __forceinline__ void spec_down_stage(float (&yr)[CH][8][B], const uint8_t *buf, const float *hh, int kn,
                                                size_t nb, size_t row_up, int gt, int chunks) {
#pragma unroll
  for (int g = 0; g < NA; ++g) {
    float h[B];
#pragma unroll
    for (int b = 0; b < B; ++b) h[b] = (g < kn) ? hh[g * B + b] : 0.f;
    const size_t go = (size_t)g * nb + row_up;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      const int ch = gt + q * kGroup;
      float wf[8];
      WT<T>::unpack(lds128z(buf, go + (size_t)ch * 16, g < kn && ch < chunks), wf);
#pragma unroll
      for (int b = 0; b < B; ++b)
#pragma unroll
        for (int e = 0; e < 8; ++e) yr[q][e][b] = fmaf(h[b], wf[e], yr[q][e][b]);
    }
  }
}

// SPEC variant: see k_layer below
// SPEC: the speculative hot prefix (pi_layer_desc.spec_freq) -- a separate instantiation, so the
// default kernel carries none of its code (it costs registers: measured slower).
// Q4: the FFN rows are INT4 records (PI_FFN_Q4, row f3; B = 1): a thread's 8-element chunk of d is
// one 32-bit word of codes and one fp16 scale, dequantised in registers (w = s (q - 8)).
// Grouped launch (GRP, pi_group_run): group k of the grid sees its own layers, input, output and
// slice of every workspace buffer (fused_alloc with groups > 1 lays them out with these strides).
__device__ __forceinline__ FusedParams group_view(const FusedParams &a, int k, int P) {
  FusedParams p = a;
  const size_t K = (size_t)k;
  p.lws = a.lws + K * a.L;
  p.x = a.x + K * a.B * a.d;
  p.y = a.y + K * a.B * a.d;
  p.xbuf = a.xbuf + K * kFusedMaxB * a.d;
  p.g = a.g + K * kFusedMaxB * a.r;
  p.ypart = a.ypart + K * P * kFusedMaxB * a.d;
  p.counts = a.counts + K * P;
  p.counts_full = a.counts_full + K * P;
  p.mask = a.mask + K * kFusedMaxB * a.words;
  p.uni = a.uni + K * a.words;
  p.bar = a.bar + K * (size_t)(P + 2) * 16;
  p.n_out = a.n_out ? a.n_out + K * a.L : nullptr;
  p.ids_out = nullptr;
  if (k) p.trace = nullptr;
  return p;
}

template <typename T, int B, bool REGLU, int CH, int NA, bool SPEC, bool Q4, bool GRP = false>
__global__ void __launch_bounds__(kFusedThreads, 1) k_layer(const FusedParams p0) {
  constexpr int RPM = fused_rpm(CH);          // max P1 rows per stage (fused_geometry)
  constexpr bool XS = B >= 2;                  // x staged in shared memory (fused_alloc: s_x)
  extern __shared__ __align__(128) uint8_t fsmem[];
  uint8_t *smem = fsmem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = GRP ? p0.group_ctas : (int)gridDim.x;
  const int grp = GRP ? (int)blockIdx.x / P : 0;
  const int c = GRP ? (int)blockIdx.x - grp * P : (int)blockIdx.x;
  const FusedParams p = GRP ? group_view(p0, grp, P) : p0;
  const int d = p.d, r = p.r, m = p.m, L = p.L;
  const int NS = p.NS, SB = p.stage_bytes, G = p.G, RP1 = p.rows_p1;

  // ---- shared memory carve-up ----
  uint8_t *stages = smem;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)NS * SB);
  uint64_t *empty = full + NS;
  uint64_t *hready = empty + NS;
  uint64_t *ids_ready = hready + NS;
  uint64_t *p2_done = ids_ready + 1;   // this CTA's phase 2 has finished (hot-neuron prefetch trigger)
  float *red = reinterpret_cast<float *>(ids_ready + 2);             // [2][8][32]
  float *hs = red + 2 * kGroupWarps * kRedStride;                    // [NS][NA*B]
  float *zbuf = hs + NS * NA * B;                                    // [2][B][wcap*32] logits (two K halves)
  float *s_b2 = zbuf + 2 * B * p.wcap * 32;                          // [wcap*32]
  float *s_bup = s_b2 + p.wcap * 32;                                 // [idcap]
  int *s_ids = reinterpret_cast<int *>(s_bup + p.idcap);             // [idcap]
  uint8_t *s_bits = reinterpret_cast<uint8_t *>(s_ids + p.idcap);    // [idcap]
  float *s_part = reinterpret_cast<float *>(fsmem + p.part_off);     // phase-4 partial sums (fused_spart)
  float *sg = s_part + fused_spart(P, p.pcap, B);                    // [B][kt*16] staging of g
  uint2 *gfrag = reinterpret_cast<uint2 *>(sg + B * p.kt * 16);       // [kt][NT][32] B fragments
  float *s_x = reinterpret_cast<float *>(gfrag + p.kt * ((3 * B + 7) / 8) * 32);   // [B][d] (XS)
  __shared__ unsigned s_gmax[B];
  __shared__ uint32_t s_slot_pos[kMaxStages];
  // SPEC: this CTA's share of the speculative hot prefix and its corrections
  __shared__ int32_t s_spec_ids[SPEC ? kMaxSpecPerCta : 1];
  __shared__ float s_bspec[SPEC ? kMaxSpecPerCta : 1];
  __shared__ float s_hspec[SPEC ? kMaxSpecPerCta : 1][B];
  __shared__ int32_t s_corr_ids[SPEC ? kMaxCorrPerCta : 1];
  __shared__ float s_corr_h[SPEC ? kMaxCorrPerCta : 1][B];
  __shared__ int s_ncorr, s_count_full;
  __shared__ __align__(8) uint64_t s_b2_arrive, s_b2_done;   // SPEC: split-phase grid barrier 2
  __shared__ __align__(8) uint64_t s_layer_done;   // defer_ring: the consumers finished layer l's tail
  __shared__ float s_ss[kGroupWarps][B];
  __shared__ float s_b1[kMaxP1PerCta];
  __shared__ int s_n, s_k0, s_k1, s_count;
  __shared__ const uint32_t *s_hot_words;   // this layer's hot bitmap (hot-first FFN order) or NULL
  unsigned long long *trace = p.trace ? p.trace + (size_t)c * 256 : nullptr;
  if (trace && tid == 0) trace[0] = globaltimer();

  // ---- work split (identical on producer and consumer side, every layer) ----
  const int chunks = d >> 3;
  const int n_p1 = (r > c) ? (r - 1 - c) / P + 1 : 0;  // rows j = c + P*k
  const int st_p1 = (n_p1 + RP1 - 1) / RP1;
  const int w0 = (int)(((int64_t)c * p.words) / P), w1 = (int)(((int64_t)(c + 1) * p.words) / P);
  const int st_p2 = (w1 - w0 + p.words_p2 - 1) / p.words_p2;
  // P2 stages that fit the ring at the layer start (the rest stream in as slots recycle; their
  // rows are L2-prefetched during the previous layer's tail)
  const int st_p2_ring = min(st_p2, max(0, NS - st_p1));
  // FFN rows: 16-bit (d * 2 bytes) or INT4 records (Q4: d/2 code bytes + d/32 fp16 scales, padded)
  const size_t row_ffn = Q4 ? (size_t)p.rec_q4 : (size_t)d * 2;
  const size_t row_up = row_ffn * (REGLU ? 2 : 1);         // bytes of one up (gate|up) row
  const size_t row_dn = row_ffn;
  const size_t row_p1 = (size_t)d * 2;                     // predictor rows stay 16-bit
  const size_t nb = row_up + row_dn;                       // bytes per neuron in a stage
  auto layer = [&](int l) -> LayerW { return p.lws ? p.lws[l] : p.lw0; };

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
      mbar_init(&hready[s], 32);   // one warp's lanes (the h writers) per ring use
    }
    mbar_init(ids_ready, 1);
    mbar_init(p2_done, 1);
    for (int s = 0; s < kMaxStages; ++s) s_slot_pos[s] = 0xffffffffu;
    mbar_init(&s_b2_arrive, 1);
    mbar_init(&s_b2_done, 1);
    mbar_init(&s_layer_done, 1);
  }
  for (int i = tid; i < p.kt * 32; i += blockDim.x) gfrag[i] = make_uint2(0u, 0u);
  if (tid == 0) {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // =====================================================================================
  // producer warp: streams layer after layer; runs ahead into the next layer's P1 and P2
  // rows while the consumers finish the current layer (bounded by the ring)
  // =====================================================================================
  if (warp == kConsumerWarps) {
    if constexpr (SPEC) {
      if (lane == 1) {
        // barrier agent: grid barrier 2 of layers with a speculative prefix is split -- the
        // consumers signal their arrival and compute the speculative neurons while this lane does
        // the global arrive and poll, then releases them through s_b2_done
        int ns = 0;
        for (int l = 0; l < L; ++l) {
          if (layer(l).n_spec <= 0) continue;
          mbar_wait(&s_b2_arrive, ns & 1);
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          unsigned long long old;
          asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(p.bar) : "memory");
          const unsigned long long target = (old / (unsigned long long)P + 1ull) * (unsigned long long)P;
          const unsigned long long t0 = globaltimer();
          while (true) {
            unsigned long long cur;
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(p.bar) : "memory");
            if (cur >= target) break;
            __nanosleep(32);
            if (globaltimer() - t0 > 4000000000ull) __trap();
          }
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          mbar_arrive(&s_b2_done);
          ++ns;
        }
        return;
      }
    }
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();
    uint32_t it = 0, trace_it0 = 0xffffffffu;
    auto acquire = [&](uint32_t bytes) -> uint8_t * {
      const int s = it % NS;
      const uint32_t use = it / NS;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      *reinterpret_cast<volatile uint32_t *>(&s_slot_pos[s]) = it;   // the slot now belongs to position it
      if (trace && it >= trace_it0 && it - trace_it0 < 56) trace[72 + it - trace_it0] = globaltimer();
      mbar_expect_tx(&full[s], bytes);
      return stages + (size_t)s * SB;
    };
    const size_t rowb2 = (size_t)p.kt * 16 * 2;   // bytes of one (padded) P2 row in the tiled layout
    for (int l = 0; l < L; ++l) {
      const LayerW lw = layer(l);
      // defer_ring (grouped launches): layer l's predictor rows are requested only once the
      // consumers have finished layer l-1's reduction (1) or its last grid barrier (2), so the
      // group's barrier and reduction round trips do not queue behind this SM's bulk loads
      if (p.defer_ring && l > 0) mbar_wait(&s_layer_done, (l - 1) & 1);
      if (l == (L > 1 ? 1 : 0)) trace_it0 = it;
      // The ring holds the layer's first NS predictor stages (issued while the previous layer
      // finished its FFN); stages >= NS can only be issued once the consumers free slots after
      // grid barrier 1, i.e. on the critical path.  When stage NS is next -- the previous
      // layer's FFN has been fully consumed, and HBM idles through its reduction and the
      // barriers -- pull those stages' rows into L2 so their ring loads hit L2.
      // The ring holds the layer's first NS predictor stages (issued while the previous layer
      // finishes its FFN); the predictor rows past them (P1 stages >= NS, P2 words past the ring
      // stages, which the consumers read straight from L2) are pulled into L2 once: before stage
      // NS is acquired, or after the last ring predictor stage.
      bool tail_done = false;
      auto prefetch_tail = [&](int li) {
        if (tail_done || li < NS) return;
        tail_done = true;
        const uint64_t keep = policy_evict_last();
        for (int st = NS; st < st_p1; ++st) {
          const int k0 = st * RP1, kn = min(RP1, n_p1 - k0);
          for (int k = 0; k < kn; ++k)
            prefetch_l2(lw.p_w1 + (size_t)(c + (k0 + k) * P) * row_p1, (uint32_t)row_p1, keep);
        }
        if (st_p2_ring < st_p2) {
          const size_t a0 = (size_t)(w0 + st_p2_ring * p.words_p2) * 32 * rowb2, a1 = (size_t)w1 * 32 * rowb2;
          for (size_t o = a0; o < a1; o += 32768)
            prefetch_l2(lw.p_w2 + o, (uint32_t)min((size_t)32768, a1 - o), keep);
        }
      };
      {
        // the small per-layer vectors the consumers read first (b1: every CTA, b2: my slice)
        // would cost an HBM round trip at the start of the layer: pull them into L2 now
        const uint64_t keep = policy_evict_last();
        if (lw.p_b1 && c == 0) prefetch_l2(lw.p_b1, (uint32_t)(((size_t)r * 2 + 15) & ~(size_t)15), keep);
        // the hot bitmap every CTA stages in its compaction (hot-first FFN order)
        if (lw.hot_words && lw.n_hot > 0 && c == 1 % P)
          prefetch_l2(lw.hot_words, (uint32_t)(((size_t)p.words * 4 + 15) & ~(size_t)15), keep);
        if (lw.p_b2) {
          const size_t a0 = ((size_t)w0 * 64) & ~(size_t)15;
          const size_t a1 = min((size_t)m * 2 & ~(size_t)15, ((size_t)min(m, w1 * 32) * 2 + 15) & ~(size_t)15);
          if (a1 > a0) prefetch_l2((const uint8_t *)lw.p_b2 + a0, (uint32_t)(a1 - a0), keep);
        }
      }
      for (int st = 0; st < st_p1; ++st, ++it) {  // phase 1: P1 rows c, c+P, ...
        prefetch_tail(st);
        const int k0 = st * RP1, kn = min(RP1, n_p1 - k0);
        uint8_t *dst = acquire((uint32_t)(kn * row_p1));
        const int s = it % NS;
        for (int k = 0; k < kn; ++k) {
          const int j = c + (k0 + k) * P;
          bulk_g2s(dst + (size_t)k * row_p1, lw.p_w1 + (size_t)j * row_p1, (uint32_t)row_p1, &full[s], pol);
        }
      }
      for (int st = 0; st < st_p2; ++st, ++it) {  // phase 2: P2 words [w0, w1), contiguous
        if (st == st_p2_ring) prefetch_tail(NS);
        prefetch_tail(st_p1 + st);
        const int wa = w0 + st * p.words_p2, wb = min(w1, wa + p.words_p2);
        const int ra = wa * 32, rb = wb * 32;   // whole (zero-padded) words
        const uint32_t bytes = (uint32_t)((rb - ra) * rowb2);
        uint8_t *dst = acquire(bytes);
        bulk_g2s(dst, lw.p_w2 + (size_t)ra * rowb2, bytes, &full[it % NS], pol);
      }
      prefetch_tail(NS);
      int n_spec_c = 0;
      if constexpr (SPEC) {
        // speculative hot prefix: static ids, no dependency on this layer's mask -- streamed once
        // this CTA's phase 2 is done, consumed while the grid synchronises and compacts
        n_spec_c = lw.n_spec > c ? (lw.n_spec - 1 - c) / P + 1 : 0;
        if (n_spec_c) mbar_wait(p2_done, l & 1);
        for (int k0 = 0; k0 < n_spec_c; k0 += G, ++it) {
          const int kn = min(G, n_spec_c - k0);
          uint8_t *dst = acquire((uint32_t)(kn * nb));
          const int s = it % NS;
          for (int k = 0; k < kn; ++k) {
            const int i = lw.spec_ids[c + (k0 + k) * P];
            bulk_g2s(dst + (size_t)k * nb, lw.w_up + (size_t)i * row_up, (uint32_t)row_up, &full[s], pol);
            bulk_g2s(dst + (size_t)k * nb + row_up, lw.w_down + (size_t)i * row_dn, (uint32_t)row_dn, &full[s], pol);
          }
        }
      }
      if (lw.n_hot) {
        // hot neurons (activation frequency >= hot_freq) are almost surely active: once this
        // CTA's phase 2 is done (its P2 stages are in, HBM idles through barrier 2 and the
        // compaction), pull this CTA's share of the first p.hot_cap of their up/down rows into
        // L2; the FFN stages of those neurons then load from L2
        if (!n_spec_c) mbar_wait(p2_done, l & 1);
        const uint64_t keep = policy_evict_last();
        const int nh = min(lw.n_hot, p.hot_cap);
        for (int k = c; k < nh; k += P) {
          const int i = lw.hot_ids[k];
          prefetch_l2(lw.w_up + (size_t)i * row_up, (uint32_t)row_up, keep);
          prefetch_l2(lw.w_down + (size_t)i * row_dn, (uint32_t)row_dn, keep);
        }
      }
      mbar_wait(ids_ready, l & 1);                 // phase 3: after the ids are published
      const int n_mine = s_k1 - s_k0;
      const uint8_t *wup = lw.w_up, *wdn = lw.w_down;
      for (int k0 = 0; k0 < n_mine; k0 += G, ++it) {
        const int kn = min(G, n_mine - k0);
        // the stage's ids first (the copies' "memory" clobbers would order each id read after
        // the previous copy): no shared-memory round trip between consecutive copies
        int sid[NA];
#pragma unroll
        for (int k = 0; k < NA; ++k) sid[k] = (k < kn) ? s_ids[k0 + k] : 0;
        uint8_t *dst = acquire((uint32_t)(kn * nb));
        const int s = it % NS;
#pragma unroll
        for (int k = 0; k < NA; ++k) {
          if (k < kn) {
            bulk_g2s(dst + (size_t)k * nb, wup + (size_t)sid[k] * row_up, (uint32_t)row_up, &full[s], pol);
            bulk_g2s(dst + (size_t)k * nb + row_up, wdn + (size_t)sid[k] * row_dn, (uint32_t)row_dn, &full[s], pol);
          }
        }
      }
      if constexpr (SPEC) {
        // corrections of speculative neurons whose bit is 0 for some token: their down rows again
        const int n_corr = s_ncorr;
        for (int k0 = 0; k0 < n_corr; k0 += G, ++it) {
          const int kn = min(G, n_corr - k0);
          uint8_t *dst = acquire((uint32_t)(kn * row_dn));
          const int s = it % NS;
          for (int k = 0; k < kn; ++k) {
            const int i = s_corr_ids[k0 + k];
            bulk_g2s(dst + (size_t)k * nb + row_up, lw.w_down + (size_t)i * row_dn, (uint32_t)row_dn, &full[s], pol);
          }
        }
      }
    }
    // drain: do not retire before the consumers released every stage
    for (uint32_t j = (it > (uint32_t)NS ? it - NS : 0); j < it; ++j) mbar_wait(&empty[j % NS], (j / NS) & 1);
    return;
  }

  // =====================================================================================
  // consumers
  // =====================================================================================
  const bool is_up = warp < kGroupWarps;
  const int gt = is_up ? tid : tid - kGroup;   // thread index inside its group
  const int gw = gt >> 5;                      // warp index inside its group
  auto stage_ptr = [&](uint32_t it) { return stages + (size_t)(it % NS) * SB; };
  uint32_t ring = 0;                           // ring position of this layer's first stage
  int n_spec_layers = 0;                       // SPEC: layers with a speculative prefix so far (s_b2_* parity)

  for (int l = 0; l < L; ++l) {
    const LayerW lw = layer(l);
    const float *xin = (l == 0) ? p.x : p.xbuf;
    float *yout = (l == L - 1) ? p.y : p.xbuf;
    unsigned long long *tr = (l == (L > 1 ? 1 : 0)) ? trace : nullptr;   // steady-state layer
    const uint32_t ring0 = ring;
    auto wait_full = [&](uint32_t it) {
      mbar_wait(&full[it % NS], (it / NS) & 1);
      if (tr && tid == 0 && it - ring0 < 56) tr[16 + it - ring0] = globaltimer();
    };
    if (tid == 0) {
      s_count = 0;
      s_count_full = 0;
      s_ncorr = 0;
      s_hot_words = lw.n_hot > 0 ? lw.hot_words : nullptr;
    }
    if (tid < B) s_gmax[tid] = 0u;
    if (tr && tid == 0) tr[0] = globaltimer();
    // SPEC: this CTA's share of the speculative hot prefix: neurons c, c + P, ... of the layer's list
    const bool spec_on = SPEC && lw.n_spec > 0;
    const int n_spec_c = spec_on && lw.n_spec > c ? (lw.n_spec - 1 - c) / P + 1 : 0;
    if constexpr (SPEC) {
      for (int k = tid; k < n_spec_c; k += kConsumers) {
        const int i = lw.spec_ids[c + k * P];
        s_spec_ids[k] = i;
        s_bspec[k] = lw.b_up ? WT<T>::to_float(lw.b_up, i) : 0.f;
      }
    }

    // up group: x chunks, in registers for the whole layer (B = 1), or -- B = 2, where registers
    // for x and the down group's y spill at the 96-register cap -- in shared memory (s_x [B][d]),
    // re-read per stage (each thread reads back only the chunks it wrote)
    float xr[XS ? 1 : CH][8][B];
    float sc[B];
    if (is_up) {
      float ssl[B];
#pragma unroll
      for (int b = 0; b < B; ++b) ssl[b] = 0.f;
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int ch = gt + q * kGroup;
#pragma unroll
        for (int b = 0; b < B; ++b) {
          float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
          if (ch < chunks) {
            a0 = __ldcg(reinterpret_cast<const float4 *>(xin + (size_t)b * d + ch * 8));
            a1 = __ldcg(reinterpret_cast<const float4 *>(xin + (size_t)b * d + ch * 8) + 1);
          }
          if constexpr (XS) {
            if (ch < chunks) {
              reinterpret_cast<float4 *>(s_x + (size_t)b * d + ch * 8)[0] = a0;
              reinterpret_cast<float4 *>(s_x + (size_t)b * d + ch * 8)[1] = a1;
            }
          } else {
            float(&xq)[8][B] = xr[XS ? 0 : q];
            xq[0][b] = a0.x; xq[1][b] = a0.y; xq[2][b] = a0.z; xq[3][b] = a0.w;
            xq[4][b] = a1.x; xq[5][b] = a1.y; xq[6][b] = a1.z; xq[7][b] = a1.w;
          }
          const float e8[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
          for (int k = 0; k < 8; ++k) ssl[b] = fmaf(e8[k], e8[k], ssl[b]);
        }
      }
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const float ss = warp_sum(ssl[b]);
        if (lane == 0) s_ss[gw][b] = ss;
      }
      if (gt < n_p1) s_b1[gt] = lw.p_b1 ? WT<T>::to_float(lw.p_b1, c + gt * P) : 0.f;
      up_sync();
#pragma unroll
      for (int b = 0; b < B; ++b) {
        float ss = 0.f;
#pragma unroll
        for (int w = 0; w < kGroupWarps; ++w) ss += s_ss[w][b];
        sc[b] = p.rmsnorm ? rsqrtf(ss / (float)d + 1e-6f) : 1.f;
      }
    } else {
      // down group: stage this CTA's b2 slice (off the per-stage critical path)
      for (int i = gt; i < (w1 - w0) * 32; i += kGroup) {
        const int row = w0 * 32 + i;
        s_b2[i] = (row < m && lw.p_b2) ? WT<T>::to_float(lw.p_b2, row) : 0.f;
      }
    }

    // ---------------- phase 1 (up group): g = act_p(s P1 x + b1) ----------------
    if (is_up) {
      for (int st = 0; st < st_p1; ++st) {
        const uint32_t it = ring + st;
        const int k0 = st * RP1, kn = min(RP1, n_p1 - k0);
        wait_full(it);
        const uint8_t *buf = stage_ptr(it);
        float acc[RPM * B];
#pragma unroll
        for (int i = 0; i < RPM * B; ++i) acc[i] = 0.f;
#pragma unroll
        for (int k = 0; k < RPM; ++k) {
#pragma unroll
          for (int q = 0; q < CH; ++q) {
            const int ch = gt + q * kGroup;
            float xq_s[XS ? 8 : 1][XS ? B : 1];
            if constexpr (XS) load_x8<B>(s_x, d, ch, ch < chunks, xq_s);
            auto &XQ = pick<XS>(xq_s, xr[XS ? 0 : q]);
            float wf[8];
            WT<T>::unpack(lds128z(buf, (size_t)k * row_p1 + (size_t)ch * 16, k < kn && ch < chunks), wf);
#pragma unroll
            for (int b = 0; b < B; ++b)
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[k * B + b] = fmaf(wf[e], XQ[e][b], acc[k * B + b]);
          }
        }
        float *rb = red + (st & 1) * kGroupWarps * kRedStride;
        up_partials<RPM * B>(acc, rb);
        if (gt == 0) {
          mbar_arrive_cnt(&hready[it % NS], 32);                // keep hready phases = ring uses
          mbar_arrive_cnt(&empty[it % NS], kConsumerWarps);     // every up warp has read the stage
        }
        if (gt < kn * B) {
          const int k = gt / B, b = gt % B;
          const int j = c + (k0 + k) * P;
          float u = up_total(rb, gt) * sc[b] + s_b1[k0 + k];
          if (p.pred_relu) u = fmaxf(u, 0.f);
          p.g[(size_t)b * r + j] = u;
        }
      }
    }
    if (tr && tid == 0) tr[1] = globaltimer();
    grid_sync(p.bar, P, tr ? tr + 204 : nullptr);
    if (tr && tid == 0) tr[2] = globaltimer();

    // ---------------- phase 2 (all 16 consumer warps): z = P2 g + b2, bits, union, counts ----------------
    {
      P2Ctx ctx{stages, full, empty, hready, s_slot_pos, zbuf, s_b2, &s_count, &s_count_full,
                spec_on ? lw.spec_words : nullptr, gfrag, s_gmax, tr, NS, SB, (int)ring + st_p1, st_p2, w0, w1, m,
                r, p.kt, p.words, p.words_p2, p.wcap * 32, ring, lw.t, p.g, p.mask, p.uni};
      p2_phase<T, B, SPEC>(ctx);
    }
    consumers_sync();
    if (tid == 0) {
      p.counts[c] = s_count;
      if (SPEC) p.counts_full[c] = s_count_full;
      mbar_arrive(p2_done);
    }
    // down group: the partial y lives in yr; SPEC keeps it from the speculative stages on (outer
    // scope), the default kernel declares it where the FFN starts (a longer live range costs spills)
    float yrs[SPEC ? CH : 1][8][B];
    const uint32_t it_spec = ring + st_p1 + st_p2;
    const int n_spec_st = (n_spec_c + G - 1) / G;
    if constexpr (SPEC) {
      if (spec_on) {
        auto ffn_up_stage = [&](uint32_t it, int kn, const float *bup_s, const uint8_t *bits_s, float (*hsave)[B]) {
          constexpr int NV = NA * B * (REGLU ? 2 : 1);
          wait_full(it);
          const uint8_t *buf = stage_ptr(it);
          float acc[NV];
#pragma unroll
          for (int i = 0; i < NV; ++i) acc[i] = 0.f;
#pragma unroll
          for (int g = 0; g < NA; ++g) {
            const size_t go = (size_t)g * nb;
#pragma unroll
            for (int q = 0; q < CH; ++q) {
              const int ch = gt + q * kGroup;
              float xq_s[XS ? 8 : 1][XS ? B : 1];
              if constexpr (XS) load_x8<B>(s_x, d, ch, ch < chunks, xq_s);
              auto &XQ = pick<XS>(xq_s, xr[XS ? 0 : q]);
              const bool ok = g < kn && ch < chunks;
              float wu[8];
              if (REGLU) {
                float wg[8];
                WT<T>::unpack(lds128z(buf, go + (size_t)ch * 16, ok), wg);
                WT<T>::unpack(lds128z(buf, go + (size_t)d * 2 + (size_t)ch * 16, ok), wu);
#pragma unroll
                for (int b = 0; b < B; ++b)
#pragma unroll
                  for (int e = 0; e < 8; ++e)
                    acc[(g * B + b) * 2 + 1] = fmaf(wg[e], XQ[e][b], acc[(g * B + b) * 2 + 1]);
              } else {
                WT<T>::unpack(lds128z(buf, go + (size_t)ch * 16, ok), wu);
              }
#pragma unroll
              for (int b = 0; b < B; ++b)
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  const int ai = REGLU ? (g * B + b) * 2 : g * B + b;
                  acc[ai] = fmaf(wu[e], XQ[e][b], acc[ai]);
                }
            }
          }
          float *rb = red + (it & 1) * kGroupWarps * kRedStride;
          up_partials<NV>(acc, rb);
          if (warp == 0) {
            if (lane < kn * B) {
              const int g = lane / B, b = lane % B;
              const float a = (REGLU ? up_total(rb, 2 * lane) : up_total(rb, lane)) * sc[b] + bup_s[g];
              const float hv = REGLU ? fmaxf(up_total(rb, 2 * lane + 1) * sc[b], 0.f) * a : fmaxf(a, 0.f);
              hs[(it % NS) * (NA * B) + lane] = (!bits_s || ((bits_s[g] >> b) & 1)) ? hv : 0.f;
              if (hsave) hsave[g][b] = hv;
            }
            __syncwarp();
            mbar_arrive(&hready[it % NS]);   // every writer lane releases its own h
          }
        };
        if (tid == 0) mbar_arrive(&s_b2_arrive);   // the agent lane arrives globally and polls
        if (!is_up) {
#pragma unroll
          for (int q = 0; q < CH; ++q)
#pragma unroll
            for (int e = 0; e < 8; ++e)
#pragma unroll
              for (int b = 0; b < B; ++b) yrs[q][e][b] = 0.f;
        }
        for (int f = 0; f < n_spec_st; ++f) {
          const uint32_t it = it_spec + f;
          const int kk = f * G, kn = min(G, n_spec_c - kk);
          if (is_up) {
            ffn_up_stage(it, kn, s_bspec + kk, nullptr, &s_hspec[kk]);
          } else {
            wait_full(it);
            mbar_wait(&hready[it % NS], (it / NS) & 1);
            spec_down_stage<T, B, CH, NA>(pick<SPEC>(yrs, yrs), stage_ptr(it), hs + (it % NS) * (NA * B), kn, nb,
                                          row_up, gt, chunks);
            __syncwarp();
            if (lane == 0) mbar_arrive_cnt(&empty[it % NS], 2);  // 8 down warps x 2
          }
        }
        mbar_wait(&s_b2_done, n_spec_layers & 1);
        ++n_spec_layers;
        consumers_sync();
      } else {
        grid_sync(p.bar, P, tr ? tr + 212 : nullptr);
      }
    } else {
      grid_sync(p.bar, P, tr ? tr + 212 : nullptr);
    }
    if (tr && tid == 0) tr[4] = globaltimer();

    // ---------------- phase 3: compaction of my share ----------------
    // One L2 round trip: all consumer threads stage the P counts, the union words and (B > 1)
    // the per-token words into the ring slot the first FFN stage will use -- free now: every
    // predictor stage has been consumed and the producer waits for ids_ready before reusing it.
    const uint32_t it_ffn = it_spec + n_spec_st;
    const bool stage_tok = B > 1 || spec_on;                             // per-token words staged
    uint32_t *c_uni = reinterpret_cast<uint32_t *>(stage_ptr(it_ffn));   // [words]
    uint32_t *c_msk = c_uni + p.words;                                   // [B][words] (stage_tok)
    int *c_cnt = reinterpret_cast<int *>(c_msk + (stage_tok ? B * p.words : 0));   // [P]
    int *c_cntf = c_cnt + P;                                              // [P] (SPEC)
    // hot-first FFN order: each CTA streams its share's prefetched hot neurons (L2 hits) first
    // (the bitmap pointer was staged at the layer start: reading it from the layer table here
    // would put a dependent L2 round trip on the compaction's critical path)
    const uint32_t *hot_words = s_hot_words;
    const bool hot_on = !SPEC && hot_words != nullptr;
    uint32_t *c_hot = reinterpret_cast<uint32_t *>(c_cntf + P);         // [words] (hot_on)
    {
      // every load of the staging first, then the shared stores: one L2 round trip (a store to
      // the generic ring pointer between loads would order each load after the previous store)
      constexpr int WPT = 4;                                              // words per thread
      uint32_t vu[WPT], vh[WPT], vm[WPT][B];
      int vc = 0, vcf = 0;
#pragma unroll
      for (int q = 0; q < WPT; ++q) {
        const int i = tid + q * kConsumers;
        const bool ok = i < p.words;
        vu[q] = ok ? __ldcg(p.uni + i) : 0u;
        vh[q] = (ok && hot_on) ? __ldg(hot_words + i) : 0u;
#pragma unroll
        for (int b = 0; b < B; ++b) vm[q][b] = (ok && stage_tok) ? __ldcg(p.mask + (size_t)b * p.words + i) : 0u;
      }
      if (tid < P) {
        vc = __ldcg(p.counts + tid);
        if (SPEC && spec_on) vcf = __ldcg(p.counts_full + tid);
      }
#pragma unroll
      for (int q = 0; q < WPT; ++q) {
        const int i = tid + q * kConsumers;
        if (i < p.words) {
          c_uni[i] = vu[q];
          if (hot_on) c_hot[i] = vh[q];
          if (stage_tok)
#pragma unroll
            for (int b = 0; b < B; ++b) c_msk[b * p.words + i] = vm[q][b];
        }
      }
      if (tid < P) {
        c_cnt[tid] = vc;
        if (SPEC && spec_on) c_cntf[tid] = vcf;
      }
      for (int i = tid + WPT * kConsumers; i < p.words; i += kConsumers) {   // m > 65536 only
        c_uni[i] = __ldcg(p.uni + i);
        if (hot_on) c_hot[i] = __ldg(hot_words + i);
        if (stage_tok)
          for (int b = 0; b < B; ++b) c_msk[b * p.words + i] = __ldcg(p.mask + (size_t)b * p.words + i);
      }
    }
    consumers_sync();
    if (warp == 0) {
      // CTA-block b owns words [b W/P, (b+1) W/P)
      constexpr int KPL = 8;  // counts per lane (P <= 256)
      int cv[KPL];
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const int b = lane * KPL + i;
        cv[i] = (b < P) ? c_cnt[b] : 0;
      }
      int lsum = 0;
#pragma unroll
      for (int i = 0; i < KPL; ++i) lsum += cv[i];
      int incl = lsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int n = __shfl_sync(0xffffffffu, incl, 31);
      const int k0 = (int)(((int64_t)c * n) / P), k1 = (int)(((int64_t)(c + 1) * n) / P);
      if (k0 < k1) {
        int pos = incl - lsum, cand = -1, cand_before = 0;
#pragma unroll
        for (int i = 0; i < KPL; ++i) {
          if (cand < 0 && pos + cv[i] > k0) {
            cand = lane * KPL + i;
            cand_before = pos;
          }
          pos += cv[i];
        }
        const uint32_t hit = __ballot_sync(0xffffffffu, cand >= 0);
        const int src = __ffs(hit) - 1;
        const int blk = __shfl_sync(0xffffffffu, cand, src);
        int before = __shfl_sync(0xffffffffu, cand_before, src);
        // walk union words from the start of block blk; keep ids with position in [k0, k1)
        int w = (int)(((int64_t)blk * p.words) / P);
        while (before < k1 && w < p.words) {
          const int ww = w + lane;
          const uint32_t u = (ww < p.words) ? c_uni[ww] : 0u;
          uint32_t bitsb[B];
#pragma unroll
          for (int b = 0; b < B; ++b) bitsb[b] = (B > 1 && ww < p.words) ? c_msk[b * p.words + ww] : u;
          const int cnt = __popc(u);
          int wincl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, wincl, o);
            if (lane >= o) wincl += t;
          }
          int my_pos = before + wincl - cnt;
          uint32_t v = u;
          while (v) {
            const int bit = __ffs(v) - 1;
            v &= v - 1;
            if (my_pos >= k0 && my_pos < k1) {
              const int slot = my_pos - k0;
              s_ids[slot] = ww * 32 + bit;
              uint8_t tb = 0;
#pragma unroll
              for (int b = 0; b < B; ++b) tb |= (uint8_t)(((bitsb[b] >> bit) & 1u) << b);
              s_bits[slot] = tb;
            }
            ++my_pos;
          }
          before += __shfl_sync(0xffffffffu, wincl, 31);
          w += 32;
        }
      }
      int nfull = n;
      if (SPEC && spec_on) {   // the layer's union count includes the speculative neurons
        int fs = 0;
#pragma unroll
        for (int i = 0; i < KPL; ++i) fs += (lane * KPL + i < P) ? c_cntf[lane * KPL + i] : 0;
        nfull = __reduce_add_sync(0xffffffffu, fs);
      }
      if (lane == 0) {
        s_n = nfull;
        s_k0 = k0;
        s_k1 = k1;
      }
      if (hot_on) {
        // stable partition of the share [k0, k1): hot neurons first (ascending), then the rest
        // (ascending) -- a fixed order given the mask.  ids_out keeps the ascending order.
        __syncwarp();
        const int nm = k1 - k0;
        int *tmp = reinterpret_cast<int *>(s_bup);   // free until the b_up gather below
        int nh = 0;
        for (int base = 0; base < nm; base += 32) {
          const int k = base + lane;
          bool hot = false;
          if (k < nm) {
            const int id = s_ids[k];
            tmp[k] = id | ((int)s_bits[k] << 24);
            hot = (c_hot[id >> 5] >> (id & 31)) & 1u;
            if (p.ids_out) p.ids_out[k0 + k] = id;
          }
          nh += __popc(__ballot_sync(0xffffffffu, hot));
        }
        __syncwarp();
        int ph = 0, pc = nh;
        const uint32_t lt = (1u << lane) - 1u;
        for (int base = 0; base < nm; base += 32) {
          const int k = base + lane;
          const bool ok = k < nm;
          const int v = ok ? tmp[k] : 0;
          const int id = v & 0xFFFFFF;
          const bool hot = ok && ((c_hot[id >> 5] >> (id & 31)) & 1u);
          const uint32_t bh = __ballot_sync(0xffffffffu, hot), bc = __ballot_sync(0xffffffffu, ok && !hot);
          if (ok) {
            const int dst = hot ? ph + __popc(bh & lt) : pc + __popc(bc & lt);
            s_ids[dst] = id;
            s_bits[dst] = (uint8_t)((unsigned)v >> 24);
          }
          ph += __popc(bh);
          pc += __popc(bc);
        }
      }
    } else if (SPEC && warp == 1) {
      // corrections: my speculative neurons whose bit is 0 for some token (ascending k, fixed order)
      int nc = 0;
      for (int kb = 0; kb < n_spec_c; kb += 32) {
        const int kk = kb + lane;
        bool need = false;
        uint32_t tb = 0;
        if (kk < n_spec_c) {
          const int i = s_spec_ids[kk];
#pragma unroll
          for (int b = 0; b < B; ++b) tb |= ((c_msk[b * p.words + (i >> 5)] >> (i & 31)) & 1u) << b;
          need = tb != (1u << B) - 1u;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, need);
        if (need) {
          const int slot = nc + __popc(bal & ((1u << lane) - 1u));
          s_corr_ids[slot] = s_spec_ids[kk];
#pragma unroll
          for (int b = 0; b < B; ++b) s_corr_h[slot][b] = ((tb >> b) & 1u) ? 0.f : -s_hspec[kk][b];
        }
        nc += __popc(bal);
      }
      if (lane == 0) s_ncorr = nc;
    }
    // generic-proxy writes to the scratch slot before the producer's TMA overwrites it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    consumers_sync();
    if (tid == 0) mbar_arrive(ids_ready);  // producer may stream this layer's FFN rows
    if (tr && tid == 0) tr[5] = globaltimer();
    const int k0 = s_k0, n_mine = s_k1 - s_k0;
    for (int k = tid; k < n_mine; k += kConsumers) {
      const int i = s_ids[k];
      s_bup[k] = lw.b_up ? WT<T>::to_float(lw.b_up, i) : 0.f;
      if (p.ids_out && !hot_on) p.ids_out[k0 + k] = i;
    }
    if (p.n_out && c == 0 && tid == 0) p.n_out[l] = s_n;
    consumers_sync();

    // ---------------- phase 3: the sparse FFN ----------------
    const int n_st = (n_mine + G - 1) / G;
    if (is_up) {
      constexpr int NV = NA * B * (REGLU ? 2 : 1);
      for (int f = 0; f < n_st; ++f) {
        const uint32_t it = it_ffn + f;
        const int kk = f * G, kn = min(G, n_mine - kk);
        wait_full(it);
        const uint8_t *buf = stage_ptr(it);
        float acc[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) acc[i] = 0.f;
#pragma unroll
        for (int g = 0; g < NA; ++g) {
          const size_t go = (size_t)g * nb;
          if constexpr (Q4) {
            // INT4 records: [gate record |] up record; per chunk a code word and its group scale
#pragma unroll
            for (int q = 0; q < CH; ++q) {
              const int ch = gt + q * kGroup;
              float xq_s[XS ? 8 : 1][XS ? B : 1];
              if constexpr (XS) load_x8<B>(s_x, d, ch, ch < chunks, xq_s);
              auto &XQ = pick<XS>(xq_s, xr[XS ? 0 : q]);
              const bool ok = g < kn && ch < chunks;
              const size_t cu = go + (REGLU ? row_ffn : 0);
              float fu[8], pu = 0.f;
              q4_unpack8(ok ? lds32(buf + cu + (size_t)ch * 4) : 0x88888888u, fu);
#pragma unroll
              for (int e = 0; e < 8; ++e) pu = fmaf(fu[e], XQ[e][0], pu);
              const float su = ok ? lds_half(buf + cu + (size_t)(d >> 1) + (size_t)(ch >> 2) * 2) : 0.f;
              const int ai = REGLU ? g * 2 : g;
              acc[ai] = fmaf(su, pu, acc[ai]);
              if (REGLU) {
                float fg[8], pg = 0.f;
                q4_unpack8(ok ? lds32(buf + go + (size_t)ch * 4) : 0x88888888u, fg);
#pragma unroll
                for (int e = 0; e < 8; ++e) pg = fmaf(fg[e], XQ[e][0], pg);
                const float sg = ok ? lds_half(buf + go + (size_t)(d >> 1) + (size_t)(ch >> 2) * 2) : 0.f;
                acc[g * 2 + 1] = fmaf(sg, pg, acc[g * 2 + 1]);
              }
            }
            continue;
          }
#pragma unroll
          for (int q = 0; q < CH; ++q) {
            const int ch = gt + q * kGroup;
            float xq_s[XS ? 8 : 1][XS ? B : 1];
            if constexpr (XS) load_x8<B>(s_x, d, ch, ch < chunks, xq_s);
            auto &XQ = pick<XS>(xq_s, xr[XS ? 0 : q]);
            const bool ok = g < kn && ch < chunks;
            float wu[8];
            if (REGLU) {
              float wg[8];
              WT<T>::unpack(lds128z(buf, go + (size_t)ch * 16, ok), wg);
              WT<T>::unpack(lds128z(buf, go + (size_t)d * 2 + (size_t)ch * 16, ok), wu);
#pragma unroll
              for (int b = 0; b < B; ++b)
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  acc[(g * B + b) * 2 + 1] = fmaf(wg[e], XQ[e][b], acc[(g * B + b) * 2 + 1]);
            } else {
              WT<T>::unpack(lds128z(buf, go + (size_t)ch * 16, ok), wu);
            }
#pragma unroll
            for (int b = 0; b < B; ++b)
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int ai = REGLU ? (g * B + b) * 2 : g * B + b;
                acc[ai] = fmaf(wu[e], XQ[e][b], acc[ai]);
              }
          }
        }
        float *rb = red + (f & 1) * kGroupWarps * kRedStride;
        up_partials<NV>(acc, rb);
        if (warp == 0) {
          if (lane < kn * B) {
            const int g = lane / B, b = lane % B;
            const int slot = kk + g;
            const float a = (REGLU ? up_total(rb, 2 * lane) : up_total(rb, lane)) * sc[b] + s_bup[slot];
            float hv = REGLU ? fmaxf(up_total(rb, 2 * lane + 1) * sc[b], 0.f) * a : fmaxf(a, 0.f);
            hs[(it % NS) * (NA * B) + lane] = ((s_bits[slot] >> b) & 1) ? hv : 0.f;
          }
          __syncwarp();
          mbar_arrive(&hready[it % NS]);   // every writer lane releases its own h
        }
      }
    } else {
      float yl[SPEC ? 1 : CH][8][B];
      float(&yr)[CH][8][B] = pick<SPEC>(yrs, yl);
      if (!spec_on) {
#pragma unroll
        for (int q = 0; q < CH; ++q)
#pragma unroll
          for (int e = 0; e < 8; ++e)
#pragma unroll
            for (int b = 0; b < B; ++b) yr[q][e][b] = 0.f;
      }
      for (int f = 0; f < n_st; ++f) {
        const uint32_t it = it_ffn + f;
        const int kn = min(G, n_mine - f * G);
        wait_full(it);
        mbar_wait(&hready[it % NS], (it / NS) & 1);
        const uint8_t *buf = stage_ptr(it);
        const float *hh = hs + (it % NS) * (NA * B);
#pragma unroll
        for (int g = 0; g < NA; ++g) {
          float h[B];
#pragma unroll
          for (int b = 0; b < B; ++b) h[b] = (g < kn) ? hh[g * B + b] : 0.f;
          const size_t go = (size_t)g * nb + row_up;
          if constexpr (Q4) {
#pragma unroll
            for (int q = 0; q < CH; ++q) {
              const int ch = gt + q * kGroup;
              const bool ok = g < kn && ch < chunks;
              float wf[8];
              q4_unpack8(ok ? lds32(buf + go + (size_t)ch * 4) : 0x88888888u, wf);
              const float hs_ = ok ? h[0] * lds_half(buf + go + (size_t)(d >> 1) + (size_t)(ch >> 2) * 2) : 0.f;
#pragma unroll
              for (int e = 0; e < 8; ++e) yr[q][e][0] = fmaf(hs_, wf[e], yr[q][e][0]);
            }
            continue;
          }
#pragma unroll
          for (int q = 0; q < CH; ++q) {
            const int ch = gt + q * kGroup;
            float wf[8];
            WT<T>::unpack(lds128z(buf, go + (size_t)ch * 16, g < kn && ch < chunks), wf);
#pragma unroll
            for (int b = 0; b < B; ++b)
#pragma unroll
              for (int e = 0; e < 8; ++e) yr[q][e][b] = fmaf(h[b], wf[e], yr[q][e][b]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_cnt(&empty[it % NS], 2);  // 8 down warps x 2
      }
      if constexpr (!SPEC) store_partial<B, CH>(yr, p.ypart + (size_t)c * B * d, d, gt, chunks);
    }
    int n_corr_st = 0;
    if constexpr (SPEC) {
      // corrections: a speculative neuron whose bit is 0 for token b gets h = -(its speculative h)
      const int n_corr = s_ncorr;
      n_corr_st = (n_corr + G - 1) / G;
      for (int f = 0; f < n_corr_st; ++f) {
        const uint32_t it = it_ffn + n_st + f;
        const int kk = f * G, kn = min(G, n_corr - kk);
        if (is_up) {
          wait_full(it);
          if (warp == 0) {
            if (lane < kn * B) hs[(it % NS) * (NA * B) + lane] = s_corr_h[kk + lane / B][lane % B];
            __syncwarp();
            mbar_arrive(&hready[it % NS]);   // every writer lane releases its own h
          }
        } else {
          wait_full(it);
          mbar_wait(&hready[it % NS], (it / NS) & 1);
          spec_down_stage<T, B, CH, NA>(pick<SPEC>(yrs, yrs), stage_ptr(it), hs + (it % NS) * (NA * B), kn, nb,
                                        row_up, gt, chunks);
          __syncwarp();
          if (lane == 0) mbar_arrive_cnt(&empty[it % NS], 2);  // 8 down warps x 2
        }
      }
    }
    if constexpr (SPEC) {
      if (!is_up) store_partial<B, CH>(yrs, p.ypart + (size_t)c * B * d, d, gt, chunks);
    }
    ring = it_ffn + n_st + n_corr_st;

    if (tr && tid == 0) tr[6] = globaltimer();
    grid_sync(p.bar, P, tr ? tr + 208 : nullptr);
    if (tr && tid == 0) tr[7] = globaltimer();

    // ---------------- phase 4: y[:, cols of CTA c] = sum over P partials + b_down ----------------
    // CTA c owns the 8-column units [u0, u1) of d (32-byte sectors).  Work item = (group of <= 8
    // partials, 4-column chunk, token): one 16-byte load per partial, all of a thread's loads in
    // flight at once; the group sums are combined in ascending group order (fixed order).
    {
      constexpr int PPG = 8;    // partials per group
      const int u0 = (int)(((int64_t)c * (d >> 3)) / P), u1 = (int)(((int64_t)(c + 1) * (d >> 3)) / P);
      const int nq = 2 * (u1 - u0);            // 4-column chunks of this CTA
      const int items = nq * B;
      const int SPL = max((P + PPG - 1) / PPG, min(32, kConsumers / max(1, items)));
      float4 *part = reinterpret_cast<float4 *>(s_part);   // [SPL][items]
      for (int idx = tid; idx < items * SPL; idx += kConsumers) {
        const int sgp = idx / items, it2 = idx - sgp * items;
        const int b = it2 / nq, j = u0 * 8 + (it2 - b * nq) * 4;
        const int c0 = (sgp * P) / SPL, c1 = ((sgp + 1) * P) / SPL;
        float4 v[PPG];
#pragma unroll
        for (int q = 0; q < PPG; ++q)
          v[q] = (c0 + q < c1) ? __ldcg(reinterpret_cast<const float4 *>(p.ypart + ((size_t)(c0 + q) * B + b) * d + j))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 acc = v[0];
#pragma unroll
        for (int q = 1; q < PPG; ++q) {
          acc.x += v[q].x; acc.y += v[q].y; acc.z += v[q].z; acc.w += v[q].w;
        }
        part[sgp * items + it2] = acc;
      }
      consumers_sync();
      for (int it2 = tid; it2 < items; it2 += kConsumers) {
        const int b = it2 / nq, j = u0 * 8 + (it2 - b * nq) * 4;
        float4 acc = part[it2];
        for (int sgp = 1; sgp < SPL; ++sgp) {
          const float4 w4 = part[sgp * items + it2];
          acc.x += w4.x; acc.y += w4.y; acc.z += w4.z; acc.w += w4.w;
        }
        if (lw.b_down) {
          acc.x += WT<T>::to_float(lw.b_down, j);
          acc.y += WT<T>::to_float(lw.b_down, j + 1);
          acc.z += WT<T>::to_float(lw.b_down, j + 2);
          acc.w += WT<T>::to_float(lw.b_down, j + 3);
        }
        *reinterpret_cast<float4 *>(yout + (size_t)b * d + j) = acc;
      }
    }
    if (tr && tid == 0) tr[8] = globaltimer();
    if (p.defer_ring == 1 && l < L - 1) {
      consumers_sync();
      if (tid == 0) mbar_arrive(&s_layer_done);
    }
    if (l < L - 1) grid_sync(p.bar, P, tr ? tr + 216 : nullptr);   // the next layer reads all of y
    if (p.defer_ring == 2 && l < L - 1 && tid == 0) mbar_arrive(&s_layer_done);
  }
}


template <typename T, int B, bool REGLU, int CH, int NA>
inline cudaError_t fused_launch_t(const FusedWork &w, const FusedParams &prm, cudaStream_t s) {
  auto kern = k_layer<T, B, REGLU, CH, NA, false, false>;
  int grid = w.P;
  if (prm.group_ctas > 0) {   // grouped launch: B = 1, d <= 8192, 16-bit rows (fused_group_supported)
    if constexpr (B == 1 && (CH <= 2 || (CH <= 4 && NA == 1))) {
      kern = k_layer<T, B, REGLU, CH, NA, false, false, true>;
      grid = w.P * w.groups;
    } else {
      return cudaErrorNotSupported;
    }
  }
  if (prm.group_ctas > 0 && (prm.spec || prm.rec_q4 > 0)) return cudaErrorNotSupported;
  // the speculative variant: d <= 8192, one or eight neurons per stage (other shapes run unspeculated,
  // which gives the same result: the default kernel ignores the speculative tables)
  if constexpr (CH <= 4 && (NA == 1 || NA == 8)) {
    if (prm.spec) kern = k_layer<T, B, REGLU, CH, NA, true, false>;
  }
  // INT4 rows (B = 1; 16-bit kernels only otherwise): the (CH, NA) shapes fused_geometry picks for records
  if constexpr (B == 1 && ((CH <= 2 && NA >= 4) || (CH >= 3 && CH <= 4 && NA == 4) || (CH >= 5 && NA == 2))) {
    if (prm.rec_q4 > 0) kern = k_layer<T, B, REGLU, CH, NA, false, true>;
  } else {
    if (prm.rec_q4 > 0) return cudaErrorNotSupported;
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, w.smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = (size_t)w.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, prm);
}

// the instantiated (CH, NA) combinations for one (T, B, REGLU); fused_supported() mirrors this list
template <typename T, int B, bool RG>
cudaError_t fused_launch_tbr(const FusedWork &w, const FusedParams &p, int CH, int NA, cudaStream_t s) {
#define PI_FL(CHV, NAV) \
  if (CH == CHV && NA == NAV) return fused_launch_t<T, B, RG, CHV, NAV>(w, p, s);
  PI_FL(1, 8) PI_FL(1, 4) PI_FL(1, 2) PI_FL(1, 1) PI_FL(2, 8) PI_FL(2, 4) PI_FL(2, 2) PI_FL(2, 1) PI_FL(3, 1) PI_FL(4, 1)
  if constexpr (B == 1) {   // wider d keeps x and y register-resident only for one token
    PI_FL(5, 1) PI_FL(6, 1) PI_FL(7, 1) PI_FL(8, 1)
    PI_FL(3, 4) PI_FL(4, 4) PI_FL(5, 2) PI_FL(6, 2) PI_FL(7, 2) PI_FL(8, 2)   // INT4 rows, 2-4 neurons per stage
  }
#undef PI_FL
  return cudaErrorNotSupported;
}

#define PI_FUSED_INSTANTIATE(T, B, RG) \
  template cudaError_t fused_launch_tbr<T, B, RG>(const FusedWork &, const FusedParams &, int, int, cudaStream_t);

}  // namespace pi
