// microbench_barrier.cu -- cost of one grid-wide barrier among 148 persistent CTAs (one per SM),
// with and without TMA bulk-copy traffic in flight on the same SMs (the k_layer situation: the
// producer warp keeps streaming weights while the consumer warps synchronise).
//   variant 0: atom.add.release.gpu + per-CTA flags written by the last arrival (k_layer today)
//   variant 1: same, relaxed atom (no release fence) -- not a correct publish, fence-cost probe
//   variant 2: fence.acq_rel.gpu by lane 0 only after bar.sync, then relaxed atom
//   variant 3: red.release.gpu arrival + every CTA polls the counter line itself
//   variant 4: per-CTA arrival flags (st.release), CTA 0 gathers and broadcasts (flag tree)
// Each consumer thread stores `st_bytes` of fp32 to global before each barrier (0 or 32 KB per CTA,
// the size of a k_layer down partial), so the release has something to drain.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/microbench_barrier.cu -o /tmp/mbb
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t *b, uint32_t par) {
  uint32_t done = 0;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
               : "=r"(done) : "r"(sa(b)), "r"(par) : "memory");
  return done;
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t n, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(n), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ unsigned long long ldacq(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kCons = 512;
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory"); }

template <int V>
__device__ __forceinline__ void gsync(unsigned long long *bar, int P, int ns, unsigned long long iep) {
  csync();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int c = blockIdx.x;
    if (V == 5 || V == 6) {
      constexpr int K = (V == 5) ? 8 : 16;
      unsigned long long *cnt = bar + 16 * 1024;   // K counters, 1 KB apart
      if (lane == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(cnt + 128 * (c % K)), "l"(1ull) : "memory");
      }
      __syncwarp();
      const unsigned long long ep = iep;
      if (lane < K) {
        const unsigned long long need = ep * (unsigned long long)((P - lane + K - 1) / K);
        while (ldacq(cnt + 128 * lane) < need) __nanosleep(ns);
      }
      __syncwarp();
    } else if (V == 4) {
      // arrival flag per CTA; CTA 0 warp 0 gathers, then writes every CTA's release flag
      unsigned long long *arr = bar + 16 * 512;
      static __shared__ unsigned long long epi;
      if (lane == 0) {
        epi = ldacq(bar + 16 * (1 + c)) + 1;  // my last seen episode + 1 (only I read my flag)
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(arr + 16 * c), "l"(epi) : "memory");
      }
      __syncwarp();
      const unsigned long long ep = epi;
      if (c == 0) {
        for (int cc = lane; cc < P; cc += 32)
          while (ldacq(arr + 16 * cc) < ep) __nanosleep(ns);
        __syncwarp();
        for (int cc = lane; cc < P; cc += 32)
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(bar + 16 * (1 + cc)), "l"(ep) : "memory");
      }
      if (lane == 0)
        while (ldacq(bar + 16 * (1 + c)) < ep) __nanosleep(ns);
    } else {
      unsigned long long old = 0;
      if (lane == 0) {
        if (V == 0) asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
        if (V == 1) asm volatile("atom.add.relaxed.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
        if (V == 2) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          asm volatile("atom.add.relaxed.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
        }
        if (V == 3) asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
      }
      old = __shfl_sync(0xffffffffu, old, 0);
      const unsigned long long ep = old / (unsigned long long)P + 1ull;
      if (V == 3) {
        if (lane == 0)
          while (ldacq(bar) < ep * (unsigned long long)P) __nanosleep(ns);
      } else {
        if (old % (unsigned long long)P == (unsigned long long)(P - 1))
          for (int cc = lane; cc < P; cc += 32)
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(bar + 16 * (1 + cc)), "l"(ep) : "memory");
        if (lane == 0)
          while (ldacq(bar + 16 * (1 + blockIdx.x)) < ep) __nanosleep(ns);
      }
    }
  }
  csync();
}

// warps 0..15: barrier loop; warp 16: TMA producer (if stream); warp 17: stage drainer
template <int V>
__global__ void __launch_bounds__(576, 1) k_bar(unsigned long long *bar, int iters, int ns, int stream,
                                                const uint8_t *src, size_t src_bytes, float *scratch,
                                                int st_floats, unsigned long long *out, int *stop) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int NS = 6, SB = 32768;
  uint64_t *full = (uint64_t *)(sm + NS * SB), *empty = full + NS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P = gridDim.x, c = blockIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 16) {
    if (!stream || lane) return;
    const size_t per = (src_bytes / P) & ~(size_t)32767;
    const uint8_t *base = src + per * c;
    size_t off = 0;
    auto drain = [&](uint32_t it) {
      for (uint32_t j = (it > (uint32_t)NS ? it - NS : 0); j < it; ++j)
        while (!mbar_try(&full[j % NS], (j / NS) & 1)) {}
    };
    if (stream == 4) {
      unsigned long long tn;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
      while (!*(volatile int *)stop) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t < tn) continue;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(32768u) : "memory");
        off += SB;
        if (off + SB > per) off = 0;
        tn += 740;
      }
      return;
    }
    const int depth = stream == 1 ? NS : stream == 2 ? 2 : 1;
    for (uint32_t it = 0;; ++it) {
      const int s = it % NS;
      if (it >= (uint32_t)depth)
        while (!mbar_try(&full[(it - depth) % NS], ((it - depth) / NS) & 1))
          if (*(volatile int *)stop) { drain(it); return; }
      if (it >= NS)
        while (!mbar_try(&empty[s], ((it / NS) - 1) & 1))
          if (*(volatile int *)stop) { drain(it); return; }
      if (*(volatile int *)stop) { drain(it); return; }
      mbar_expect(&full[s], SB);
      bulk(sm + s * SB, base + off, SB, &full[s]);
      off += SB;
      if (off + SB > per) off = 0;
    }
  }
  if (warp == 17) {
    if (!stream || stream == 4 || lane) return;
    for (uint32_t it = 0;; ++it) {
      const int s = it % NS;
      while (!mbar_try(&full[s], (it / NS) & 1))
        if (*(volatile int *)stop) return;
      mbar_arrive(&empty[s]);
    }
  }
  unsigned long long t0 = 0;
  for (int i = 0; i < iters; ++i) {
    if (i == 8) {
      csync();
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    }
    for (int k = tid; k < st_floats; k += kCons) __stcg(scratch + (size_t)c * st_floats + k, (float)(i + k));
    gsync<V>(bar, P, ns, (unsigned long long)(i + 1));
  }
  if (tid == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[c] = t1 - t0;
    atomicAdd(stop, 1);   // once every CTA is done, stop > 0 everywhere soon after; producers exit
  }
}

template <int V>
float run(unsigned long long *bar, int iters, int ns, int stream, const uint8_t *src, size_t sb, float *scr, int stf,
          unsigned long long *out, int *stop, int P) {
  cudaMemset(bar, 0, 1 << 20);
  cudaMemset(stop, 0, 4);
  auto k = k_bar<V>;
  const int smem = 6 * 32768 + 256;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(P);
  cfg.blockDim = dim3(576);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, bar, iters, ns, stream, src, sb, scr, stf, out, stop);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return -1; }
  unsigned long long h[256];
  cudaMemcpy(h, out, P * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < P; ++i) mx = h[i] > mx ? h[i] : mx;
  return (float)mx / (iters - 8) / 1000.f;
}

int main() {
  int P = 0;
  cudaDeviceGetAttribute(&P, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *bar, *out;
  int *stop;
  uint8_t *src;
  float *scr;
  const size_t sb = (size_t)4 << 30;
  cudaMalloc(&bar, 1 << 20);
  cudaMalloc(&out, 256 * 8);
  cudaMalloc(&stop, 4);
  cudaMalloc(&src, sb);
  cudaMemset(src, 1, sb);
  cudaMalloc(&scr, (size_t)P * 8192 * 4);
  const int iters = 2008;
  printf("P=%d; us per barrier (max over CTAs)\n", P);
  for (int stf : {0, 8192})
    for (int stream : {0, 1, 2, 3, 4})
      for (int ns : {32}) {
        float v0 = run<0>(bar, iters, ns, stream, src, sb, scr, stf, out, stop, P);
        float v1 = run<1>(bar, iters, ns, stream, src, sb, scr, stf, out, stop, P);
        float v2 = run<2>(bar, iters, ns, stream, src, sb, scr, stf, out, stop, P);
        float v3 = run<3>(bar, iters, ns, stream, src, sb, scr, stf, out, stop, P);
        float v4 = run<4>(bar, iters, ns, stream, src, sb, scr, stf, out, stop, P);
        float v5 = run<5>(bar, iters, ns, stream, src, sb, scr, stf, out, stop, P);
        float v6 = run<6>(bar, iters, ns, stream, src, sb, scr, stf, out, stop, P);
        printf("store %5d B/CTA stream %d nanosleep %3d : atom.rel+flags %.3f | relaxed %.3f | fence+relaxed %.3f | "
               "poll-counter %.3f | flag-tree %.3f | split8-red %.3f | split16-red %.3f\n",
               stf * 4, stream, ns, v0, v1, v2, v3, v4, v5, v6);
      }
  return 0;
}
