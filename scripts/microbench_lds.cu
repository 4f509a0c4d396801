// microbench_lds.cu -- shared-memory read rate of the k_layer P2 inner loop pattern (8 LDS.128 per
// lane + 64 FMA + transpose reduction per 4 rows), 16 warps per CTA, 148 CTAs, optionally with a
// TMA producer streaming HBM into other ring slots of the same shared memory.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/microbench_lds.cu -o /tmp/mbl
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
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

template <int MODE>  // 0: 8 loads interleaved (compiler order) 1: loads batched via volatile asm, 2: LDS.32
__global__ void __launch_bounds__(576, 1) k(const uint8_t *src, size_t src_bytes, int stream, int iters, float *out,
                                            unsigned long long *cyc, int *stop) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int NS = 4, SB = 32768;   // 4 streaming slots + 2 compute slots
  uint8_t *cbuf = sm + NS * SB;       // 64 KB read by the compute warps
  uint64_t *full = (uint64_t *)(sm + (NS + 2) * SB), *empty = full + NS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 2 * SB / 4; i += 576) ((uint32_t *)cbuf)[i] = 0x3f803f80u ^ (i * 2654435761u & 0x00ff00ffu);
  __syncthreads();
  if (warp == 16) {
    if (!stream || lane) return;
    const size_t per = (src_bytes / gridDim.x) & ~(size_t)32767;
    const uint8_t *base = src + per * blockIdx.x;
    size_t off = 0;
    uint32_t it = 0;
    for (;; ++it) {
      const int s = it % NS;
      bool stopped = false;
      if (it >= NS)
        while (!mbar_try(&empty[s], ((it / NS) - 1) & 1))
          if (*(volatile int *)stop) { stopped = true; break; }
      if (stopped || *(volatile int *)stop) break;
      mbar_expect(&full[s], SB);
      bulk(sm + s * SB, base + off, SB, &full[s]);
      off += SB;
      if (off + SB > per) off = 0;
    }
    for (uint32_t j = (it > (uint32_t)NS ? it - NS : 0); j < it; ++j)
      while (!mbar_try(&full[j % NS], (j / NS) & 1)) {}
    return;
  }
  if (warp == 17) {
    if (!stream || lane) return;
    for (uint32_t it = 0;; ++it) {
      const int s = it % NS;
      while (!mbar_try(&full[s], (it / NS) & 1))
        if (*(volatile int *)stop) return;
      mbar_arrive(&empty[s]);
    }
  }
  if (MODE == 2) {
    // dependent shared-load chain (latency): idx = cbuf32[idx], 64 KB region, stride 1 KB + 4 B
    uint32_t *c32 = (uint32_t *)cbuf;
    for (int i = tid; i < 2 * SB / 4; i += 512) c32[i] = (uint32_t)((i + 257) % (2 * SB / 4));
    asm volatile("bar.sync 1, 512;" ::: "memory");
    uint32_t idx = (uint32_t)(warp * 64 + lane);
    const long long c0 = clock64();
    for (int itr = 0; itr < iters; ++itr) {
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(idx) : "r"(sa(c32 + idx)));
    }
    const long long c1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 16 + warp] = (unsigned long long)(c1 - c0);
    if (idx == 0xffffffffu) out[tid] = 1.f;
    asm volatile("bar.sync 1, 512;" ::: "memory");
    if (tid == 0) atomicAdd(stop, 1);
    return;
  }
  // compute warps: each iteration, 4 rows of r = 512 bf16 from cbuf (row-major, 1 KB rows)
  float g[2][8];
  for (int q = 0; q < 2; ++q)
    for (int e = 0; e < 8; ++e) g[q][e] = 0.001f * (lane + q + e);
  float acc_out = 0.f;
  const long long c0 = clock64();
  for (int itr = 0; itr < iters; ++itr) {
    const int rb0 = ((warp * 4 + itr * 64) & 63);
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    uint4 w[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint8_t *pp = cbuf + (size_t)(rb0 + i) * 1024 + (lane + 32 * q) * 16;
        if (MODE == 1)
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(w[i][q].x), "=r"(w[i][q].y), "=r"(w[i][q].z), "=r"(w[i][q].w) : "r"(sa(pp)));
        else
          w[i][q] = *(const uint4 *)pp;
      }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t u[4] = {w[i][q].x, w[i][q].y, w[i][q].z, w[i][q].w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          v[i] = fmaf(__uint_as_float(u[h] << 16), g[q][2 * h], v[i]);
          v[i] = fmaf(__uint_as_float(u[h] & 0xffff0000u), g[q][2 * h + 1], v[i]);
        }
      }
    // transpose reduction of 4 values
    {
      const bool up2 = lane & 2;
      float s0 = up2 ? v[0] : v[2], k0 = up2 ? v[2] : v[0];
      float s1 = up2 ? v[1] : v[3], k1 = up2 ? v[3] : v[1];
      v[0] = k0 + __shfl_xor_sync(0xffffffffu, s0, 2);
      v[1] = k1 + __shfl_xor_sync(0xffffffffu, s1, 2);
      const bool up1 = lane & 1;
      float s = up1 ? v[0] : v[1], kk = up1 ? v[1] : v[0];
      float r = kk + __shfl_xor_sync(0xffffffffu, s, 1);
      for (int o = 4; o < 32; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
      acc_out += r;
    }
  }
  const long long c1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 16 + warp] = (unsigned long long)(c1 - c0);
  if (acc_out == 1.2345f) out[tid] = acc_out;
  asm volatile("bar.sync 1, 512;" ::: "memory");
  if (tid == 0) atomicAdd(stop, 1);
}

template <int MODE>
void run(const uint8_t *src, size_t sb, int stream, int iters, float *out, unsigned long long *cyc, int *stop, int P,
         int warps_active) {
  cudaMemset(stop, 0, 4);
  const int smem = 6 * 32768 + 128;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<MODE><<<P, 576, smem>>>(src, sb, stream, iters, out, cyc, stop);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  static unsigned long long h[148 * 16];
  cudaMemcpy(h, cyc, P * 16 * 8, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < P * 16; ++i) s += h[i];
  const double per_it = s / (P * 16) / iters;
  // bytes read per iteration by all 16 warps of a CTA: 16 * 4 rows * 1 KB
  if (MODE == 2)
    printf("mode 2 stream %d : dependent LDS latency %.1f cycles (16 warps chasing)\n", stream, per_it);
  else
    printf("mode %d stream %d : %.0f cycles per iteration per warp -> %.1f B/clk/SM of LDS\n", MODE, stream, per_it,
           16.0 * 4096 / per_it);
  fflush(stdout);
}

int main() {
  int P = 0;
  cudaDeviceGetAttribute(&P, cudaDevAttrMultiProcessorCount, 0);
  uint8_t *src;
  const size_t sb = (size_t)2 << 30;
  cudaMalloc(&src, sb);
  cudaMemset(src, 1, sb);
  float *out;
  unsigned long long *cyc;
  int *stop;
  cudaMalloc(&out, 4096 * 4);
  cudaMalloc(&cyc, 148 * 16 * 8);
  cudaMalloc(&stop, 4);
  for (int stream : {0, 1}) {
    run<0>(src, sb, stream, 2000, out, cyc, stop, P, 16);
    run<1>(src, sb, stream, 2000, out, cyc, stop, P, 16);
    run<2>(src, sb, stream, 20000, out, cyc, stop, P, 16);
  }
  return 0;
}
