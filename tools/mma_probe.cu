// mma_probe.cu -- issue-to-completion throughput of back-to-back tcgen05.mma on one SM
// (kind::tf32 128 x N x 8 with A from shared memory or from TMEM; kind::f16 128 x N x 16 bf16),
// the denominator of the tensor-core GEMM's pacing (tools/gemm_trace.py).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe tools/mma_probe.cu && /tmp/mma_probe
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) {   // K-major, SWIZZLE_64B rows of 64 B
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

template <int N, int MODE, int GROUP = 0>   // MODE 0: tf32 SS, 1: tf32 TS (A in TMEM), 2: bf16 SS; GROUP > 0: commit every GROUP MMAs
__global__ void probe(int reps, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float *>(smem)[i] = 0.f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc_tf32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t idesc_bf16 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = kdesc(su32(smem)), db = kdesc(su32(smem + 32 * 1024));
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (MODE == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm), "l"(da), "l"(db), "r"(idesc_tf32), "r"(r));
      else if (MODE == 1)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tm), "r"(tm + 256), "l"(db), "r"(idesc_tf32), "r"(r));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm), "l"(da), "l"(db), "r"(idesc_bf16), "r"(r));
      if (GROUP > 0 && r % GROUP == GROUP - 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(su32(&bar)));
    out[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int MODE, int GROUP = 0>
void run(const char *name) {
  unsigned long long *d, h[148];
  cudaMalloc(&d, sizeof(h));
  cudaFuncSetAttribute(probe<N, MODE, GROUP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int reps = 4096;
  probe<N, MODE, GROUP><<<148, 128, 96 * 1024>>>(reps, d);
  probe<N, MODE, GROUP><<<148, 128, 96 * 1024>>>(reps, d);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double cyc = (double)h[0] / reps;
  const double kk = MODE == 2 ? 16 : 8;
  const double flop = 2.0 * 128 * N * kk;
  printf("%-28s N=%3d: %7.1f cycles / MMA  %7.0f FLOP/clk/SM  (%s)\n", name, N, cyc, flop / cyc,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}


// The GEMM's MMA-warp pattern: per k-block 6 TS MMAs (hi.lo, lo.hi, hi.hi over 2 k-steps) on a
// stage s of S (B descriptors and A TMEM columns change with s), then optionally an mbarrier
// wait on an already-completed barrier + tcgen05.fence (WAIT) per k-block, a commit every G.
template <int N, int S, int G, int WAIT, bool FENCE>
__global__ void pattern(int nkb, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar, gbar, done_bar, gbar2[2];
  __shared__ uint32_t tbase, flag;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<float *>(smem)[i] = 0.f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&gbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&done_bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&gbar2[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&gbar2[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar)) : "memory");   // phase 0 done
    flag = 1;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (WAIT == 5 ? warp == 0 : threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64();
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % S;
      if (WAIT == 1 || (WAIT == 3 && kb % G == 0)) {   // try_wait per k-block / per group
        uint32_t done = 0;
        while (!done)
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(done) : "r"(su32(&bar)) : "memory");
      }
      if (WAIT == 5 && kb % G == 0) {   // named barrier (g & 1) + 1 with warp 1, whole warp 0
        if ((kb / G) & 1) asm volatile("bar.sync 2, 64;" ::: "memory");
        else asm volatile("bar.sync 1, 64;" ::: "memory");
      }
      if (WAIT == 4) {   // acquire-load spin on a shared-memory flag (no mbarrier op) per k-block
        uint32_t v = 0;
        while (v == 0) asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(su32(&flag)) : "memory");
      }
      if (WAIT == 2) {   // test_wait (non-blocking) per k-block
        uint32_t done = 0;
        while (!done)
          asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(done) : "r"(su32(&bar)) : "memory");
      }
      if (FENCE) asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t st = su32(smem + s * 24 * 1024);
      const uint32_t ta = tm + 256 + 32 * (s % 8);
      uint32_t leader = 1;
      if (WAIT == 5) asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(leader));
      if (leader)
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const uint64_t dbh = kdesc(st + kk * 32), dbl = kdesc(st + 12 * 1024 + kk * 32);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tm), "r"(ta + 8 * kk), "l"(dbl), "r"(idesc), "r"(kb + kk));
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tm), "r"(ta + 16 + 8 * kk), "l"(dbh), "r"(idesc), "r"(1));
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tm), "r"(ta + 8 * kk), "l"(dbh), "r"(idesc), "r"(1));
      }
      if (kb % G == G - 1 && leader)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            su32(WAIT == 5 ? &gbar2[(kb / G) & 1] : &gbar)));
      if (WAIT == 5) __syncwarp();
    }
    if (threadIdx.x == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&done_bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(su32(&done_bar)));
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  if (WAIT == 5 && warp == 1) {   // the waiter: one arrival per group on named barrier 1 (64 threads)
    for (int kb = 0; kb < nkb; kb += G) {
      const int gg = kb / G;
      if (gg >= 2) {   // back-pressure as in the GEMM: group gg's stages are free once group gg - 2 completed
        const int gw = gg - 2;
        uint32_t done = 0;
        while (!done)
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(done) : "r"(su32(&gbar2[gw & 1])), "r"((gw >> 1) & 1) : "memory");
      }
      if ((kb / G) & 1) asm volatile("bar.arrive 2, 64;" ::: "memory");
      else asm volatile("bar.arrive 1, 64;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int S, int G, int WAIT, bool FENCE>
void run_pattern(const char *name) {
  unsigned long long *d, h[148];
  cudaMalloc(&d, sizeof(h));
  cudaFuncSetAttribute(pattern<N, S, G, WAIT, FENCE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int nkb = 400;
  pattern<N, S, G, WAIT, FENCE><<<148, 128, 200 * 1024>>>(nkb, d);
  pattern<N, S, G, WAIT, FENCE><<<148, 128, 200 * 1024>>>(nkb, d);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-44s N=%3d: %7.1f cycles / k-block (6 MMAs = %d cycles of pipe)  (%s)\n", name, N, (double)h[0] / nkb,
         6 * N / 2, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  run<64, 0>("tf32 SS 128xNx8");
  run<128, 0>("tf32 SS 128xNx8");
  run<160, 0>("tf32 SS 128xNx8");
  run<256, 0>("tf32 SS 128xNx8");
  run<128, 1>("tf32 TS (A in TMEM) 128xNx8");
  run<256, 1>("tf32 TS (A in TMEM) 128xNx8");
  run<128, 2>("bf16 SS 128xNx16");
  run<256, 2>("bf16 SS 128xNx16");
  run<128, 0, 6>("tf32 SS, commit every 6");
  run<128, 0, 12>("tf32 SS, commit every 12");
  run<128, 0, 1>("tf32 SS, commit every 1");
  run_pattern<128, 8, 4, 0, false>("pattern: no wait, no fence, commit/4");
  run_pattern<128, 8, 4, 1, false>("pattern: try_wait/kb, commit/4");
  run_pattern<128, 8, 4, 2, false>("pattern: test_wait/kb, commit/4");
  run_pattern<128, 8, 4, 3, false>("pattern: try_wait/group, commit/4");
  run_pattern<128, 8, 4, 3, true>("pattern: try_wait/group + fence/kb, commit/4");
  run_pattern<128, 8, 4, 0, true>("pattern: fence/kb only, commit/4");
  run_pattern<128, 8, 4, 4, true>("pattern: flag spin + fence/kb, commit/4");
  run_pattern<128, 8, 4, 5, true>("pattern: named barrier/group + fence/kb, c/4");
  run_pattern<128, 8, 1, 5, true>("pattern: named barrier/kb + fence/kb, c/1");
  run_pattern<160, 6, 3, 4, true>("pattern: flag spin + fence/kb, commit/3");
  run_pattern<160, 6, 3, 3, false>("pattern: try_wait/group, commit/3");
  return 0;
}
