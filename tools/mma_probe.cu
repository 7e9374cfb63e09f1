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

int main() {
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
  return 0;
}
