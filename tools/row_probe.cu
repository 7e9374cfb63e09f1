// row_probe.cu -- what random-row read-modify-write of 3 x [rows x d] fp32 tables can reach on
// one B200 (the access pattern of sparse Adam, K-new-5): N distinct sorted random rows of a
// 10.76 M-row table (the Freebase per-GPU shard), p / m / v read + written (24 d bytes per row).
// Variants: warp per row with registers (W), TMA bulk copies into shared memory (T), and a
// sequential-rows control (rows 0..N-1).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 row_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <vector>
#include <algorithm>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int IT>
__global__ void __launch_bounds__(256) warp_rows(const int64_t *rows, int n, int d4, float4 *p, float4 *m, float4 *v) {
  const int u = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (u >= n) return;
  const int64_t off = rows[u] * d4;
  float4 P[IT], M[IT], V[IT];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int c = lane + 32 * it;
    if (c < d4) { P[it] = p[off + c]; M[it] = m[off + c]; V[it] = v[off + c]; }
  }
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int c = lane + 32 * it;
    if (c < d4) {
      M[it].x = 0.9f * M[it].x + 0.1f * P[it].x; V[it].y += 1.f; P[it].z -= 1e-3f * M[it].x;
      p[off + c] = P[it]; m[off + c] = M[it]; v[off + c] = V[it];
    }
  }
}

// one thread per float4 column, one CTA of 128 threads per row (100 active at d = 400)
__global__ void __launch_bounds__(128) cta_rows(const int64_t *rows, int n, int d4, float4 *p, float4 *m, float4 *v) {
  const int u = blockIdx.x, c = threadIdx.x;
  if (u >= n || c >= d4) return;
  const int64_t off = rows[u] * d4 + c;
  float4 P = p[off], M = m[off], V = v[off];
  M.x = 0.9f * M.x + 0.1f * P.x; V.y += 1.f; P.z -= 1e-3f * M.x;
  p[off] = P; m[off] = M; v[off] = V;
}

__device__ __forceinline__ uint32_t su(const void *q) { return (uint32_t)__cvta_generic_to_shared(q); }
__global__ void __launch_bounds__(128) tma_rows(const int64_t *rows, int n, int d, float *p, float *m, float *v, int S) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bars[4][8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, d4 = d / 4;
  const int nw = gridDim.x * 4, gw = blockIdx.x * 4 + w;
  float *wr = sm + (size_t)w * S * 3 * d;
  if (lane == 0) for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bars[w][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int k) {
    const int u = gw + k * nw;
    if (u >= n) return;
    const int s = k % S;
    const int64_t r = rows[u];
    float *dst = wr + (size_t)s * 3 * d;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bars[w][s])), "r"(12u * d) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(dst)), "l"(p + r * d), "r"(4 * d), "r"(su(&bars[w][s])) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(dst + d)), "l"(m + r * d), "r"(4 * d), "r"(su(&bars[w][s])) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(dst + 2 * d)), "l"(v + r * d), "r"(4 * d), "r"(su(&bars[w][s])) : "memory");
  };
  if (lane == 0) for (int k = 0; k < S; ++k) issue(k);
  for (int k = 0;; ++k) {
    const int u = gw + k * nw;
    if (u >= n) break;
    const int s = k % S;
    uint32_t done = 0, par = (k / S) & 1;
    while (!done) asm volatile("{\n.reg .pred q;\nmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\nselp.u32 %0, 1, 0, q;\n}\n" : "=r"(done) : "r"(su(&bars[w][s])), "r"(par) : "memory");
    const float4 *sp = reinterpret_cast<const float4 *>(wr + (size_t)s * 3 * d);
    const int64_t off = rows[u] * d4;
    for (int c = lane; c < d4; c += 32) {
      float4 P = sp[c], M = sp[d4 + c], V = sp[2 * d4 + c];
      M.x = 0.9f * M.x + 0.1f * P.x; V.y += 1.f; P.z -= 1e-3f * M.x;
      reinterpret_cast<float4 *>(p)[off + c] = P; reinterpret_cast<float4 *>(m)[off + c] = M; reinterpret_cast<float4 *>(v)[off + c] = V;
    }
    __syncwarp();
    if (lane == 0) issue(k + S);
  }
}

int main() {
  const int64_t R = 10756769;
  const int d = 400, d4 = d / 4;
  float *p, *m, *v;
  CK(cudaMalloc(&p, R * d * 4)); CK(cudaMalloc(&m, R * d * 4)); CK(cudaMalloc(&v, R * d * 4));
  CK(cudaMemset(p, 0, R * d * 4)); CK(cudaMemset(m, 0, R * d * 4)); CK(cudaMemset(v, 0, R * d * 4));
  char *flush; CK(cudaMalloc(&flush, 512 << 20));
  int64_t *drows; CK(cudaMalloc(&drows, 8 * 400000));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  CK(cudaFuncSetAttribute(tma_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  std::mt19937_64 rng(1);
  printf("rows,pattern,variant,us,GBps\n");
  for (int n : {2400, 12000, 50000, 200000}) {
    for (int pat = 0; pat < 2; ++pat) {
      std::vector<int64_t> rows(n);
      if (pat == 0) { std::vector<int64_t> all; for (int i = 0; i < n; ++i) rows[i] = (int64_t)(rng() % R); std::sort(rows.begin(), rows.end()); rows.erase(std::unique(rows.begin(), rows.end()), rows.end()); }
      else for (int i = 0; i < n; ++i) rows[i] = i;
      const int nn = (int)rows.size();
      CK(cudaMemcpy(drows, rows.data(), 8 * nn, cudaMemcpyHostToDevice));
      for (int var = 0; var < 5; ++var) {
        float best = 1e9;
        for (int rep = 0; rep < 7; ++rep) {
          CK(cudaMemset(flush, rep, 512 << 20));
          cudaEventRecord(a);
          if (var == 0) warp_rows<4><<<(nn + 7) / 8, 256>>>(drows, nn, d4, (float4 *)p, (float4 *)m, (float4 *)v);
          if (var == 1) cta_rows<<<nn, 128>>>(drows, nn, d4, (float4 *)p, (float4 *)m, (float4 *)v);
          if (var >= 2) {
            const int S = var == 2 ? 2 : (var == 3 ? 3 : 6);
            const int cpsm = std::max(1, 220 * 1024 / (4 * S * 12 * d + 1024));
            const int grid = std::min(148 * cpsm, (nn + 3) / 4);
            tma_rows<<<grid, 128, 4 * S * 12 * d>>>(drows, nn, d, p, m, v, S);
          }
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          float ms; cudaEventElapsedTime(&ms, a, b);
          if (rep > 0) best = std::min(best, ms);
        }
        const char *nm[] = {"warp_regs", "cta_per_row", "tma_S2", "tma_S3", "tma_S6"};
        printf("%d,%s,%s,%.1f,%.0f\n", nn, pat ? "sequential" : "random", nm[var], best * 1e3, 24.0 * d * nn / (best * 1e-3) / 1e9);
      }
    }
  }
  CK(cudaGetLastError());
  return 0;
}
