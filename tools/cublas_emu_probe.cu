// cublas_emu_probe.cu -- cuBLAS SGEMM: native fp32 vs the BF16x9 fp32 emulation (cuBLAS 12.9,
// Blackwell tensor cores) on the BetaE MLP shapes: time (CUDA events) and error / (|A||B|) vs fp64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 cublas_emu_probe.cu -lcublas
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <random>
#include <algorithm>

int main() {
  cublasHandle_t h;
  cublasCreate(&h);
  struct S { int m, n, k; } shapes[] = {{1536, 1600, 800}, {1536, 1600, 1600}, {1536, 400, 1600}, {1600, 1600, 1536}, {1024, 400, 400}};
  std::mt19937 rng(1);
  std::normal_distribution<float> nd;
  printf("m,n,k,mode,us,TFLOPs,err_max,err_mean\n");
  for (auto s : shapes) {
    const int m = s.m, n = s.n, k = s.k;
    std::vector<float> A((size_t)m * k), B((size_t)k * n), C((size_t)m * n);
    for (auto &x : A) x = std::max(nd(rng), 0.f);                                   // ReLU activations
    for (auto &x : B) x = nd(rng) * powf(10.f, -3.f * (rng() % 1000) / 1000.f);     // mixed-sign, 3 decades
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    // reference on a sample of 4096 outputs (column-major C = A B with A [m x k], B [k x n])
    std::vector<int> ri(4096), ci(4096);
    for (int t = 0; t < 4096; ++t) { ri[t] = rng() % m; ci[t] = rng() % n; }
    for (int mode = 0; mode < 2; ++mode) {
      cublasSetMathMode(h, mode ? CUBLAS_FP32_EMULATED_BF16X9_MATH : CUBLAS_DEFAULT_MATH);
      if (mode) cublasSetEmulationStrategy(h, CUBLAS_EMULATION_STRATEGY_EAGER);
      const float one = 1.f, zero = 0.f;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      float best = 1e9;
      for (int rep = 0; rep < 10; ++rep) {
        cudaEventRecord(a);
        cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, m, n, k, &one, dA, m, dB, k, &zero, dC, m);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
      }
      cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
      double emax = 0, esum = 0;
      for (int t = 0; t < 4096; ++t) {
        double ref = 0, absr = 0;
        for (int kk = 0; kk < k; ++kk) {
          const double p = (double)A[(size_t)kk * m + ri[t]] * (double)B[(size_t)ci[t] * k + kk];
          ref += p; absr += fabs(p);
        }
        const double e = fabs(C[(size_t)ci[t] * m + ri[t]] - ref) / std::max(absr, 1e-30);
        emax = std::max(emax, e); esum += e;
      }
      printf("%d,%d,%d,%s,%.1f,%.1f,%.2e,%.2e\n", m, n, k, mode ? "bf16x9" : "sgemm", best * 1e3,
             2.0 * m * n * k / (best * 1e-3) / 1e12, emax, esum / 4096);
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dC);
  }
  return 0;
}
