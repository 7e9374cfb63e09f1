// kg_common.cuh -- device helpers shared by the sm_100a kernels of libkg.so.
// (Product path.  Shares nothing with oracle/.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Programmatic dependent launch: every kernel of the library waits for its predecessor grids
// (memory visible) before touching their outputs.  In a captured step graph the kernel-to-
// kernel edges are programmatic (kg_api.cu make_programmatic), so a kernel is launched while
// its predecessor drains; outside such edges the instruction is a no-op.
#define KG_GRID_DEP_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

namespace kg {

enum Kind { GQE = 0, Q2B = 1, BETAE = 2, TRANSE = 3, ROTATE = 4, DISTMULT = 5, COMPLEX = 6 };

constexpr float kBetaLo = 0.05f;   // A8 positivity floor
constexpr float kBetaHi = 1e9f;    // A8 ceiling

__device__ __forceinline__ float sigmoidf_(float x) { return 1.f / (1.f + __expf(-x)); }

// softplus(z) = log(1 + e^z), stable in both tails.
__device__ __forceinline__ float softplusf_(float z) {
  return z > 0.f ? z + log1pf(expf(-z)) : log1pf(expf(z));
}
// exact-ish sigmoid for the loss adjoint (expf, not the fast intrinsic)
__device__ __forceinline__ float sigm_(float x) {
  return x >= 0.f ? 1.f / (1.f + expf(-x)) : expf(x) / (1.f + expf(x));
}

// digamma psi(x), x > 0: upward recurrence to x >= 6, then the asymptotic series.
__device__ __forceinline__ float digammaf_(float x) {
  float r = 0.f;
#pragma unroll 1
  while (x < 6.f) { r -= 1.f / x; x += 1.f; }
  const float f = 1.f / (x * x);
  const float t = f * (-1.f / 12.f + f * (1.f / 120.f + f * (-1.f / 252.f + f * (1.f / 240.f + f * (-1.f / 132.f)))));
  return r + logf(x) - 0.5f / x + t;
}

// trigamma psi'(x), x > 0.
__device__ __forceinline__ float trigammaf_(float x) {
  float r = 0.f;
#pragma unroll 1
  while (x < 6.f) { r += 1.f / (x * x); x += 1.f; }
  const float ix = 1.f / x, f = ix * ix;
  return r + ix + 0.5f * f + ix * f * (1.f / 6.f - f * (1.f / 30.f - f * (1.f / 42.f - f * (1.f / 30.f))));
}

__device__ __forceinline__ float lnbetaf_(float a, float b) { return lgammaf(a) + lgammaf(b) - lgammaf(a + b); }

__device__ __forceinline__ float beta_act(float x) { return fminf(fmaxf(x + 1.f, kBetaLo), kBetaHi); }
// clamp passes the gradient on the closed interval (A19)
__device__ __forceinline__ float beta_act_grad(float x) {
  const float y = x + 1.f;
  return (y >= kBetaLo && y <= kBetaHi) ? 1.f : 0.f;
}

// splitmix64 finaliser; counter-based uniform identical to kggen.counter_uniform.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ float counter_uniform(uint64_t seed, uint64_t stream, uint64_t idx, float lo, float hi) {
  const uint64_t s = mix64(seed ^ (stream * 0x9E3779B97F4A7C15ull));
  const uint64_t h = mix64(s + idx * 0xD1B54A32D192ED03ull);
  const float u = __fmul_rn((float)(uint32_t)(h >> 40), 5.9604644775390625e-08f);  // 2^-24
  return __fadd_rn(lo, __fmul_rn(__fsub_rn(hi, lo), u));
}

template <int N>
__device__ __forceinline__ float half_warp_sum(float v) {
#pragma unroll
  for (int o = N / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction (fixed tree order).  `red` needs blockDim/32 floats.
__device__ __forceinline__ float block_sum(float v, float *red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  if (w == 0) {
    s = l < nw ? red[l] : 0.f;
    s = warp_sum(s);
    if (l == 0) red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

}  // namespace kg
