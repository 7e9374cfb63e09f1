// k_gemm.cu -- dense contractions of the query DAG on the 5th-generation tensor
// cores (tcgen05, TMEM accumulators, TMA), fp32-accurate through a 3xTF32 split.
//
// The BetaE projection MLP (reading A9; Table 1 'MLP') and the d x d
// DeepSet / attention MLPs (A4, A5; Table 1) are plain dense
// contractions Y = X W^T, dX = dY W, dW = dY^T X over the batch rows: they
// belong on the tensor cores.  kind::tf32 reads 19 significant bits; fp32
// parity (1e-5, BASELINE north_star) needs the classic split
//     x = hi + lo,  hi = trunc_tf32(x),  lo = x - hi (exact),
//     x.y ~= hi_x.hi_y + hi_x.lo_y + lo_x.hi_y        (error ~ 2^-21 |x||y|)
// i.e. three tcgen05.mma per K-step into the same fp32 TMEM accumulator.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "kg_common.cuh"
#include "kg_launch.h"

namespace kg {

constexpr int GBM = 128;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)));
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(su32(bar)), "r"(parity));
}

// out[c][r] = in[r][c]: in [R][C] (ld_in), out [C][R] (ld_out); 32 x 32 tiles through shared memory.
__global__ void transpose_kernel(const float *__restrict__ in, int R, int Cc, int ld_in, float *__restrict__ out,
                                 int ld_out) {
  KG_GRID_DEP_WAIT();
  __shared__ float t[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int r = r0 + y, c = c0 + threadIdx.x;
    t[y][threadIdx.x] = (r < R && c < Cc) ? in[(int64_t)r * ld_in + c] : 0.f;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int c = c0 + y, r = r0 + threadIdx.x;
    if (c < Cc && r < R) out[(int64_t)c * ld_out + r] = t[threadIdx.x][y];
  }
}
void launch_transpose(const float *in, int R, int Cc, int ld_in, float *out, int ld_out, cudaStream_t st) {
  if (R <= 0 || Cc <= 0) return;
  dim3 grid((Cc + 31) / 32, (R + 31) / 32), block(32, 8);
  { transpose_kernel<<<grid, block, 0, st>>>(in, R, Cc, ld_in, out, ld_out); ++g_launches; }
}

// C = beta C + alpha sum_z P[z] (+ bias) (ReLU) (masked): the fixed-order combine of the split-K
// partials, 4 consecutive columns per thread (N % 4 == 0 and ldc % 4 == 0: float4 path).
__global__ void gemm_reduce_kernel(const float *__restrict__ P, int splits, int M, int N, float *C, int ldc,
                                   const float *bias, int relu, float beta, float alpha, const float *mask) {
  KG_GRID_DEP_WAIT();
  const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4;
  if (e >= (int64_t)M * N) return;
  const int row = (int)(e / N), n = (int)(e - (int64_t)row * N);
  const int64_t MN = (int64_t)M * N;
  const int64_t co = (int64_t)row * ldc + n;
  if (!(N & 3) && !(ldc & 3)) {
    float4 v = __ldcs(reinterpret_cast<const float4 *>(P + e));
    for (int z = 1; z < splits; ++z) {
      const float4 q = __ldcs(reinterpret_cast<const float4 *>(P + z * MN + e));
      v.x += q.x; v.y += q.y; v.z += q.z; v.w += q.w;
    }
    v.x *= alpha; v.y *= alpha; v.z *= alpha; v.w *= alpha;
    if (bias) { v.x += bias[n]; v.y += bias[n + 1]; v.z += bias[n + 2]; v.w += bias[n + 3]; }
    if (relu) { v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f); }
    float4 *c = reinterpret_cast<float4 *>(C + co);
    if (beta != 0.f) {
      const float4 o = *c;
      v.x += beta * o.x; v.y += beta * o.y; v.z += beta * o.z; v.w += beta * o.w;
    }
    if (mask) {
      const float4 y = *reinterpret_cast<const float4 *>(mask + co);
      if (!(y.x > 0.f)) v.x = 0.f;
      if (!(y.y > 0.f)) v.y = 0.f;
      if (!(y.z > 0.f)) v.z = 0.f;
      if (!(y.w > 0.f)) v.w = 0.f;
    }
    *c = v;
    return;
  }
  for (int j = 0; j < 4 && e + j < MN; ++j) {   // generic: 4 consecutive flat elements
    const int64_t f = e + j;
    const int r = (int)(f / N), c = (int)(f - (int64_t)r * N);
    float v = 0.f;
    for (int z = 0; z < splits; ++z) v += P[z * MN + f];
    v *= alpha;
    if (bias) v += bias[c];
    if (relu) v = fmaxf(v, 0.f);
    float *o = C + (int64_t)r * ldc + c;
    if (beta != 0.f) v += beta * *o;
    if (mask && !(mask[(int64_t)r * ldc + c] > 0.f)) v = 0.f;
    *o = v;
  }
}


// ================================================================ v2: TMA + warp specialisation
// Tile 128 (M) x BN (N) x KB (K; KB = 16, or 32 for K-major B at 64- to 160-wide tiles), 10 warps
// with fixed roles:
//   warp 0      TMA producer: cp.async.bulk.tensor of the raw fp32 A / B tiles into stage s
//               (zero fill out of bounds), completion on full[s];
//   warp 1      TMEM allocator + MMA issuer: per k-block KB / 8 K-steps x 3 tcgen05.mma
//               (hi.hi, hi.lo, lo.hi), one commit per group of k-blocks;
//   warps 2-9   split + drain + epilogue (two teams on alternate k-blocks): lo = x - trunc_tf32(x)
//               of the landed A tile into tensor memory (kind::tf32 reads
//               the raw fp32 words of a K-major tile as hi = trunc_tf32(x)), then tcgen05.ld of
//               the accumulator quarter their warp may access (lanes 32 (w % 4) ..) -> per-warp
//               staging tile -> bias / ReLU / beta C -> coalesced row stores.
// kind::tf32 reads K-major operands only (the idesc transpose bits give zeros, measured), so
// an operand stored MN-major (A [K][M], B [K][N], e.g. both operands of dW = dY^T X) is
// brought in as raw 32 x 16 boxes and the split warps transpose it while splitting, writing
// hi and lo K-major tiles; no global transpose pass.
// K-major smem tiles: rows of KB fp32 (64 B, SWIZZLE_64B, 8-row groups 512 B apart; or 128 B,
// SWIZZLE_128B, 1024 B apart).
#ifndef KG_G2CW
#define KG_G2CW 8
#endif
constexpr int G2CW = KG_G2CW;                          // split / epilogue warps
constexpr int G2T = 64 + 32 * G2CW, G2K = 16;
#ifndef KG_GEMM_KB32
#define KG_GEMM_KB32 1
#endif
// ATM (the fp32-accurate modes): A's hi / lo tiles go to tensor memory, so a stage holds
// A raw, B raw, [B hi if BMN], B lo; otherwise (LOWP) A raw, B raw, [A hi], [B hi], A lo, B lo.
// S stages (even) in G = S / 2 groups of k-blocks: the MMA warp commits once per group
// (a tcgen05.commit drains the tensor pipe: ~200 cycles, tools/mma_probe.cu), and the
// producer refills a group's stages when the group two back has completed.
// OCC = 2: a narrow-tile form with two resident CTAs per SM (half the TMEM columns -- 256 -- and
// under half the shared memory each), so the small d x d contractions of concurrent DAG branches
// (Q2B center / offset, weight gradients) share the SMs instead of queueing behind each other
// KB: k-block depth, 16 (SWIZZLE_64B rows of 64 B) or 32 (SWIZZLE_128B rows of 128 B: half the
// TMA row requests, handshakes and commits per MMA; K-major operands only)
template <int BN, bool AMN, bool BMN, bool ATM = true, bool DRAIN = true, int OCC = 1, int KB = 16> struct G2Cfg {
  static constexpr int kA = GBM * KB * 4, kB = BN * KB * 4;           // bytes of one tile
  static constexpr int kStage = ATM ? kA + kB + (BMN ? kB : 0) + kB : 2 * (kA + kB) + (AMN ? kA : 0) + (BMN ? kB : 0);
  // stages: shared memory (224 KB budget), at most 8, and (ATM) 32 TMEM columns each after
  // the accumulator(s)
  static constexpr int kTmemCols = OCC == 2 ? 256 : 512;
  // SACC: one drained accumulator instead of two (160-wide, 32-deep: two 160-column accumulators
  // would leave TMEM for only three 64-column A stages); the MMA of group g + 1 then waits for the
  // drain of group g
  static constexpr bool kSacc = DRAIN && KB == 32 && BN > 128;
  static constexpr int kTmemFit = ATM ? (kTmemCols - (DRAIN && !kSacc ? 2 * BN : BN)) / (2 * KB) : 8;   // A hi + lo per stage
  static constexpr int kSmemFit = ((OCC == 2 ? 108 : 224) * 1024) / kStage;
  static constexpr int kFit = kSmemFit < 8 ? (kSmemFit < kTmemFit ? kSmemFit : kTmemFit) : (8 < kTmemFit ? 8 : kTmemFit);
  static constexpr int kStages = kFit >= 2 ? (kFit / 2) * 2 : 2;
  static constexpr int kGroup = kStages / 2;
  // shared-memory stages (TMA destinations) beyond the TMEM A stages (drained fp32 mode): the
  // producer refills a stage once the group holding its previous k-block has completed, so
  // kSmemStages - kStages extra stages let the loads run that many k-blocks further ahead of the
  // split (tools/gemm_trace.py: ~1,000 cycles from TMA issue to landed, against ~750 cycles per
  // k-block of MMA work at 128 x 160)
  static constexpr int kSmemStages0 = kSmemFit < kStages + kGroup ? kSmemFit : kStages + kGroup;
#ifndef KG_GEMM_SMEM_STAGES_DECOUPLED
#define KG_GEMM_SMEM_STAGES_DECOUPLED 1
#endif
  static constexpr int kSmemStages =
      (KG_GEMM_SMEM_STAGES_DECOUPLED && ATM && DRAIN && kSmemStages0 > kStages) ? kSmemStages0 : kStages;
  static constexpr int kSmem = kSmemStages * kStage + 1024;
  static constexpr int oAhi = kA + kB, oBhi = ATM ? kA + kB : oAhi + (AMN ? kA : 0);
  static constexpr int oAlo = oBhi + (BMN ? kB : 0), oBlo = ATM ? oAlo : oAlo + kA;
  static constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                     ((uint32_t)(GBM >> 4) << 24);
};
template <int KB = 16>
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t saddr, int kk) {
  uint64_t d = (uint64_t)(((saddr + kk * 32) >> 4) & 0x3FFF);   // K-step = 32 B inside the KB * 4 B row
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * KB * 4) >> 4) << 32;                     // 8-row groups 512 / 1024 B apart
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(KB == 32 ? 2 : 4) << 61;                      // SWIZZLE_128B / SWIZZLE_64B
  return d;
}
// byte offset of 16-byte chunk q (k = 4q .. 4q+3) of row r in a K-major SWIZZLE_64B tile
template <int KB = 16>
__device__ __forceinline__ uint32_t sw_off(int r, int q) {
  if (KB == 32) return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((q ^ (r & 7)) << 4));   // SWIZZLE_128B
  return (uint32_t)((r >> 3) * 512 + (r & 7) * 64 + ((q ^ ((r >> 1) & 3)) << 4));
}
__device__ __forceinline__ uint32_t sw64_off(int r, int q) {
  return (uint32_t)((r >> 3) * 512 + (r & 7) * 64 + ((q ^ ((r >> 1) & 3)) << 4));
}

// Named (hardware) barriers between the split warps and the MMA warp.  The MMA warp must
// not wait on an mbarrier (or poll shared memory) while its MMAs are in flight: that stalls
// the tensor pipe ~200 cycles per wait (tools/mma_probe.cu, "pattern" rows: 592 vs 385
// cycles per 16-deep k-block); a bar.sync does not (385).
// k-block barriers: one split team (4 warps) + the MMA warp; drain barriers: both teams + MMA warp
constexpr int kTeamBar = 32 * (G2CW / 2) + 32, kAllBar = 32 * G2CW + 32;
template <int N> __device__ __forceinline__ void nbar_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(N) : "memory");
}
template <int N> __device__ __forceinline__ void nbar_arrive(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(N) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}\n" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void mbar_init(uint64_t *b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap *tm, uint64_t *bar, void *dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(su32(bar)), "r"(x), "r"(y)
      : "memory");
}
// A operand from tensor memory ([a_tmem]: 128 lanes = rows, one 32-bit column per k), B from
// shared memory: the MMA reads only B through the shared-memory port
template <uint32_t IDESC>
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem, uint32_t a_tmem, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %3, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n}\n" ::"r"(tmem),
      "r"(a_tmem), "l"(b), "r"(acc), "r"(IDESC));
}
template <uint32_t IDESC>
__device__ __forceinline__ void mma_tf32_i(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}
// one operand tile (rows r0 .. r0 + R, k0 .. k0 + 16) into dst: K-major one SWIZZLE_64B box;
// MN-major R / 32 unswizzled boxes of 32 (rows) x 16 (k), 2048 B each ([k][32 rows])
template <bool MN, int R, int KB = 16>
__device__ __forceinline__ void load_op(const CUtensorMap *tm, uint64_t *bar, uint8_t *dst, int r0, int k0) {
  if (MN) {
#pragma unroll
    for (int c = 0; c < R / 32; ++c) tma_load_2d(tm, bar, dst + c * (32 * KB * 4), r0 + 32 * c, k0);
  } else {
    tma_load_2d(tm, bar, dst, k0, r0);
  }
}
// lo = x - trunc_tf32(x), rounded to the nearest tf32 (cvt.rna): the MMA then reads lo exactly
// instead of truncating it again (a one-sided error of ~2^-22 |x| per operand that accumulates
// linearly over K; tools/gemm_precision.py)
__device__ __forceinline__ float rna_tf32(float x) {
#ifdef KG_TF32_LO_TRUNC
  return x;
#else
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
#endif
}
__device__ __forceinline__ float4 tf32_lo(float4 v) {
  float4 l;
  l.x = rna_tf32(v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u));
  l.y = rna_tf32(v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u));
  l.z = rna_tf32(v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u));
  l.w = rna_tf32(v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
  return l;
}
__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float4 bf16r4(float4 v) { return make_float4(bf16r(v.x), bf16r(v.y), bf16r(v.z), bf16r(v.w)); }
// split one landed operand tile of R rows (32 G2CW threads, ct = 0 ..).  LOWP (the bf16 score
// mode): the operand is rounded to bf16 (RNE) instead -- K-major in place, MN-major into hi --
// and the one MMA per K-step multiplies bf16-exact values (exact products, fp32 accumulation)
template <bool MN, int R, bool LOWP = false, int KB = 16>
__device__ __forceinline__ void split_op(uint8_t *raw, uint8_t *hi, uint8_t *lo, int ct, int nthr) {
  constexpr int Q = KB / 4;   // 16-byte chunks per row
  if (LOWP && !MN) {
#pragma unroll 4
    for (int c = ct; c < R * Q; c += nthr) {
      float4 *p = reinterpret_cast<float4 *>(raw + c * 16);
      *p = bf16r4(*p);
    }
    return;
  }
  if (!MN) {   // K-major: same (swizzled) offsets, lo only
#pragma unroll 4
    for (int c = ct; c < R * Q; c += nthr) {
      const float4 v = *reinterpret_cast<const float4 *>(raw + c * 16);
      *reinterpret_cast<float4 *>(lo + c * 16) = tf32_lo(v);
    }
  } else {     // MN-major raw [R/32][16 k][32 rows] -> K-major SW64 hi and lo, 4 k per chunk
#pragma unroll 4
    for (int c = ct; c < R * Q; c += nthr) {
      const int r = c % R, q = c / R;
      const float *src = reinterpret_cast<const float *>(raw + (r >> 5) * (32 * KB * 4)) + (r & 31);
      float4 v;
      v.x = src[(4 * q + 0) * 32];
      v.y = src[(4 * q + 1) * 32];
      v.z = src[(4 * q + 2) * 32];
      v.w = src[(4 * q + 3) * 32];
      const uint32_t o = sw_off<KB>(r, q);
      if (LOWP) {
        *reinterpret_cast<float4 *>(hi + o) = bf16r4(v);
        continue;
      }
      const float4 l = tf32_lo(v);
      *reinterpret_cast<float4 *>(hi + o) = v;
      *reinterpret_cast<float4 *>(lo + o) = l;
    }
  }
}

// DRAIN (fp32-accurate mode, reading A24): the tensor cores accumulate only one group of G
// k-blocks (K = 16 G: 6 G MMAs) into one of two TMEM accumulators; the split warps then drain
// that group into fp32 registers (round-to-nearest adds) while the MMA warp fills the other
// one.  The error of the TMEM accumulation grows with the number of MMAs chained into one
// accumulator (tools/gemm_precision.py: 15-25x SGEMM's at K = 800-1600); groups of <= 24 MMAs
// bring it to SGEMM's.
#ifdef KG_GEMM_TRACE
// tools/gemm_trace.py: globaltimer stamps of CTA (0, 0, 0), per k-block: [0] producer issued the
// loads, [1] split warp 2 saw full, [2] split warp 2 arrived conv, [3] MMA warp saw conv,
// [4] MMA issued (before commit); [5] per chunk: drain begin / end
__device__ unsigned long long g_gemm_trace[8][512];
__device__ __forceinline__ unsigned long long gt_now() { return (unsigned long long)clock64(); }   // SM cycles
#define GT(k, i) do { if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (i) < 512) g_gemm_trace[k][i] = gt_now(); } while (0)
}  // namespace kg
extern "C" int gemm_trace_get(unsigned long long *out) {
  return (int)cudaMemcpyFromSymbol(out, kg::g_gemm_trace, sizeof(unsigned long long) * 8 * 512);
}
namespace kg {
#else
#define GT(k, i) do {} while (0)
#endif
template <int BN, bool AMN, bool BMN, bool DRAIN, bool LOWP = false, int OCC = 1, int KB = 16>
__global__ void __launch_bounds__(G2T, OCC)
    gemm_tf32x3_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const __grid_constant__ CUtensorMap tmBl, GemmArgs g) {
  KG_GRID_DEP_WAIT();
  using Cfg = G2Cfg<BN, AMN, BMN, !LOWP, DRAIN, OCC, KB>;
  static_assert(KB == 16 || (KB == 32 && !BMN && !LOWP), "32-deep k-blocks: K-major B (A K- or MN-major)");
  constexpr int S = Cfg::kStages, G = Cfg::kGroup, SM = Cfg::kSmemStages;
  static_assert(SM >= S && SM <= S + G, "shared-memory stages");
  // TMEM columns: a power of 2 >= 32 holding one (or, drained, two) BN-column accumulators
  constexpr bool SACC = Cfg::kSacc;
  constexpr int kNeed = DRAIN && !SACC ? 2 * BN : BN;
  // ATM (every fp32-accurate mode): the A operand's hi / lo tiles of each stage live in tensor
  // memory (32 columns per stage after the accumulators), written by the split warps with
  // tcgen05.st; the MMAs then read only B from shared memory.  Shared-memory traffic per
  // k-block (128 x 128): TMA 16 KB + split 24 KB + MMA 24 KB = 64 KB instead of 96 KB (the
  // split stage was bound by the 128 B/clk shared-memory port: tools/gemm_trace.py).
  constexpr bool ATM = !LOWP;
  constexpr int kACol = kNeed;
  constexpr int kCols = ATM ? Cfg::kTmemCols : kNeed <= 32 ? 32 : kNeed <= 64 ? 64 : kNeed <= 128 ? 128 : kNeed <= 256 ? 256 : 512;
  static_assert(!ATM || (kACol % 32 == 0 && kACol + 2 * KB * S <= kCols && G2CW == 8), "TMEM A stages");
  static_assert(S == 2 * G && G >= 2 && S + 3 <= 16, "two groups of stages in flight, k-blocks of both split teams in "
                "each; named barrier ids 1 .. S + 2");
  // 32-column chunks of the tile; the NG = G2CW / 4 warps of a TMEM lane quarter take the
  // chunks round-robin (chunk = grp + NG i)
  constexpr int NG = G2CW / 4, kChunks = BN / 32, kCI = (kChunks + NG - 1) / NG;
  static_assert(BN % 32 == 0 && kNeed <= 512 && G2CW % 4 == 0, "tile width / split warps");
  static_assert(!DRAIN || kCI <= 3, "the drained accumulator is held in registers");
  extern __shared__ uint8_t gsm_raw[];
  // 1024-byte aligned (SWIZZLE tiles), derived from the shared-memory symbol itself so the
  // compiler keeps the address space: LDS / STS in the split and the epilogue, not generic LD / ST
  uint8_t *sm = gsm_raw + ((1024u - (su32(gsm_raw) & 1023u)) & 1023u);
  // full[s]: TMA landed (mbarrier); split of k-block kb done: named barrier 1 + kb % S; gdone[g &
  // 1]: the MMAs of group g completed (mbarrier, one commit per group: frees its stages for
  // the producer and hands its accumulator to the drain); drain of group g done: named
  // barrier 1 + S + (g & 1).  (Barrier ids <= 1 + 8 + 1 < 16; 0 is __syncthreads.)
  // gdone[g & 3]: four group barriers -- the producer waits for a group up to three behind the
  // one it loads for (SM <= S + G), so the bucket of a group cannot have moved on a full phase
  __shared__ __align__(8) uint64_t full_bar[SM];
  __shared__ __align__(8) uint64_t done_bar, gdone[4];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * BN;
  const bool bpre = !BMN && !LOWP && g.B_lo != nullptr;   // B's lo plane comes from global memory
  const int nkb_all = (g.K + KB - 1) / KB;
  const int kb0 = blockIdx.z * g.kbs, nkb = min(nkb_all, kb0 + g.kbs) - kb0;   // split-K range

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    if (bpre) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmBl)) : "memory");
    for (int s = 0; s < SM; ++s) mbar_init(&full_bar[s], 1);
    mbar_init(&done_bar, 1);
    for (int b = 0; b < 4; ++b) mbar_init(&gdone[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % SM;
        if (kb >= SM) {   // the stage's previous k-block kb - SM: its group has completed
          const int gw = (kb - SM) / G;
          mbar_wait(&gdone[gw & 3], (gw >> 2) & 1);
        }
        uint8_t *st = sm + s * Cfg::kStage;
        mbar_expect_tx(&full_bar[s], Cfg::kA + Cfg::kB + (bpre ? Cfg::kB : 0));
        const int k0 = (kb0 + kb) * KB;
        load_op<AMN, GBM, KB>(&tmA, &full_bar[s], st, m0, k0);
        load_op<BMN, BN, KB>(&tmB, &full_bar[s], st + Cfg::kA, n0, k0);
        if (bpre) load_op<false, BN, KB>(&tmBl, &full_bar[s], st + Cfg::oBlo, n0, k0);   // B's lo plane
        GT(0, kb);
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the loop (named barriers are warp-aligned); one elected lane issues
    const bool leader = elect_one();
    {
      const int ngr = (nkb + G - 1) / G;
      for (int gi = 0; gi < ngr; ++gi) {
        if (DRAIN && !SACC && gi >= 2) nbar_sync<kAllBar>(1 + S + (gi & 1));      // group gi-2 drained
        if (DRAIN && SACC && gi >= 1) nbar_sync<kAllBar>(1 + S + ((gi - 1) & 1));  // group gi-1 drained
        GT(7, 256 + gi);
        const uint32_t tm = DRAIN && !SACC ? tmem + (uint32_t)((gi & 1) * BN) : tmem;
        const int kbe = min(nkb, gi * G + G);
        for (int kb = gi * G; kb < kbe; ++kb) {
          const int s = kb % S, sms = kb % SM;   // TMEM A stage, shared-memory stage
          const bool first = DRAIN ? (kb == gi * G) : (kb == 0);
          nbar_sync<kTeamBar>(1 + s);                          // k-block kb split (team kb & 1)
          GT(3, kb);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (leader) {
            const uint32_t st = su32(sm + sms * Cfg::kStage);
            const uint32_t ah = AMN ? st + Cfg::oAhi : st, bh = BMN ? st + Cfg::oBhi : st + Cfg::kA;
            const uint32_t al = st + Cfg::oAlo, bl = st + Cfg::oBlo;
            const uint32_t ta = tmem + (uint32_t)(kACol + 2 * KB * s);   // this stage's A: hi at +0, lo at +KB
  #pragma unroll
            for (int kk = 0; kk < KB / 8; ++kk) {   // K = 8 tf32 per MMA
              const uint64_t dbh = kmajor_desc<KB>(bh, kk), dbl = kmajor_desc<KB>(bl, kk);
              if (ATM) {
                mma_tf32_ts<Cfg::kIdesc>(tm, ta + 8 * kk, dbl, !(first && kk == 0));        // hi.lo
                mma_tf32_ts<Cfg::kIdesc>(tm, ta + KB + 8 * kk, dbh, 1);                     // lo.hi
                mma_tf32_ts<Cfg::kIdesc>(tm, ta + 8 * kk, dbh, 1);                          // hi.hi
                continue;
              }
              const uint64_t dah = kmajor_desc<KB>(ah, kk), dal = kmajor_desc<KB>(al, kk);
              if (LOWP) {   // bf16-rounded operands: one MMA
                mma_tf32_i<Cfg::kIdesc>(tm, dah, dbh, !(first && kk == 0));
                continue;
              }
              // small terms first: hi.lo, lo.hi, then hi.hi
              mma_tf32_i<Cfg::kIdesc>(tm, dah, dbl, !(first && kk == 0));
              mma_tf32_i<Cfg::kIdesc>(tm, dal, dbh, 1);
              mma_tf32_i<Cfg::kIdesc>(tm, dah, dbh, 1);
            }
            GT(4, kb);
          }
          __syncwarp();
        }
        if (leader) mma_commit(&gdone[gi & 3]);
        __syncwarp();
        GT(6, 256 + gi);
      }
      if (leader) mma_commit(&done_bar);
    }
  } else {
    // ---- split (and transpose the MN-major operands)
    const int ct = tid - 64;
    const int q = warp & 3, half = (warp - 2) >> 2;   // lane quarter, chunk group (0 .. NG-1)
    // DRAIN: this thread's share of the accumulator tile -- row 32 q + lane, columns
    // 32 half + 64 i + j (i < 2, j < 32): the same columns its epilogue writes
    float acc[DRAIN ? kCI : 1][32];
    if (DRAIN) {
#pragma unroll
      for (int i = 0; i < (DRAIN ? kCI : 1); ++i)
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[i][j] = 0.f;
    }
    auto drain = [&](int c) {
      if (ct == 0) GT(6, c);
      mbar_wait(&gdone[c & 3], (c >> 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int i = 0; i < (DRAIN ? kCI : 1); ++i) {
        if (half + NG * i >= kChunks) continue;
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
            "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((SACC ? 0 : (c & 1) * BN) + 32 * (half + NG * i))));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[i][j] += __uint_as_float(r[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      nbar_arrive<kAllBar>(1 + S + (c & 1));
      if (ct == 0) GT(7, c);
    };
    // two teams of four warps (one per TMEM lane quarter: warps 2-5 and 6-9) split alternate
    // k-blocks (S is even: a stage always belongs to the same team), so one k-block's split
    // latency chain (loads, tcgen05.st, fences) overlaps the other's
    const int team = half, tct = ct - 128 * team;
    const int ngr = (nkb + G - 1) / G;
    int dn = 0;   // next group this thread drains (DRAIN)
    for (int kb = team; kb < nkb; kb += 2) {
      // TMEM stage s was last used by k-block kb - S (group g - 2): drained by this thread
      // before this iteration (DRAIN), so its MMAs are complete
      const int s = kb % S, sms = kb % SM;
      mbar_wait(&full_bar[sms], (kb / SM) & 1);
      if (ct == 0) GT(1, kb);
      uint8_t *st = sm + sms * Cfg::kStage;
      if (ATM) {
        // A: row r = 32 q + lane of the tile (this warp's TMEM lane quarter), all KB k in halves
        // of 16: hi = trunc_tf32(x), lo = rna_tf32(x - hi) -> tcgen05.st of 16 columns each
        const int r = 32 * q + lane;
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(kACol + 2 * KB * s);
#pragma unroll
        for (int h16 = 0; h16 < KB / 16; ++h16) {
          float v[16];
          if (!AMN) {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const float4 x = *reinterpret_cast<const float4 *>(st + sw_off<KB>(r, 4 * h16 + jj));
              v[4 * jj + 0] = x.x; v[4 * jj + 1] = x.y; v[4 * jj + 2] = x.z; v[4 * jj + 3] = x.w;
            }
          } else {   // raw MN-major boxes [GBM / 32][KB k][32 rows]
            const float *src = reinterpret_cast<const float *>(st + (r >> 5) * (32 * KB * 4)) + (r & 31);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = src[(16 * h16 + i) * 32];
          }
          uint32_t hb[16], lb[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint32_t hh = __float_as_uint(v[i]) & 0xFFFFE000u;
            hb[i] = hh;
            lb[i] = __float_as_uint(rna_tf32(v[i] - __uint_as_float(hh)));
          }
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta + 16 * h16),
              "r"(hb[0]), "r"(hb[1]), "r"(hb[2]), "r"(hb[3]), "r"(hb[4]), "r"(hb[5]), "r"(hb[6]), "r"(hb[7]), "r"(hb[8]),
              "r"(hb[9]), "r"(hb[10]), "r"(hb[11]), "r"(hb[12]), "r"(hb[13]), "r"(hb[14]), "r"(hb[15])
              : "memory");
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta + KB + 16 * h16),
              "r"(lb[0]), "r"(lb[1]), "r"(lb[2]), "r"(lb[3]), "r"(lb[4]), "r"(lb[5]), "r"(lb[6]), "r"(lb[7]), "r"(lb[8]),
              "r"(lb[9]), "r"(lb[10]), "r"(lb[11]), "r"(lb[12]), "r"(lb[13]), "r"(lb[14]), "r"(lb[15])
              : "memory");
        }
      } else {
        split_op<AMN, GBM, LOWP, KB>(st, st + Cfg::oAhi, st + Cfg::oAlo, tct, 128);
      }
      if (!bpre) split_op<BMN, BN, LOWP, KB>(st + Cfg::kA, st + Cfg::oBhi, st + Cfg::oBlo, tct, 128);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic stores -> tensor-core reads
      if (ATM) {
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      }
      nbar_arrive<kTeamBar>(1 + s);
      if (ct == 0) GT(2, kb);
      if (ct == 32 * G2CW - 32) GT(5, kb);   // the last split warp
      // DRAIN: once this team has split its part of group c, group c - 1 is drained
      if (DRAIN) {
        const int gnext = kb + 2 < nkb ? (kb + 2) / G : ngr;
        while (dn < gnext - 1) drain(dn++);
      }
    }
    if (DRAIN) while (dn < ngr) drain(dn++);
    // ---- epilogue: TMEM -> registers (thread = accumulator row) -> per-warp 32 x 33 staging
    // tile in the (now idle) pipeline smem -> coalesced row stores (lane = column)
    mbar_wait(&done_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // warp w may read TMEM lanes 32 (w % 4) ..; the G2CW / 4 warps of a quarter take turns on
    // its 32-column chunks
    float *T = reinterpret_cast<float *>(sm) + (warp - 2) * 32 * 33;
#pragma unroll
    for (int ci = 0; ci < kCI; ++ci) {
      const int c0 = 32 * (half + NG * ci);
      if (half + NG * ci >= kChunks || n0 + c0 >= g.N) break;
      uint32_t r[32];
      if (DRAIN) {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(acc[DRAIN ? ci : 0][j]);
      } else {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
          "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) T[lane * 33 + j] = __uint_as_float(r[j]);
      __syncwarp();
      const int n = n0 + c0 + lane;
      if (n < g.N) {
        const float bn = g.bias ? g.bias[n] : 0.f;
        const int rlim = min(32, g.M - (m0 + q * 32));
#pragma unroll 4
        for (int i = 0; i < rlim; ++i) {
          const int row = m0 + q * 32 + i;
          float v = T[i * 33 + lane];
          if (g.P) {   // split-K: raw partial sums, combined by gemm_reduce_kernel
            g.P[((int64_t)blockIdx.z * g.M + row) * g.N + n] = v;
          } else {
            float *c = g.C + (int64_t)row * g.ldc + n;
            v = fmaf(g.alpha, v, bn);
            if (g.relu) v = fmaxf(v, 0.f);
            if (g.beta != 0.f) v += g.beta * *c;
            *c = v;
          }
        }
      }
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
}

// Pre-split weights (B operands): for W [R][C], lo = rna_tf32(W - trunc_tf32(W)) in W's layout,
// and the transposed pair WT = W^T [C][R], WT_lo = lo^T (the backward's dX = dY W reads W as a
// K-major [in][out] operand).  32 x 32 tiles through shared memory; one launch for all jobs.
__global__ void wsplit_kernel(WSplitJobs J, int part) {   // part 0: lo; 1: t, tlo
  KG_GRID_DEP_WAIT();
  const WSplitJob &jb = J.j[blockIdx.z];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  if (r0 >= jb.R || c0 >= jb.C) return;
  __shared__ float th[32][33], tl[32][33];
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int r = r0 + y, c = c0 + threadIdx.x;
    if (r < jb.R && c < jb.C) {
      const float x = jb.w[(int64_t)r * jb.C + c];
      const float l = rna_tf32(x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u));
      if (part == 0) jb.lo[(int64_t)r * jb.C + c] = l;
      th[y][threadIdx.x] = x;
      tl[y][threadIdx.x] = l;
    }
  }
  if (part == 0) return;
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int c = c0 + y, r = r0 + threadIdx.x;
    if (c < jb.C && r < jb.R) {
      jb.t[(int64_t)c * jb.R + r] = th[threadIdx.x][y];
      jb.tlo[(int64_t)c * jb.R + r] = tl[threadIdx.x][y];
    }
  }
}
void launch_wsplit(const WSplitJobs &J, int part, cudaStream_t st) {
  if (J.n <= 0) return;
  int mr = 0, mc = 0;
  for (int i = 0; i < J.n; ++i) { mr = std::max(mr, J.j[i].R); mc = std::max(mc, J.j[i].C); }
  dim3 grid((mc + 31) / 32, (mr + 31) / 32, J.n), block(32, 8);
  { wsplit_kernel<<<grid, block, 0, st>>>(J, part); ++g_launches; }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  // resolved once; a function-local static is initialised thread-safely (with a plain
  // "tried" flag a second host thread could see the flag before the pointer and fall back
  // to cuBLAS for its first GEMM -- different rounding than the other ranks)
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  return fn;
}
// fp32 operand with `rows` GEMM rows (M or N) and K columns, stored with leading dimension ld:
//   K-major  [rows][ld]: dims {K, rows}, box {16, box_rows}, SWIZZLE_64B
//   MN-major [K][ld]:    dims {rows, K}, box {32, 16},       no swizzle (one box per 32 rows)
bool make_tmap(CUtensorMap *tm, const float *base, int rows, int K, int ld, int box_rows, bool mn, int kb = 16) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)(mn ? rows : K), (cuuint64_t)(mn ? K : rows)};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {mn ? 32u : (cuuint32_t)kb, mn ? (cuuint32_t)kb : (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             mn ? CU_TENSOR_MAP_SWIZZLE_NONE : (kb == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B),
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// returns the number of K splits (0: not launched); raw: the kernel writes the raw partial
// products [splits][M][N] into `part` (even unsplit) and the caller's kernel combines them
template <int BN, bool AMN, bool BMN, bool DRAIN, bool LOWP = false, int OCC = 1, int KB = 16>
int launch_v2(const GemmArgs &g0, float *part, int64_t part_cap, cudaStream_t st, bool raw = false) {
  using Cfg = G2Cfg<BN, AMN, BMN, !LOWP, DRAIN, OCC, KB>;
  CUtensorMap ta, tb, tbl;
  if (!make_tmap(&ta, g0.A, g0.M, g0.K, g0.lda, GBM, AMN, KB) || !make_tmap(&tb, g0.B, g0.N, g0.K, g0.ldb, BN, BMN, KB))
    return 0;
  if (g0.B_lo && !BMN && !LOWP) {
    if (!make_tmap(&tbl, g0.B_lo, g0.N, g0.K, g0.ldb, BN, false, KB)) return 0;
  } else {
    tbl = tb;
  }
  static const bool configured =   // thread-safe one-time attribute (concurrent host threads)
      cudaFuncSetAttribute(gemm_tf32x3_tma_kernel<BN, AMN, BMN, DRAIN, LOWP, OCC, KB>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem) == cudaSuccess;
  (void)configured;
  GemmArgs g = g0;
  const int tiles = ((g.N + BN - 1) / BN) * ((g.M + GBM - 1) / GBM);
  const int nkb = (g.K + KB - 1) / KB;
  // split K to fill the SMs while every split keeps >= 128 of K (8 16-deep k-blocks; measured
  // best of 8 / 16 / none)
  int splits = std::max(1, std::min(148 * OCC / std::max(tiles, 1), nkb / (128 / KB)));
  if (g0.force & 1) splits = 1;
  while (splits > 1 && (!part || (int64_t)splits * g.M * g.N > part_cap)) --splits;
  g.kbs = (nkb + splits - 1) / splits;
  splits = (nkb + g.kbs - 1) / g.kbs;
  g.P = splits > 1 ? part : nullptr;
  if (raw) {
    if (!part || (int64_t)splits * g.M * g.N > part_cap) return 0;
    g.P = part;
  }
  dim3 grid((g.N + BN - 1) / BN, (g.M + GBM - 1) / GBM, splits);
  { gemm_tf32x3_tma_kernel<BN, AMN, BMN, DRAIN, LOWP, OCC, KB><<<grid, G2T, Cfg::kSmem, st>>>(ta, tb, tbl, g); ++g_launches; }
  if (raw) return splits;
  if (splits > 1) {
    const int64_t n4 = ((int64_t)g.M * g.N + 3) / 4;
    { gemm_reduce_kernel<<<(int)((n4 + 255) / 256), 256, 0, st>>>(part, splits, g.M, g.N, g.C, g.ldc, g.bias, g.relu,
                                                                 g.beta, g.alpha, g.mask); ++g_launches; }
  } else if (g.mask) {
    // a separate pass: a dependent global load per element in the epilogue's row loop was
    // latency-bound (C5-betae 2u DAG backward 0.10 -> 0.15 ms)
    launch_relu_mask(g.C, g.mask, g.M, g.N, st);
  }
  return splits;
}
// 32-deep k-blocks (SWIZZLE_128B) where both operands are K-major and the TMEM budget keeps two
// groups of >= 2 stages: the drained fp32 mode, one CTA per SM, 64 / 128-wide tiles
template <int BN, bool DRAIN, bool LOWP, int OCC> constexpr bool kUseKB32() {
  return KG_GEMM_KB32 && DRAIN && !LOWP && OCC == 1 && (BN == 64 || BN == 96 || BN == 128 || BN == 160);
}
template <int BN, bool DRAIN, bool LOWP = false, int OCC = 1>
int launch_v2_any(const GemmArgs &g, float *part, int64_t part_cap, cudaStream_t st, bool raw = false) {
  if (g.a_mn) return g.b_mn ? launch_v2<BN, true, true, DRAIN, LOWP, OCC>(g, part, part_cap, st, raw)
                            : launch_v2<BN, true, false, DRAIN, LOWP, OCC, kUseKB32<BN, DRAIN, LOWP, OCC>() ? 32 : 16>(
                                  g, part, part_cap, st, raw);
  if (g.b_mn) return launch_v2<BN, false, true, DRAIN, LOWP, OCC>(g, part, part_cap, st, raw);
  return launch_v2<BN, false, false, DRAIN, LOWP, OCC, kUseKB32<BN, DRAIN, LOWP, OCC>() ? 32 : 16>(g, part, part_cap, st, raw);
}
}  // namespace

bool gemm_tc_accepts(const GemmArgs &g) {
  return g.M > 0 && g.N > 0 && g.K > 0 && !(reinterpret_cast<uintptr_t>(g.A) & 15) &&
         !(reinterpret_cast<uintptr_t>(g.B) & 15) && !(reinterpret_cast<uintptr_t>(g.B_lo) & 15) &&
         !(g.B_lo && g.b_mn) && !(g.lda & 3) && !(g.ldb & 3) && !(g.mask && g.ldc != g.N) &&
         tmap_encoder() != nullptr;
}

// C = beta C + op(A) op(B)^T (+ bias) (ReLU) on the tensor cores.  A is [M][K] (a_mn: [K][M]),
// B is [N][K] (b_mn: [K][N]), 16-byte aligned with ld % 4 == 0 (gemm_tc_accepts).  When the
// output has fewer tiles than SMs, K is split over blockIdx.z (at most one wave of CTAs: 192 KB
// of shared memory per CTA) into `part` (capacity part_cap floats).
static int launch_gemm_sel(const GemmArgs &g, float *part, int64_t part_cap, cudaStream_t st, bool raw) {
  if (!gemm_tc_accepts(g)) return 0;
  const int64_t t256 = (int64_t)((g.N + 255) / 256) * ((g.M + GBM - 1) / GBM);
  const bool wide = g.N > 128 && t256 >= 100;   // enough 128 x 256 tiles to fill the GPU
  if (g.lowp) return launch_v2_any<128, false, true>(g, part, part_cap, st, raw);
  if (g.force) {
    const GemmArgs &f = g;
    const int bn = (g.force >> 1) & 3;
    auto go = [&](auto tag) -> int {
      constexpr int BN = decltype(tag)::value;
      return f.drain ? launch_v2_any<BN, true>(f, part, part_cap, st, raw) : launch_v2_any<BN, false>(f, part, part_cap, st, raw);
    };
    if (g.force & 8) return f.drain ? launch_v2_any<64, true, false, 2>(f, part, part_cap, st, raw) : 0;   // 2 per SM
    if (g.force & 16) return f.drain ? launch_v2_any<96, true>(f, part, part_cap, st, raw) : 0;           // 96 wide
    if (bn == 1) return go(std::integral_constant<int, 64>());
    if (bn == 3) return go(std::integral_constant<int, 160>());
    return go(std::integral_constant<int, 128>());
  }
  // (the two-per-SM narrow form, force bit 3, for every N <= 512 contraction of the step: neutral at
  // C5-q2b / C5-betae -- the concurrent branches' GEMMs did not gain from sharing SMs)
  if (g.drain) {
    // wave quantisation: e.g. 1536 x 1600 is 156 tiles of 128 x 128 (two waves on 148 SMs) but
    // 120 tiles of 128 x 160 (one)
    const int64_t t128 = (int64_t)((g.N + 127) / 128) * ((g.M + GBM - 1) / GBM);
    const int64_t t160 = (int64_t)((g.N + 159) / 160) * ((g.M + GBM - 1) / GBM);
    if (t128 > 148 && t160 <= 148) return launch_v2_any<160, true>(g, part, part_cap, st, raw);
    // under half the SMs with a K too short to split (>= 8 k-blocks per split): 128 x 64
    // tiles, twice the CTAs (e.g. the ComplEx scores S = Q E^T, 1024 x 1024 x 200: 64 -> 128)
    const int nkb = (g.K + G2K - 1) / G2K;
    const int64_t t64 = (int64_t)((g.N + 63) / 64) * ((g.M + GBM - 1) / GBM);
    if (2 * t128 <= 148 && nkb < 16 && t64 <= 148 && t64 > t128) return launch_v2_any<64, true>(g, part, part_cap, st, raw);
    // short K (<= 512, K-major operands: 32-deep k-blocks) with one wave of 128 x 64 tiles: those,
    // unsplit (tools/gemm_variants.py, ncu GEMM + combine: 1024 x 400 x 400 11.3 -> 9.8 us,
    // 512 x 1600 x 400 13.6 -> 10.5 us, 1536 x 400 x 400 12.5 -> 10.4 us)
    // (and K <= 1024 where the 128 x 64 tiles alone fill two thirds of the SMs: 512 x 1600 x 800
    // 17.7 -> 16.0 us)
    if (kUseKB32<64, true, false, 1>() && !g.b_mn && t64 <= 148 && (g.K <= 512 || (g.K <= 1024 && t64 >= 96))) {
      GemmArgs u = g;
      u.force |= 1;   // no split-K
      return launch_v2_any<64, true>(u, part, part_cap, st, raw);
    }
    // weight gradients dW = dY^T X with few 128 x 128 tiles and a long K: 128 x 160 tiles split
    // two ways fill more SMs (1600 x 800 x 1536: 91 tiles -> 130 CTAs, 36.9 -> 33.0 us)
    if (g.a_mn && !g.b_mn && t128 < 100 && 2 * t160 <= 148 && g.K >= 1024)
      return launch_v2_any<160, true>(g, part, part_cap, st, raw);
    // SM coverage: 96-wide tiles when they give a markedly fuller single wave than 128-wide ones
    // (e.g. 512 x 1600 x 1600: 52 tiles x 2 splits = 104 CTAs -> 68 x 2 = 136), K-major B
    if (kUseKB32<96, true, false, 1>() && !g.b_mn) {
      const int nkb32 = (g.K + 31) / 32;
      const int64_t t96 = (int64_t)((g.N + 95) / 96) * ((g.M + GBM - 1) / GBM);
      const int64_t c128 = t128 * std::max<int64_t>(1, std::min<int64_t>(148 / std::max<int64_t>(t128, 1), nkb32 / 4));
      const int64_t c96 = t96 * std::max<int64_t>(1, std::min<int64_t>(148 / std::max<int64_t>(t96, 1), nkb32 / 4));
      if (t96 <= 148 && 20 * c96 > 23 * c128) return launch_v2_any<96, true>(g, part, part_cap, st, raw);
    }
    return launch_v2_any<128, true>(g, part, part_cap, st, raw);
  }
  return wide ? launch_v2_any<256, false>(g, part, part_cap, st, raw) : launch_v2_any<128, false>(g, part, part_cap, st, raw);
}

bool launch_gemm_tc(const GemmArgs &g, float *part, int64_t part_cap, cudaStream_t st) {
  return launch_gemm_sel(g, part, part_cap, st, false) > 0;
}
// The raw partial products only: [splits][M][N] fp32 into part (bias / relu / beta / mask of g are
// not applied); returns the number of splits (0: not launched).  The caller's kernel sums the
// splits in ascending order (the sums of gemm_reduce_kernel) and applies its own epilogue.
int launch_gemm_tc_raw(const GemmArgs &g, float *part, int64_t part_cap, cudaStream_t st) {
  return launch_gemm_sel(g, part, part_cap, st, true);
}

}  // namespace kg
