// k_gemm.cu -- dense contractions of the query DAG on the 5th-generation tensor
// cores (tcgen05, TMEM accumulators), fp32-accurate through a 3xTF32 split.
//
// The BetaE projection MLP (reading A9; Table 1 'MLP') and the d x d
// DeepSet / attention MLPs (A4, A5; Table 1) are plain dense
// contractions Y = X W^T, dX = dY W, dW = dY^T X over the batch rows: they
// belong on the tensor cores.  kind::tf32 reads 19 significant bits; fp32
// parity (1e-5, BASELINE north_star) needs the classic split
//     x = hi + lo,  hi = rna_tf32(x),  lo = x - hi (exact),
//     x.y ~= hi_x.hi_y + hi_x.lo_y + lo_x.hi_y        (error ~ 2^-21 |x||y|)
// i.e. three tcgen05.mma per K-step into the same fp32 TMEM accumulator.
//
// Tile 128 (M) x 128 (N) x 32 (K), one CTA of 4 warps per output tile:
//   * cp.async copies the raw fp32 operand tiles (K-major; transposed
//     operands are transposed by a separate kernel first) straight into their
//     128-byte-swizzled 8-row atoms (the SWIZZLE_128B canonical layout the UMMA
//     smem descriptors read), 3 stages in flight; all threads then split each
//     landed tile in place into hi and a separate lo tile;
//   * one elected thread issues 4 K-steps x 3 MMAs per stage and commits them
//     to the stage's mbarrier, which gates the refill of that stage;
//   * epilogue: tcgen05.ld (32 lanes x 32 columns per warp and load) ->
//     optional bias, ReLU, C += -> global.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "kg_common.cuh"
#include "kg_launch.h"

namespace kg {

constexpr int GBM = 128, GBN = 128, GBK = 32, GSTAGES = 3, GTHREADS = 256;
constexpr int GCH = GBM * GBK / 4 / GTHREADS;   // 16-byte chunks per thread per tile
constexpr int GTILE = GBM * GBK * 4;          // 16 KB: one operand tile (hi or lo)
constexpr int GSTAGE = 4 * GTILE;             // A_hi, A_lo, B_hi, B_lo
constexpr int GSMEM = GSTAGES * GSTAGE + 1024;  // + alignment slack

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                   // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;         // stride byte offset
  d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                   // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = 128.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(GBN >> 3) << 17) |
                            ((uint32_t)(GBM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
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
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// byte offset of 16-byte chunk ch (k = 4 ch .. 4 ch + 3) of row `row` in a K-major SW128 tile
__device__ __forceinline__ uint32_t sw_chunk(int row, int ch) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((ch ^ (row & 7)) << 4));
}

// cp.async the raw fp32 128 x 32 tile rows [r0, r0+128) x k [k0, k0+32) of a K-major operand
// (stored [rows][ld], ld % 4 == 0) into its swizzled position (zero-filled outside).
__device__ __forceinline__ void load_tile_async(const float *__restrict__ G, int ld, int rows, int K, int r0, int k0,
                                                uint8_t *dst, int tid) {
#pragma unroll
  for (int j = 0; j < GCH; ++j) {
    const int f = tid + GTHREADS * j, row = f >> 3, ch = f & 7;
    const int r = r0 + row, k = k0 + ch * 4;
    const int bytes = (r < rows && k < K) ? min(16, (K - k) * 4) : 0;
    const float *src = bytes ? G + (int64_t)r * ld + k : G;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(su32(dst + sw_chunk(row, ch))), "l"(src),
                 "r"(bytes));
  }
}
// in place: hi slot holds the raw fp32 values -> hi = rna_tf32(x) there, lo = x - hi in the lo tile
__device__ __forceinline__ void split_tile(uint8_t *hi, uint8_t *lo, int tid) {
#pragma unroll
  for (int j = 0; j < GCH; ++j) {
    const int off = (tid + GTHREADS * j) * 16;
    float4 v = *reinterpret_cast<float4 *>(hi + off), h, l;
    h.x = tf32_rna(v.x); h.y = tf32_rna(v.y); h.z = tf32_rna(v.z); h.w = tf32_rna(v.w);
    l.x = v.x - h.x; l.y = v.y - h.y; l.z = v.z - h.z; l.w = v.w - h.w;
    *reinterpret_cast<float4 *>(hi + off) = h;
    *reinterpret_cast<float4 *>(lo + off) = l;
  }
}

// C[M][N] (ldc) = beta * C + op(A) op(B)^T (+ bias[n]) (ReLU), op(A) = [M][K], op(B) = [N][K].
__global__ void __launch_bounds__(GTHREADS, 1) gemm_tf32x3_kernel(GemmArgs g) {
  extern __shared__ uint8_t gsm_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t empty_bar[GSTAGES];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "n"(GBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < GSTAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty_bar[s])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&done_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  const int nkb_all = (g.K + GBK - 1) / GBK;
  const int kb0 = blockIdx.z * g.kbs, nkb = min(nkb_all, kb0 + g.kbs) - kb0;   // split-K range
  // prologue: raw tiles of the first GSTAGES - 1 k-blocks in flight
#pragma unroll
  for (int p = 0; p < GSTAGES - 1; ++p) {
    if (p < nkb) {
      uint8_t *st = sm + p * GSTAGE;
      load_tile_async(g.A, g.lda, g.M, g.K, m0, (kb0 + p) * GBK, st, tid);
      load_tile_async(g.B, g.ldb, g.N, g.K, n0, (kb0 + p) * GBK, st + 2 * GTILE, tid);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb % GSTAGES;
    // refill the stage of k-block kb + GSTAGES - 1 once the MMAs that read it (kb - 1) are done
    const int kn = kb + GSTAGES - 1;
    if (kn < nkb) {
      const int sn = kn % GSTAGES;
      if (kb >= 1) mbar_wait(&empty_bar[sn], ((kb - 1) / GSTAGES) & 1);
      uint8_t *st = sm + sn * GSTAGE;
      load_tile_async(g.A, g.lda, g.M, g.K, m0, (kb0 + kn) * GBK, st, tid);
      load_tile_async(g.B, g.ldb, g.N, g.K, n0, (kb0 + kn) * GBK, st + 2 * GTILE, tid);
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(GSTAGES - 1));   // k-block kb has landed (this thread)
    __syncthreads();                                                  // ... for every thread
    uint8_t *st = sm + s * GSTAGE;
    split_tile(st, st + GTILE, tid);
    split_tile(st + 2 * GTILE, st + 3 * GTILE, tid);
    asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy stores -> tensor-core (async proxy) reads
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ah = su32(st), al = su32(st + GTILE), bh = su32(st + 2 * GTILE), bl = su32(st + 3 * GTILE);
#pragma unroll
      for (int kk = 0; kk < GBK / 8; ++kk) {          // K = 8 tf32 (32 bytes) per MMA
        const uint32_t o = kk * 32;
        const uint64_t dah = sw128_desc(ah + o), dal = sw128_desc(al + o);
        const uint64_t dbh = sw128_desc(bh + o), dbl = sw128_desc(bl + o);
        mma_tf32(tmem, dah, dbh, (kb | kk) != 0);
        mma_tf32(tmem, dah, dbl, 1);
        mma_tf32(tmem, dal, dbh, 1);
      }
      mma_commit(&empty_bar[s]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  if (tid == 0) mma_commit(&done_bar);
  mbar_wait(&done_bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");

  // epilogue: warp w owns accumulator lanes (rows) 32 (w % 4) .. + 31 and column half w / 4
  const int row = m0 + (warp & 3) * 32 + lane;
#pragma unroll 1
  for (int c0 = (warp >> 2) * (GBN / 2); c0 < (warp >> 2) * (GBN / 2) + GBN / 2; c0 += 32) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (row < g.M && g.P) {        // split-K: raw partial sums, combined by gemm_reduce_kernel
      float *prow = g.P + ((int64_t)blockIdx.z * g.M + row) * g.N;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int n = n0 + c0 + j;
        if (n < g.N) prow[n] = __uint_as_float(r[j]);
      }
    } else if (row < g.M) {
      float *crow = g.C + (int64_t)row * g.ldc;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int n = n0 + c0 + j;
        if (n < g.N) {
          float v = __uint_as_float(r[j]);
          if (g.bias) v += g.bias[n];
          if (g.relu) v = fmaxf(v, 0.f);
          if (g.beta != 0.f) v += g.beta * crow[n];
          crow[n] = v;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(GBN));
}

// out[c][r] = in[r][c]: in [R][C] (ld_in), out [C][R] (ld_out); 32 x 32 tiles through shared memory.
__global__ void transpose_kernel(const float *__restrict__ in, int R, int Cc, int ld_in, float *__restrict__ out,
                                 int ld_out) {
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

// C = beta C + sum_z P[z] (+ bias) (ReLU): the fixed-order combine of the split-K partials.
__global__ void gemm_reduce_kernel(const float *__restrict__ P, int splits, int M, int N, float *C, int ldc,
                                   const float *bias, int relu, float beta) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * N) return;
  const int row = (int)(e / N), n = (int)(e - (int64_t)row * N);
  float v = 0.f;
  for (int z = 0; z < splits; ++z) v += P[(int64_t)z * M * N + e];
  if (bias) v += bias[n];
  if (relu) v = fmaxf(v, 0.f);
  float *c = C + (int64_t)row * ldc + n;
  if (beta != 0.f) v += beta * *c;
  *c = v;
}

// Operands must be K-major with ld % 4 == 0 (kg_api.cu transposes the others).  When the
// output has fewer tiles than SMs, K is split over blockIdx.z (at most one wave of CTAs:
// 192 KB of shared memory per CTA) into `part` (capacity part_cap floats).
void launch_gemm_tc(const GemmArgs &g0, float *part, int64_t part_cap, cudaStream_t st) {
  if (g0.M <= 0 || g0.N <= 0) return;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gemm_tf32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GSMEM);
    configured = true;
  }
  GemmArgs g = g0;
  const int tiles = ((g.N + GBN - 1) / GBN) * ((g.M + GBM - 1) / GBM);
  const int nkb = (g.K + GBK - 1) / GBK;
  int splits = std::max(1, std::min(148 / std::max(tiles, 1), nkb / 4));
  while (splits > 1 && (!part || (int64_t)splits * g.M * g.N > part_cap)) --splits;
  g.kbs = (nkb + splits - 1) / splits;
  splits = (nkb + g.kbs - 1) / g.kbs;
  g.P = splits > 1 ? part : nullptr;
  dim3 grid((g.N + GBN - 1) / GBN, (g.M + GBM - 1) / GBM, splits);
  { gemm_tf32x3_kernel<<<grid, GTHREADS, GSMEM, st>>>(g); ++g_launches; }
  if (splits > 1) {
    const int64_t n = (int64_t)g.M * g.N;
    { gemm_reduce_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(part, splits, g.M, g.N, g.C, g.ldc, g.bias, g.relu,
                                                                g.beta); ++g_launches; }
  }
}

}  // namespace kg
