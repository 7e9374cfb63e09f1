// k_adam.cu -- parameter init, deterministic segment-reduce + sparse Adam,
// relation-gradient reduce, dense Adam, bias column sums.
//
// PAPER.md §4.2: only the rows of V_q, N_q, A_q (and their Adam
// moments) are read/written per step; §4.1: theta_D is updated
// densely after the AllReduce.  Adam per reading A15 (textbook bias
// correction; bc = [1 - beta1^t, 1 - beta2^t] computed on device by the loss
// kernel).  All reductions run in a fixed order (no atomics).
#include "kg_common.cuh"
#include "kg_launch.h"

namespace kg {

// ------------------------------------------------------------------ init (A23)
__global__ void init_rows_kernel(float *p, int64_t rows, int d, int64_t row0, int64_t row_step, uint64_t seed,
                                 uint64_t stream, float lo, float hi) {
  KG_GRID_DEP_WAIT();
  const int64_t n = rows * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lr = e / d, c = e - lr * d;
    const uint64_t g = (uint64_t)(row0 + lr * row_step);
    p[e] = counter_uniform(seed, stream, g * (uint64_t)d + (uint64_t)c, lo, hi);
  }
}
__global__ void init_flat_kernel(float *p, int64_t n, uint64_t seed, uint64_t stream, float lo, float hi) {
  KG_GRID_DEP_WAIT();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    p[e] = counter_uniform(seed, stream, (uint64_t)e, lo, hi);
}

static int grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = 148 * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

void launch_init_rows(float *p, int64_t rows, int d, int64_t row0, int64_t row_step, uint64_t seed, uint64_t stream,
                      float lo, float hi, cudaStream_t st) {
  if (rows <= 0) return;
  { init_rows_kernel<<<grid_for(rows * d, 256), 256, 0, st>>>(p, rows, d, row0, row_step, seed, stream, lo, hi); ++g_launches; }
}
void launch_init_flat(float *p, int64_t n, uint64_t seed, uint64_t stream, float lo, float hi, cudaStream_t st) {
  if (n <= 0) return;
  { init_flat_kernel<<<grid_for(n, 256), 256, 0, st>>>(p, n, seed, stream, lo, hi); ++g_launches; }
}

// ------------------------------------------------------------------ Adam
// h = {beta1, 1 - beta1, beta2, 1 - beta2} (the complements formed in double on the host:
// 1 - beta2 in fp32 would lose ~1e-5 of its value), eps; bc = {1 - beta1^t, 1 - beta2^t}.
struct AdamHyper { float b1, omb1, b2, omb2, eps; };
// ibc = {1 / (1 - beta1^t), 1 / (1 - beta2^t)} (formed in double by the loss kernel);
// lr1 = lr * ibc[0].  p -= lr * (m / bc1) / (sqrt(v / bc2) + eps) with the divisions by the
// bias corrections as multiplications and the last one as a 2-ulp reciprocal-divide.
__device__ __forceinline__ void adam1(float &p, float &m, float &v, float g, float lr1, const AdamHyper &h,
                                      float ibc2) {
  m = fmaf(h.b1, m, h.omb1 * g);
  v = fmaf(h.b2, v, h.omb2 * g * g);
  p -= lr1 * __fdividef(m, sqrtf(v * ibc2) + h.eps);
}
__device__ __forceinline__ void adam4(float4 &p, float4 &m, float4 &v, const float4 g, float lr1, const AdamHyper &h,
                                      float ibc2) {
  adam1(p.x, m.x, v.x, g.x, lr1, h, ibc2);
  adam1(p.y, m.y, v.y, g.y, lr1, h, ibc2);
  adam1(p.z, m.z, v.z, g.z, lr1, h, ibc2);
  adam1(p.w, m.w, v.w, g.w, lr1, h, ibc2);
}
static AdamHyper hyper(double b1, double b2, double eps) {
  return AdamHyper{(float)b1, (float)(1.0 - b1), (float)b2, (float)(1.0 - b2), (float)eps};
}

// ---------------------------------------------------------------- segment reduce
// Occurrence rows X[L][w] are grouped by the dedup's sorted positions s (perm[s] =
// occurrence, inv[perm[s]] = its distinct index u, seg[u] = first sorted position
// of u).  Hot ids (Zipf anchors / relations) have long segments, so a segment is
// cut into "pieces": a piece starts at every segment head and at every multiple
// of kPiece.  Phase 1 sums each piece (kPiece independent loads in flight per
// thread) into PS[piece start]; phase 2 sums the pieces of a segment in
// ascending order.  The order of every sum is a fixed function of the sorted
// positions: deterministic, no atomics (P:L343 merge).  Segments of length 1
// skip phase 1.
constexpr int kPiece = 16;

__global__ void __launch_bounds__(128) seg_piece_kernel(const int32_t *perm, const int32_t *inv, const int32_t *seg,
                                                        int L, const float *X, int w4, float *PS) {
  KG_GRID_DEP_WAIT();
  __shared__ int s_row[kPiece], s_beg[kPiece], s_len[kPiece];
  const int c0 = blockIdx.x * kPiece;
  const int n = min(kPiece, L - c0);
  if (threadIdx.x < n) {
    const int s = c0 + threadIdx.x, r = perm[s], u = inv[r];
    s_row[threadIdx.x] = r;
    s_beg[threadIdx.x] = seg[u];
    s_len[threadIdx.x] = seg[u + 1] - seg[u];
  }
  __syncthreads();
  const float4 *X4 = reinterpret_cast<const float4 *>(X);
  float4 *P4 = reinterpret_cast<float4 *>(PS);
  for (int c = threadIdx.x; c < w4; c += blockDim.x) {
    float4 v[kPiece];
#pragma unroll
    for (int i = 0; i < kPiece; ++i)
      if (i < n && s_len[i] > 1) v[i] = X4[(int64_t)s_row[i] * w4 + c];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int start = -1;
#pragma unroll
    for (int i = 0; i < kPiece; ++i) {
      if (i >= n || s_len[i] <= 1) continue;
      const int s = c0 + i;
      if (s == s_beg[i] || start < 0) {           // a new piece (segment head or chunk start)
        if (start >= 0) P4[(int64_t)start * w4 + c] = acc;
        acc = v[i];
        start = s;
      } else {
        acc.x += v[i].x; acc.y += v[i].y; acc.z += v[i].z; acc.w += v[i].w;
      }
    }
    if (start >= 0) P4[(int64_t)start * w4 + c] = acc;
  }
}

__device__ __forceinline__ float4 segment_sum(const int32_t *perm, const float4 *X4, const float4 *P4, int s0, int s1,
                                              int w4, int c) {
  if (s1 - s0 == 1) return X4[(int64_t)perm[s0] * w4 + c];
  float4 g = P4[(int64_t)s0 * w4 + c];
  for (int s = (s0 / kPiece + 1) * kPiece; s < s1; s += kPiece) {
    const float4 o = P4[(int64_t)s * w4 + c];
    g.x += o.x; g.y += o.y; g.z += o.z; g.w += o.w;
  }
  return g;
}

// Phase 2 for theta_E: one warp per distinct row u, lanes over float4 columns:
// G_u, then Adam on (p, m, v) of the row (local row = id / world).  Every touched
// row is updated, including rows whose gradient is zero (A16).
__global__ void __launch_bounds__(256) sparse_adam_kernel(const int64_t *uniq, const int32_t *seg,
                                                          const int32_t *perm, const int32_t *U_dev, const float *OG,
                                                          const float *PS, int d, int world, float *ent, float *m,
                                                          float *v, float *grad_out, const float *lr_dev, AdamHyper hy,
                                                          const float *bc, const int *flags, int apply,
                                                          int64_t skip_key) {
  KG_GRID_DEP_WAIT();
  const int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (u >= *U_dev || uniq[u] == skip_key) return;   // skip_key: the empty-slot key of bucketed exchanges
  const int d4 = d >> 2, s0 = seg[u], s1 = seg[u + 1];
  const bool upd = apply && !flags[0];
  const float lr1 = *lr_dev * bc[0], ibc2 = bc[1];
  const int64_t rowoff = (uniq[u] / world) * d4;
  const float4 *X4 = reinterpret_cast<const float4 *>(OG), *P4 = reinterpret_cast<const float4 *>(PS);
  float4 *pe = reinterpret_cast<float4 *>(ent) + rowoff, *pm = reinterpret_cast<float4 *>(m) + rowoff,
         *pv = reinterpret_cast<float4 *>(v) + rowoff;
  // d <= 2048: at most 16 float4 per lane; issue the row's p, m, v loads before the arithmetic
  constexpr int kMaxIt = 4;
  for (int c0 = 0; c0 < d4; c0 += 32 * kMaxIt) {
    float4 P[kMaxIt], Mm[kMaxIt], V[kMaxIt], Gq[kMaxIt];
#pragma unroll
    for (int it = 0; it < kMaxIt; ++it) {
      const int c = c0 + lane + 32 * it;
      if (c >= d4) continue;
      Gq[it] = segment_sum(perm, X4, P4, s0, s1, d4, c);
      if (upd) { P[it] = pe[c]; Mm[it] = pm[c]; V[it] = pv[c]; }
    }
#pragma unroll
    for (int it = 0; it < kMaxIt; ++it) {
      const int c = c0 + lane + 32 * it;
      if (c >= d4) continue;
      if (grad_out) reinterpret_cast<float4 *>(grad_out)[(int64_t)u * d4 + c] = Gq[it];
      if (!upd) continue;
      adam4(P[it], Mm[it], V[it], Gq[it], lr1, hy, ibc2);
      pe[c] = P[it]; pm[c] = Mm[it]; pv[c] = V[it];
    }
  }
}

void launch_sparse_adam(const int64_t *uniq, const int32_t *seg, const int32_t *perm, const int32_t *inv,
                        const int32_t *U_dev, int L, const float *OG, float *PS, int d, int world, float *ent,
                        float *m, float *v, float *grad_out, const float *lr, double beta1, double beta2, double eps,
                        const float *bc, const int *flags, int apply, cudaStream_t st, int64_t skip_key) {
  if (L <= 0) return;
  { seg_piece_kernel<<<(L + kPiece - 1) / kPiece, 128, 0, st>>>(perm, inv, seg, L, OG, d / 4, PS); ++g_launches; }
  { sparse_adam_kernel<<<(L + 7) / 8, 256, 0, st>>>(uniq, seg, perm, U_dev, OG, PS, d, world, ent, m, v,
                                                              grad_out, lr, hyper(beta1, beta2, eps), bc, flags,
                                                              apply, skip_key); ++g_launches; }
}

// Phase 2 for the relation rows: RGU[u] = sum of the occurrence rows of relation u.
__global__ void __launch_bounds__(256) rel_reduce_kernel(const int32_t *seg, const int32_t *perm,
                                                         const int32_t *U_dev, const float *RG, const float *PS,
                                                         int dr, float *RGU) {
  KG_GRID_DEP_WAIT();
  const int w4 = dr >> 2;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int u = (int)(e / w4), c = (int)(e - (int64_t)u * w4);
  if (u >= *U_dev) return;
  reinterpret_cast<float4 *>(RGU)[(int64_t)u * w4 + c] =
      segment_sum(perm, reinterpret_cast<const float4 *>(RG), reinterpret_cast<const float4 *>(PS), seg[u],
                  seg[u + 1], w4, c);
}
void launch_rel_reduce(const int32_t *seg, const int32_t *perm, const int32_t *inv, const int32_t *U_dev, int Lr,
                       const float *RG, float *PS, int dr, float *RGU, cudaStream_t st) {
  if (Lr <= 0) return;
  { seg_piece_kernel<<<(Lr + kPiece - 1) / kPiece, 128, 0, st>>>(perm, inv, seg, Lr, RG, dr / 4, PS); ++g_launches; }
  const int64_t n = (int64_t)Lr * (dr / 4);
  { rel_reduce_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(seg, perm, U_dev, RG, PS, dr, RGU); ++g_launches; }
}

// rel_seg[r] = index of relation r's reduced gradient row, valid iff rel_stamp[r] == stamp.
// (Avoids zeroing / reading a dense |R| x d gradient for the untouched relation rows.)
__global__ void rel_stamp_kernel(const int64_t *uniq_rel, const int32_t *U_dev, int32_t *rel_seg,
                                 int64_t *rel_stamp, const int64_t *stamp) {
  KG_GRID_DEP_WAIT();
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= *U_dev) return;
  const int64_t r = uniq_rel[u];
  rel_seg[r] = u;
  rel_stamp[r] = *stamp;
}
void launch_rel_stamp(const int64_t *uniq_rel, const int32_t *U_dev, int Lmax, int32_t *rel_seg, int64_t *rel_stamp,
                      const int64_t *stamp, cudaStream_t st) {
  { rel_stamp_kernel<<<(Lmax + 255) / 256, 256, 0, st>>>(uniq_rel, U_dev, rel_seg, rel_stamp, stamp); ++g_launches; }
}

// Dense Adam over theta_D (A17: every element, every step).  Streaming kernel:
// each thread issues the loads of kE float4 elements (p, m, v, g) before any
// arithmetic, evict-first cache hints (the 300 MB of Adam state is touched once
// per step), no grid cap (one pass).
// REL: the relation tables, nseg segments of [R][width] stored back to back
// (Q2B: rel_center, rel_offset); the gradient of row r of segment s is
// RGU[rel_seg[r]][s*width + c] when relation r was used by this step
// (rel_stamp[r] == stamp), else 0.  !REL: the operator weights, gradient g.
constexpr int kE = 2;

// q = n / D for n < 2^32 via a 64-bit reciprocal (exact for n < 2^40 / D).
struct FastDiv {
  uint64_t mul;
  uint32_t d;
};
static FastDiv fastdiv(uint32_t d) { return FastDiv{(((uint64_t)1 << 40) + d - 1) / d, d}; }
__device__ __forceinline__ uint32_t fdiv(uint32_t n, FastDiv f) { return (uint32_t)(((uint64_t)n * f.mul) >> 40); }

// Relation tables: flat stream over nseg * R rows of w4 float4; the gradient of row r
// of segment s is RGU[rel_seg[r]][s*w4 + c] when relation r was used by this step
// (rel_stamp[r] == stamp), else 0 (A17).  kE float4 per thread, loads issued first.
// untouched_only: update only the relation rows this step does not use (g = 0, A17) -- they
// depend on no gradient of the step, so the update runs early, concurrently with the
// ALU-bound scoring; the touched rows follow in dense_adam_rel_touched_kernel.
__global__ void __launch_bounds__(256) dense_adam_rel_kernel(float4 *p, float4 *m, float4 *v, int n4, FastDiv fw4,
                                                             int R, int nseg, const float *RGU,
                                                             const int32_t *rel_seg, const int64_t *rel_stamp,
                                                             const int64_t *stamp_dev, const float *lr_dev,
                                                             AdamHyper hy, const float *bc, const int *flags,
                                                             int untouched_only) {
  KG_GRID_DEP_WAIT();
  if (flags[0]) return;
  const float lr1 = *lr_dev * bc[0], ibc2 = bc[1];
  const int64_t stamp = *stamp_dev;
  const int w4 = (int)fw4.d;
  const int base = blockIdx.x * (256 * kE) + threadIdx.x;
  float4 P[kE], Mm[kE], V[kE], G[kE];
  bool skip[kE];
#pragma unroll
  for (int k = 0; k < kE; ++k) {
    const int e = base + k * 256;
    skip[k] = e >= n4;
    if (skip[k]) continue;
    const int row = (int)fdiv((uint32_t)e, fw4), c4 = e - row * w4;
    const int sidx = row >= R ? 1 : 0, r = row - sidx * R;
    const bool used = rel_stamp[r] == stamp;
    skip[k] = untouched_only && used;
    if (skip[k]) continue;
    P[k] = __ldcs(p + e);
    Mm[k] = __ldcs(m + e);
    V[k] = __ldcs(v + e);
    G[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (used) G[k] = reinterpret_cast<const float4 *>(RGU)[(int64_t)rel_seg[r] * nseg * w4 + sidx * w4 + c4];
  }
#pragma unroll
  for (int k = 0; k < kE; ++k) {
    const int e = base + k * 256;
    if (skip[k]) continue;
    adam4(P[k], Mm[k], V[k], G[k], lr1, hy, ibc2);
    __stcs(p + e, P[k]);
    __stcs(m + e, Mm[k]);
    __stcs(v + e, V[k]);
  }
}

// The relation rows used by this step: row runiq[u] of each of the nseg segments, gradient
// RGU[u][s][c] (the relation-occurrence reduce), u < *rU.
__global__ void __launch_bounds__(256) dense_adam_rel_touched_kernel(float4 *p, float4 *m, float4 *v, int R, int w4,
                                                                     int nseg, const float *RGU,
                                                                     const int64_t *runiq, const int32_t *rU,
                                                                     const float *lr_dev, AdamHyper hy,
                                                                     const float *bc, const int *flags) {
  KG_GRID_DEP_WAIT();
  if (flags[0]) return;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int per = nseg * w4;
  const int u = (int)(e / per);
  if (u >= *rU) return;
  const int rem = (int)(e - (int64_t)u * per), s = rem / w4, c4 = rem - s * w4;
  const int64_t idx = ((int64_t)s * R + runiq[u]) * w4 + c4;
  const float lr1 = *lr_dev * bc[0], ibc2 = bc[1];
  float4 P = p[idx], Mm = m[idx], V = v[idx];
  adam4(P, Mm, V, reinterpret_cast<const float4 *>(RGU)[e], lr1, hy, ibc2);
  p[idx] = P;
  m[idx] = Mm;
  v[idx] = V;
}

// Operator weights: flat stream, kE float4 per thread, loads issued first.
__global__ void __launch_bounds__(256) dense_adam_kernel(float4 *p, float4 *m, float4 *v, const float4 *g, int n4,
                                                         const float *lr_dev, AdamHyper hy, const float *bc,
                                                         const int *flags) {
  KG_GRID_DEP_WAIT();
  if (flags[0]) return;
  const float lr1 = *lr_dev * bc[0], ibc2 = bc[1];
  const int base = blockIdx.x * (256 * kE) + threadIdx.x;
  float4 P[kE], Mm[kE], V[kE], G[kE];
#pragma unroll
  for (int k = 0; k < kE; ++k) {
    const int e = base + k * 256;
    if (e >= n4) continue;
    P[k] = __ldcs(p + e);
    Mm[k] = __ldcs(m + e);
    V[k] = __ldcs(v + e);
    G[k] = __ldcs(g + e);
  }
#pragma unroll
  for (int k = 0; k < kE; ++k) {
    const int e = base + k * 256;
    if (e >= n4) continue;
    adam4(P[k], Mm[k], V[k], G[k], lr1, hy, ibc2);
    __stcs(p + e, P[k]);
    __stcs(m + e, Mm[k]);
    __stcs(v + e, V[k]);
  }
}

void launch_dense_adam_rel(float *p, float *m, float *v, int R, int width, int nseg, const float *RGU,
                           const int32_t *rel_seg, const int64_t *rel_stamp, const int64_t *stamp, const float *lr,
                           double beta1, double beta2, double eps, const float *bc, const int *flags,
                           cudaStream_t st, int untouched_only) {
  const int n4 = nseg * R * (width / 4);
  if (n4 <= 0) return;
  { dense_adam_rel_kernel<<<(n4 + 256 * kE - 1) / (256 * kE), 256, 0, st>>>(
        reinterpret_cast<float4 *>(p), reinterpret_cast<float4 *>(m), reinterpret_cast<float4 *>(v), n4,
        fastdiv((uint32_t)(width / 4)), R, nseg, RGU, rel_seg, rel_stamp, stamp, lr, hyper(beta1, beta2, eps), bc,
        flags, untouched_only); ++g_launches; }
}
void launch_dense_adam_rel_touched(float *p, float *m, float *v, int R, int width, int nseg, const float *RGU,
                                   const int64_t *runiq, const int32_t *rU, int Lr, const float *lr, double beta1,
                                   double beta2, double eps, const float *bc, const int *flags, cudaStream_t st) {
  const int64_t n = (int64_t)Lr * nseg * (width / 4);
  if (n <= 0) return;
  { dense_adam_rel_touched_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<float4 *>(p), reinterpret_cast<float4 *>(m), reinterpret_cast<float4 *>(v), R, width / 4,
        nseg, RGU, runiq, rU, lr, hyper(beta1, beta2, eps), bc, flags); ++g_launches; }
}

void launch_dense_adam(float *p, float *m, float *v, const float *g, int64_t n, const float *lr, double beta1,
                       double beta2, double eps, const float *bc, const int *flags, cudaStream_t st) {
  const int n4 = (int)(n / 4);
  if (n4 <= 0) return;
  { dense_adam_kernel<<<(n4 + 256 * kE - 1) / (256 * kE), 256, 0, st>>>(
        reinterpret_cast<float4 *>(p), reinterpret_cast<float4 *>(m), reinterpret_cast<float4 *>(v),
        reinterpret_cast<const float4 *>(g), n4, lr, hyper(beta1, beta2, eps), bc, flags); ++g_launches; }
}

// out[c] = sum_r X[r*ld + c]; 32 columns x 32 row-lanes per block, fixed-order smem reduce.
__global__ void __launch_bounds__(1024) colsum_kernel(const float *X, int rows, int cols, int ld, float *out) {
  KG_GRID_DEP_WAIT();
  __shared__ float red[32][33];
  const int cx = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cx;
  float s = 0.f;
  if (c < cols)
    for (int r = ry; r < rows; r += 32) s += X[(int64_t)r * ld + c];
  red[ry][cx] = s;
  __syncthreads();
  if (ry == 0 && c < cols) {
    float t = 0.f;
    for (int k = 0; k < 32; ++k) t += red[k][cx];
    out[c] = t;
  }
}
void launch_colsum(const float *X, int rows, int cols, int ld, float *out, cudaStream_t st) {
  { colsum_kernel<<<(cols + 31) / 32, 1024, 0, st>>>(X, rows, cols, ld, out); ++g_launches; }
}

}  // namespace kg
