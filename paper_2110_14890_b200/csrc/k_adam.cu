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
  const int64_t n = rows * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lr = e / d, c = e - lr * d;
    const uint64_t g = (uint64_t)(row0 + lr * row_step);
    p[e] = counter_uniform(seed, stream, g * (uint64_t)d + (uint64_t)c, lo, hi);
  }
}
__global__ void init_flat_kernel(float *p, int64_t n, uint64_t seed, uint64_t stream, float lo, float hi) {
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
__device__ __forceinline__ void adam1(float &p, float &m, float &v, float g, float lr, const AdamHyper &h, float bc1,
                                      float bc2) {
  m = h.b1 * m + h.omb1 * g;
  v = h.b2 * v + h.omb2 * g * g;
  p -= lr * (m / bc1) / (sqrtf(v / bc2) + h.eps);
}
__device__ __forceinline__ void adam4(float4 &p, float4 &m, float4 &v, const float4 g, float lr, const AdamHyper &h,
                                      float bc1, float bc2) {
  adam1(p.x, m.x, v.x, g.x, lr, h, bc1, bc2);
  adam1(p.y, m.y, v.y, g.y, lr, h, bc1, bc2);
  adam1(p.z, m.z, v.z, g.z, lr, h, bc1, bc2);
  adam1(p.w, m.w, v.w, g.w, lr, h, bc1, bc2);
}
static AdamHyper hyper(double b1, double b2, double eps) {
  return AdamHyper{(float)b1, (float)(1.0 - b1), (float)b2, (float)(1.0 - b2), (float)eps};
}

// One warp per distinct row u: G_u = sum of its occurrence gradients in
// ascending position order (anchors, answers, pool, A16), then Adam on
// (p, m, v) of the row (local row = id / world).  Every touched row is updated,
// including rows whose gradient is zero (A16).
__global__ void __launch_bounds__(256) sparse_adam_kernel(const int64_t *uniq, const int32_t *seg,
                                                          const int32_t *perm, const int32_t *U_dev, const float *OG,
                                                          int d, int world, float *ent, float *m, float *v,
                                                          float *grad_out, float lr, AdamHyper hy,
                                                          const float *bc, const int *flags, int apply) {
  const int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (u >= *U_dev) return;
  const int s0 = seg[u], s1 = seg[u + 1];
  const bool upd = apply && !flags[0];
  const int64_t row = uniq[u] / world;
  const float bc1 = bc[0], bc2 = bc[1];
  const int d4 = d >> 2;
  for (int c = lane; c < d4; c += 32) {
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = s0; s < s1; ++s) {
      const float4 o = reinterpret_cast<const float4 *>(OG + (int64_t)perm[s] * d)[c];
      g.x += o.x; g.y += o.y; g.z += o.z; g.w += o.w;
    }
    if (grad_out) reinterpret_cast<float4 *>(grad_out + (int64_t)u * d)[c] = g;
    if (!upd) continue;
    float4 *pp = reinterpret_cast<float4 *>(ent + row * d) + c;
    float4 *mp = reinterpret_cast<float4 *>(m + row * d) + c;
    float4 *vp = reinterpret_cast<float4 *>(v + row * d) + c;
    float4 P = *pp, Mm = *mp, V = *vp;
    adam4(P, Mm, V, g, lr, hy, bc1, bc2);
    *pp = P; *mp = Mm; *vp = V;
  }
}

void launch_sparse_adam(const int64_t *uniq, const int32_t *seg, const int32_t *perm, const int32_t *U_dev, int Lmax,
                        const float *OG, int d, int world, float *ent, float *m, float *v, float *grad_out, float lr,
                        double beta1, double beta2, double eps, const float *bc, const int *flags, int apply,
                        cudaStream_t st) {
  const int warps = 8;
  { sparse_adam_kernel<<<(Lmax + warps - 1) / warps, warps * 32, 0, st>>>(uniq, seg, perm, U_dev, OG, d, world, ent, m,
                                                                        v, grad_out, lr, hyper(beta1, beta2, eps), bc,
                                                                        flags, apply); ++g_launches; }
}

// Relation occurrence gradients -> one row per distinct relation (fixed order).
__global__ void __launch_bounds__(256) rel_reduce_kernel(const int32_t *seg, const int32_t *perm,
                                                         const int32_t *U_dev, const float *RG, int dr, float *RGU) {
  const int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (u >= *U_dev) return;
  const int s0 = seg[u], s1 = seg[u + 1];
  for (int c = lane; c < dr; c += 32) {
    float g = 0.f;
    for (int s = s0; s < s1; ++s) g += RG[(int64_t)perm[s] * dr + c];
    RGU[(int64_t)u * dr + c] = g;
  }
}
void launch_rel_reduce(const int32_t *seg, const int32_t *perm, const int32_t *U_dev, int Lmax, const float *RG,
                       int dr, float *RGU, cudaStream_t st) {
  { rel_reduce_kernel<<<(Lmax + 7) / 8, 256, 0, st>>>(seg, perm, U_dev, RG, dr, RGU); ++g_launches; }
}

// rel_seg[r] = index of relation r's reduced gradient row, valid iff rel_stamp[r] == stamp.
// (Avoids zeroing / reading a dense |R| x d gradient for the untouched relation rows.)
__global__ void rel_stamp_kernel(const int64_t *uniq_rel, const int32_t *U_dev, int32_t *rel_seg,
                                 int64_t *rel_stamp, int64_t stamp) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= *U_dev) return;
  const int64_t r = uniq_rel[u];
  rel_seg[r] = u;
  rel_stamp[r] = stamp;
}
void launch_rel_stamp(const int64_t *uniq_rel, const int32_t *U_dev, int Lmax, int32_t *rel_seg, int64_t *rel_stamp,
                      int64_t stamp, cudaStream_t st) {
  { rel_stamp_kernel<<<(Lmax + 255) / 256, 256, 0, st>>>(uniq_rel, U_dev, rel_seg, rel_stamp, stamp); ++g_launches; }
}

// Dense Adam over a relation table [R][width] (A17: every row, g = 0 if unused).
__global__ void __launch_bounds__(256) dense_adam_rel_kernel(float *p, float *m, float *v, int R, int width,
                                                             const float *RGU, int rg_stride, int rg_col,
                                                             const int32_t *rel_seg, const int64_t *rel_stamp,
                                                             int64_t stamp, float lr, AdamHyper hy,
                                                             const float *bc, const int *flags) {
  if (flags[0]) return;
  const int w4 = width >> 2;
  const int64_t n4 = (int64_t)R * w4;
  const float bc1 = bc[0], bc2 = bc[1];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / w4), c4 = (int)(e - (int64_t)r * w4);
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rel_stamp[r] == stamp) g = *reinterpret_cast<const float4 *>(RGU + (int64_t)rel_seg[r] * rg_stride + rg_col + c4 * 4);
    float4 P = reinterpret_cast<float4 *>(p)[e], Mm = reinterpret_cast<float4 *>(m)[e], V = reinterpret_cast<float4 *>(v)[e];
    adam4(P, Mm, V, g, lr, hy, bc1, bc2);
    reinterpret_cast<float4 *>(p)[e] = P;
    reinterpret_cast<float4 *>(m)[e] = Mm;
    reinterpret_cast<float4 *>(v)[e] = V;
  }
}
void launch_dense_adam_rel(float *p, float *m, float *v, int R, int width, const float *RGU, int rg_stride,
                           int rg_col, const int32_t *rel_seg, const int64_t *rel_stamp, int64_t stamp, float lr,
                           double beta1, double beta2, double eps, const float *bc, const int *flags, cudaStream_t st) {
  const int64_t n4 = (int64_t)R * (width / 4);
  { dense_adam_rel_kernel<<<grid_for(n4, 256), 256, 0, st>>>(p, m, v, R, width, RGU, rg_stride, rg_col, rel_seg,
                                                           rel_stamp, stamp, lr, hyper(beta1, beta2, eps), bc, flags); ++g_launches; }
}

__global__ void __launch_bounds__(256) dense_adam_kernel(float *p, float *m, float *v, const float *g, int64_t n4,
                                                         float lr, AdamHyper hy, const float *bc,
                                                         const int *flags) {
  if (flags[0]) return;
  const float bc1 = bc[0], bc2 = bc[1];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
    float4 P = reinterpret_cast<float4 *>(p)[e], Mm = reinterpret_cast<float4 *>(m)[e], V = reinterpret_cast<float4 *>(v)[e];
    adam4(P, Mm, V, reinterpret_cast<const float4 *>(g)[e], lr, hy, bc1, bc2);
    reinterpret_cast<float4 *>(p)[e] = P;
    reinterpret_cast<float4 *>(m)[e] = Mm;
    reinterpret_cast<float4 *>(v)[e] = V;
  }
}
void launch_dense_adam(float *p, float *m, float *v, const float *g, int64_t n, float lr, double beta1, double beta2,
                       double eps, const float *bc, const int *flags, cudaStream_t st) {
  if (n <= 0) return;
  { dense_adam_kernel<<<grid_for(n / 4, 256), 256, 0, st>>>(p, m, v, g, n / 4, lr, hyper(beta1, beta2, eps), bc, flags); ++g_launches; }
}

// out[c] = sum_r X[r*ld + c]; 32 columns x 32 row-lanes per block, fixed-order smem reduce.
__global__ void __launch_bounds__(1024) colsum_kernel(const float *X, int rows, int cols, int ld, float *out) {
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
