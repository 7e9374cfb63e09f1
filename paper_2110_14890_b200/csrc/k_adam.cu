// k_adam.cu -- parameter init, deterministic segment-reduce + sparse Adam,
// relation-gradient reduce, dense Adam, bias column sums.
//
// PAPER.md §4.2: only the rows of V_q, N_q, A_q (and their Adam
// moments) are read/written per step; §4.1: theta_D is updated
// densely after the AllReduce.  Adam per reading A15 (textbook bias
// correction; bc = [1 - beta1^t, 1 - beta2^t] computed on device by the loss
// kernel).  All reductions run in a fixed order (no atomics).
#include <algorithm>

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

// Fused segment reduce + sparse Adam for theta_E (a12 + a13): one launch, no atomics on
// rows, every row staged through shared memory by bulk copies (TMA, cp.async.bulk), so a
// warp keeps its whole row in flight without holding it in registers.  The sorted
// occurrence positions are cut into the pieces defined above (a piece starts at every
// segment head and at every multiple of kPiece).  One warp per item:
//
//  * chunk item (c, q), items [0, nch * NS), launched first (the hot rows' chains are the
//    longest): sorted positions [kPiece c, kPiece c + kPiece) x the q-th of NS column
//    slices.  The occurrence rows of every repeated segment in the chunk are copied in
//    together (one bulk copy of the slice per position) and summed into their pieces in
//    position order.  A segment inside one piece gets its Adam update here, on the slice
//    (its p, m, v slices were prefetched to L2 with the copies).  A segment of several
//    pieces (hot Zipf anchors) writes each piece sum to PS[piece start]; the item
//    completing the last piece of (u, q) -- arrival counter cnt[u * kSlices + q], reset by
//    that item -- sums the pieces in ascending order and applies Adam to the slice.
//  * head item u, items [nch * NS, nch * NS + L): a distinct row with ONE occurrence
//    (every pool row but a few, most answers; hrow[u] >= 0): bulk copies of its p, m, v
//    rows and of its gradient row into the warp's shared memory, one mbarrier, then Adam
//    with lanes over float4 columns and coalesced stores.  Repeated rows return at once.
//
// Every sum runs in a fixed order (deterministic run to run).  With `early`, index loads
// and the p / m / v copies go out before griddepcontrol.wait: the row ids come from the
// dedup at the start of the step and theta_E / m / v are written by no kernel of the step
// before this one; only the occurrence gradients (and flags) wait for the predecessor.
constexpr int kSlices = 16;   // column slices per row (counter stride): d <= 16 * 32 * 4
#ifndef KG_SA_PROBE
#define KG_SA_PROBE 0         // tools/sparse_probe.py variants: 1 head items only, 2 chunk items only, 3 trace
#endif
#if KG_SA_PROBE == 3
__device__ unsigned long long g_sa_trace[1 << 16][4];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SA_T(k) do { if (lane == 0 && w < (1 << 16)) g_sa_trace[w][k] = gtime(); } while (0)
}  // namespace kg
extern "C" int probe_trace(unsigned long long *out) {
  return (int)cudaMemcpyFromSymbol(out, kg::g_sa_trace, sizeof(unsigned long long) * (1 << 18));
}
extern "C" int probe_trace_clear() {
  static unsigned long long z[1 << 18];
  return (int)cudaMemcpyToSymbol(kg::g_sa_trace, z, sizeof(z));
}
namespace kg {
#else
#define SA_T(k) do {} while (0)
#endif

__device__ __forceinline__ void add4(float4 &a, const float4 &b) { a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w; }
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t *b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void bar_wait0(uint64_t *b) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done)
                 : "r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

template <bool EARLY>
__global__ void __launch_bounds__(128, 8) sparse_adam_fused_kernel(const int64_t *uniq, const int32_t *seg,
                                                                   const int32_t *perm, const int32_t *sinv,
                                                                   const int32_t *hrow, const int32_t *U_dev, int L,
                                                                   const float *OG, float *PS, int32_t *cnt, int d,
                                                                   int world, int ns, int sw, int wbytes, float *ent,
                                                                   float *m, float *v, float *grad_out,
                                                                   const float *lr_dev, AdamHyper hy, const float *bc,
                                                                   const int *flags, int apply, int64_t skip_key) {
  extern __shared__ __align__(128) uint8_t sa_smem[];
  __shared__ __align__(8) uint64_t sa_bar[4];
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = blockIdx.x * 4 + wi;
  const int d4 = d >> 2;
  float4 *sm = reinterpret_cast<float4 *>(sa_smem + (size_t)wi * wbytes);
  uint64_t *bar = &sa_bar[wi];
  const float4 *X4 = reinterpret_cast<const float4 *>(OG);
  float4 *P4 = reinterpret_cast<float4 *>(PS);
  float4 *E4 = reinterpret_cast<float4 *>(ent), *M4 = reinterpret_cast<float4 *>(m),
         *V4 = reinterpret_cast<float4 *>(v), *GO4 = reinterpret_cast<float4 *>(grad_out);
  const int nch = (L + kPiece - 1) / kPiece;

  if (w >= nch * ns) {
    // ---------------------------------------------------------------- head item
    const int u = w - nch * ns;
#if KG_SA_PROBE == 2
    return;
#endif
    SA_T(0);
    if (!EARLY) KG_GRID_DEP_WAIT();
    // u < L <= the capacity of hrow / uniq: the three loads go out together, U is checked after
    const int Ud = *U_dev, r0 = hrow[u];          // r0: the row's one occurrence, -1 if repeated
    const int64_t key = uniq[u];
    if (u >= Ud || r0 < 0) return;                // repeated rows: the chunk items
    if (key == skip_key) return;                  // the empty-slot key of bucketed exchanges
    const int64_t rowoff = (key / world) * d4;
    const uint32_t rb = (uint32_t)d * 4u;
    SA_T(1);
    if (lane == 0) {
      bar_init(bar);
      bar_expect(bar, (apply ? 4u : 1u) * rb);
      if (apply) {                                // smem: [P | M | V | G]
        bulk_g2s(sm, E4 + rowoff, rb, bar);
        bulk_g2s(sm + d4, M4 + rowoff, rb, bar);
        bulk_g2s(sm + 2 * d4, V4 + rowoff, rb, bar);
      }
    }
    if (EARLY) KG_GRID_DEP_WAIT();
    if (lane == 0) bulk_g2s(sm + 3 * d4, X4 + (int64_t)r0 * d4, rb, bar);
    const bool upd = apply && !(flags[0] | flags[1]);          // the step's go / no-go, after the wait
    const float lr1 = *lr_dev * bc[0], ibc2 = bc[1];
    __syncwarp();
    bar_wait0(bar);
    SA_T(2);
    for (int c = lane; c < d4; c += 32) {
      const float4 G = sm[3 * d4 + c];
      if (GO4) GO4[(int64_t)u * d4 + c] = G;
      if (!upd) continue;
      float4 P = sm[c], Mm = sm[d4 + c], V = sm[2 * d4 + c];
      adam4(P, Mm, V, G, lr1, hy, ibc2);
      E4[rowoff + c] = P; M4[rowoff + c] = Mm; V4[rowoff + c] = V;
    }
    SA_T(3);
    return;
  }

  // ------------------------------------------------------------------ chunk item (c, q)
#if KG_SA_PROBE == 1
  return;
#endif
  SA_T(0);
  const int c = w / ns, q = w - c * ns;
  const int base = c * kPiece;
  const int n = min(kPiece, L - base);
  const int c0 = q * sw, cw = min(sw, d4 - c0);   // this slice: float4 columns [c0, c0 + cw)
  const int col = c0 + lane;
  const bool cv = lane < cw;
  // lane j < n: the occurrence at sorted position base + j
  int pj = 0, uj = 0, s0j = 0, s1j = 0;
  int64_t kj = 0;
  if (!EARLY) KG_GRID_DEP_WAIT();
  if (lane < n) {
    pj = perm[base + lane];
    uj = sinv[base + lane];
    s0j = seg[uj];
    s1j = seg[uj + 1];
    kj = uniq[uj];
  }
  const bool rep = lane < n && s1j - s0j > 1 && kj != skip_key;
  const unsigned rep_mask = __ballot_sync(0xffffffffu, rep);
  if (!rep_mask) return;
  SA_T(1);
  // piece starts: a segment head or the chunk's first position; piece ends
  const unsigned start_mask = __ballot_sync(0xffffffffu, rep && (base + lane == s0j || lane == 0));
  const unsigned cont_mask = rep_mask & ~start_mask;
  const unsigned end_mask = rep_mask & ~(cont_mask >> 1);
  // the p, m, v slices of the segments starting in this piece to L2 now -- single-piece ones are
  // updated here, multi-piece (hot) ones by the item completing their last piece, which then
  // finds them in L2 instead of paying a DRAM round trip after the piece sums
  if (apply && base + lane == s0j && ((start_mask >> lane) & 1u)) {
    const int64_t off = (kj / world) * d4 + c0;
    for (int k = 0; k < cw; k += 8) {           // 128-byte lines
      prefetch_l2(E4 + off + k); prefetch_l2(M4 + off + k); prefetch_l2(V4 + off + k);
    }
  }
  const uint32_t sb = (uint32_t)cw * 16u;
  if (lane == 0) {
    bar_init(bar);
    bar_expect(bar, (uint32_t)__popc(rep_mask) * sb);
  }
  __syncwarp();
  if (EARLY) KG_GRID_DEP_WAIT();
  if (rep) bulk_g2s(sm + lane * sw, X4 + (int64_t)pj * d4 + c0, sb, bar);   // slot j = position j
  const bool upd = apply && !(flags[0] | flags[1]);
  const float lr1 = *lr_dev * bc[0], ibc2 = bc[1];
  bar_wait0(bar);
  SA_T(2);
  // (1) pieces in position order: single-piece segments take their update now; the pieces
  // of longer segments go to PS, and the item completing a segment's last piece keeps it
  int pend_u[2] = {0, 0}, pend_s0[2] = {0, 0}, pend_s1[2] = {0, 0}, npend = 0;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int jst = 0;
  for (int j = 0; j < n; ++j) {
    if (!((rep_mask >> j) & 1u)) continue;
    const float4 xv = cv ? sm[j * sw + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    if ((start_mask >> j) & 1u) { acc = xv; jst = j; }
    else add4(acc, xv);
    if (!((end_mask >> j) & 1u)) continue;
    const int u = __shfl_sync(0xffffffffu, uj, jst), s0 = __shfl_sync(0xffffffffu, s0j, jst),
              s1 = __shfl_sync(0xffffffffu, s1j, jst);
    const int64_t key = __shfl_sync(0xffffffffu, kj, jst);
    const int npieces = (s1 - 1) / kPiece - s0 / kPiece + 1;
    if (npieces > 1) {
      if (cv) __stcg(P4 + (int64_t)(base + jst) * d4 + col, acc);
      __threadfence();
      __syncwarp();
      int last = 0;
      if (lane == 0) last = atomicAdd(cnt + (int64_t)u * kSlices + q, 1) == npieces - 1;
      if (__shfl_sync(0xffffffffu, last, 0)) {   // at most 2 per chunk: its first and last run
        if (npend == 0) { pend_u[0] = u; pend_s0[0] = s0; pend_s1[0] = s1; }
        else { pend_u[1] = u; pend_s0[1] = s0; pend_s1[1] = s1; }
        ++npend;
      }
      continue;
    }
    if (!cv) continue;
    if (GO4) GO4[(int64_t)u * d4 + col] = acc;
    if (!upd) continue;
    const int64_t off = (key / world) * d4 + col;
    float4 P = E4[off], Mm = M4[off], V = V4[off];
    adam4(P, Mm, V, acc, lr1, hy, ibc2);
    E4[off] = P; M4[off] = Mm; V4[off] = V;
  }
  // (2) the segments completed here: all pieces' sums (kB in flight), added in ascending
  // order, then Adam on the slice
  SA_T(3);
  if (!npend) return;
  __threadfence();
  for (int pi = 0; pi < npend; ++pi) {
    const int u = pi ? pend_u[1] : pend_u[0], s0 = pi ? pend_s0[1] : pend_s0[0], s1 = pi ? pend_s1[1] : pend_s1[0];
    if (lane == 0) cnt[(int64_t)u * kSlices + q] = 0;       // ready for the next step
    if (!cv) continue;
    const int64_t off = (uniq[u] / world) * d4 + col;
    float4 P, Mm, V;
    if (upd) { P = E4[off]; Mm = M4[off]; V = V4[off]; }  // the row's slice in flight first
    float4 G = __ldcg(P4 + (int64_t)s0 * d4 + col);
    constexpr int kB = 8;
    for (int sp = (s0 / kPiece + 1) * kPiece; sp < s1; sp += kB * kPiece) {
      const int nk = min(kB, (s1 - sp + kPiece - 1) / kPiece);
      float4 y[kB];
#pragma unroll
      for (int k = 0; k < kB; ++k)
        y[k] = k < nk ? __ldcg(P4 + (int64_t)(sp + k * kPiece) * d4 + col) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < kB; ++k)
        if (k < nk) add4(G, y[k]);
    }
    if (GO4) GO4[(int64_t)u * d4 + col] = G;
    if (!upd) continue;
    adam4(P, Mm, V, G, lr1, hy, ibc2);
    E4[off] = P; M4[off] = Mm; V4[off] = V;
  }
}

// cnt: [L][kSlices] int32, zero before the first call (the kernel leaves it zero).
void launch_sparse_adam(const int64_t *uniq, const int32_t *seg, const int32_t *perm, const int32_t *sinv,
                        const int32_t *hrow, const int32_t *U_dev, int L, const float *OG, float *PS, int32_t *cnt,
                        int d, int world, float *ent, float *m, float *v, float *grad_out, const float *lr,
                        double beta1, double beta2, double eps, const float *bc, const int *flags, int apply,
                        cudaStream_t st, int64_t skip_key, int early) {
  if (L <= 0) return;
  const AdamHyper hy = hyper(beta1, beta2, eps);
  const int d4 = d / 4;
  const int ns = (d4 + 31) / 32, sw = (d4 + ns - 1) / ns;        // slices of <= 32 float4
  const int wbytes = (int)((std::max(4 * d4, kPiece * sw) * 16 + 127) / 128 * 128);
  const int items = (L + kPiece - 1) / kPiece * ns + L;
  const int smem = 4 * wbytes;
  auto kern = early ? sparse_adam_fused_kernel<true> : sparse_adam_fused_kernel<false>;
  static int configured[2] = {0, 0};   // the largest dynamic smem opted into, per instantiation
  int &cfg = configured[early ? 1 : 0];
  if (smem > 48 * 1024 && smem > cfg) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cfg = smem;
  }
  kern<<<(items + 3) / 4, 128, smem, st>>>(uniq, seg, perm, sinv, hrow, U_dev, L, OG, PS, cnt, d, world, ns, sw,
                                           wbytes, ent, m, v, grad_out, lr, hy, bc, flags, apply, skip_key);
  ++g_launches;
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
  if (flags[0] | flags[1]) return;   // flags[1]: a failure found after the loss check (p2p barrier)
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
  if (flags[0] | flags[1]) return;   // flags[1]: a failure found after the loss check (p2p barrier)
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
  if (flags[0] | flags[1]) return;   // flags[1]: a failure found after the loss check (p2p barrier)
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
// Every bias gradient of one DAG node in one launch (blockIdx.y = job): the same per-column
// fixed-order sums as colsum_kernel.
__global__ void __launch_bounds__(1024) colsum_multi_kernel(ColsumJobs J) {
  KG_GRID_DEP_WAIT();
  __shared__ float red[32][33];
  const ColsumJob &jb = J.j[blockIdx.y];
  const int cx = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cx;
  if (blockIdx.x * 32 >= jb.cols) return;
  float s = 0.f;
  if (c < jb.cols)
    for (int r = ry; r < jb.rows; r += 32) s += jb.X[(int64_t)r * jb.ld + c];
  red[ry][cx] = s;
  __syncthreads();
  if (ry == 0 && c < jb.cols) {
    float t = 0.f;
    for (int k = 0; k < 32; ++k) t += red[k][cx];
    jb.out[c] = t;
  }
}
void launch_colsum_multi(const ColsumJobs &J, cudaStream_t st) {
  if (J.n <= 0) return;
  int mc = 0;
  for (int i = 0; i < J.n; ++i) mc = std::max(mc, J.j[i].cols);
  { colsum_multi_kernel<<<dim3((mc + 31) / 32, J.n), 1024, 0, st>>>(J); ++g_launches; }
}

}  // namespace kg
