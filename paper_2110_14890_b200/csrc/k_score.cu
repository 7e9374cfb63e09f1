// k_score.cu -- shared-negative scoring, Eq. 1 loss and the scoring backward.
//
// PAPER.md §4.3: M queries x |N| shared negatives, "M x |N| pairs of
// distances ... box or beta ... KL divergence ... customized CUDA kernel ...
// operation fusion"; Eq. 1; Dist per Table 1 and
// Table 2; DNF min over disjuncts (A11).
//
// Three CUDA-core "generalised GEMM" kernels, all deterministic (no atomics):
//   pair_fwd   out (i, j), reduce over units k:  D_ij, Eq. 1 epilogue -> per-pair
//              adjoint coefficient C[t][i][j], loss partials per (j-tile, i)
//   pair_bwd_q out (r, k), reduce over pool j:   dQ[r][k] += sum_j C_rj dD/dq_rk
//   pair_bwd_v out (j, k), reduce over rows r:   dV[j][k]  = sum_r C_rj dD/dv_jk
// plus the per-query positive kernel (D+, its adjoint, its gradients) and the
// BetaE digamma / lgamma precomputations.
//
// Feature layout (A1): row r of Q holds QF features of U units each,
// Q[r][f*U + k]; raw entity rows are d floats; the BetaE entity feature row is
// 9 planes of m = d/2: [Pa | Pb | A | B | TA | TB | TAB | GA | GB] with
// A = e(x_alpha), B = e(x_beta), Pa = psi(A) - psi(A+B), Pb = psi(B) - psi(A+B),
// TA = psi'(A), TB = psi'(B), TAB = psi'(A+B), GA/GB = d e / d x (clamp mask).
#include <algorithm>
#include <type_traits>

#include <climits>
#include <cstdlib>

#include "kg_common.cuh"
#include "kg_launch.h"

namespace kg {

// ---------------------------------------------------------------- models
struct ML2 {   // GQE, TransE: ||q - v||_2 (A2)
  static constexpr bool kRowAlpha = false;
  static constexpr int QF = 1, EF = 1, EOFF = 0, BQ_EF = 1, BQ_EOFF = 0, BV_EF = 1, BV_EOFF = 0, AV = 1, OUTF = 1;
  static constexpr bool kL2 = true, kBeta = false;
  __device__ static float acc(const float *q, const float *e, float) { const float t = q[0] - e[0]; return t * t; }
  __device__ static float fin(float s, float, float) { return sqrtf(s); }
  __device__ static void bq(const float *q, const float *e, float c, float, float *dq) { dq[0] += c * (q[0] - e[0]); }
  __device__ static void bv(const float *q, const float *e, float c, float, float *a) { a[0] += c * (e[0] - q[0]); }
  // fused backward: dq += dD/dq * C, dv += dD/dv * C   (C here is c_ij / D_ij, A2 adjoint)
  static constexpr int BF = 1, BOFF = 0, BQF = QF;
  __device__ static void grad(const float *q, const float *e, float c, float, float *dq, float *dv) {
    const float ct = c * (q[0] - e[0]);
    dq[0] += ct;
    dv[0] -= ct;
  }
};
struct MBox {  // Q2B: sum ReLU(|v-c| - o) + alpha * min(|v-c|, o) (A7)
  static constexpr bool kRowAlpha = true;   // dq[1] += alpha * sum_j c after the j loop
  static constexpr int QF = 2, EF = 1, EOFF = 0, BQ_EF = 1, BQ_EOFF = 0, BV_EF = 1, BV_EOFF = 0, AV = 1, OUTF = 1;
  static constexpr bool kL2 = false, kBeta = false;
  // ReLU(d - o) + alpha min(d, o) = d + (alpha - 1) min(d, o), d = |v - c| (o >= 0)
  __device__ static float acc(const float *q, const float *e, float al) {
    const float dl = fabsf(e[0] - q[0]);
    return fmaf(al - 1.f, fminf(dl, q[1]), dl);
  }
  __device__ static float fin(float s, float, float) { return s; }
  __device__ static void bq(const float *q, const float *e, float c, float al, float *dq) {
    const float dl = e[0] - q[0], a = fabsf(dl), o = q[1];
    const float s = (dl > 0.f) ? 1.f : ((dl < 0.f) ? -1.f : 0.f);
    const float outb = a > o ? 1.f : 0.f, inb = a < o ? 1.f : 0.f;
    dq[0] -= c * s * (outb + al * inb);                 // dD/dc = -s([a>o] + alpha[a<o])
    dq[1] += c * (-outb + al * (a >= o ? 1.f : 0.f));   // dD/do = -[a>o] + alpha[a>=o]  (A19)
  }
  __device__ static void bv(const float *q, const float *e, float c, float al, float *acc_) {
    const float dl = e[0] - q[0], a = fabsf(dl), o = q[1];
    const float s = (dl > 0.f) ? 1.f : ((dl < 0.f) ? -1.f : 0.f);
    acc_[0] += c * s * ((a > o ? 1.f : 0.f) + al * (a < o ? 1.f : 0.f));
  }
  static constexpr int BF = 1, BOFF = 0, BQF = QF;
  __device__ static void grad(const float *q, const float *e, float c, float al, float *dq, float *dv) {
    // t = v - c, a = |t|, W = [a > o] + alpha [a < o]:  dD/dv = sign(t) W (sign(0) = 0),
    // dD/dc = -dD/dv, dD/do = alpha - W (= alpha - 1 | 0 | alpha for a > o | a < o | a == o);
    // the alpha * c part of dD/do is added once per row by the caller (A7, A19).
    const float t = e[0] - q[0], a = fabsf(t), o = q[1];
    const float W = (a > o) ? 1.f : ((a < o) ? al : 0.f);
    const float cw = c * W;
    const float cg = (t == 0.f) ? 0.f : __int_as_float(__float_as_int(cw) ^ (__float_as_int(t) & 0x80000000));
    dq[0] -= cg;
    dv[0] += cg;
    dq[1] -= cw;
  }
};
struct MBeta {  // KL(Beta(entity) || Beta(query)) summed over m (A10), direct per-unit differences (A22)
  static constexpr bool kRowAlpha = false;
  static constexpr int QF = 2, EF = 4, EOFF = 0, BQ_EF = 2, BQ_EOFF = 0, BV_EF = 7, BV_EOFF = 2, AV = 2, OUTF = 2;
  static constexpr bool kL2 = false, kBeta = true;
  // e = [Pa, Pb, A, B]
  __device__ static float acc(const float *q, const float *e, float) { return (e[2] - q[0]) * e[0] + (e[3] - q[1]) * e[1]; }
  __device__ static float fin(float s, float cq, float cv) { return s + cq - cv; }
  __device__ static void bq(const float *, const float *e, float c, float, float *dq) { dq[0] -= c * e[0]; dq[1] -= c * e[1]; }
  __device__ static void bv(const float *q, const float *, float c, float, float *a) { a[0] += c * q[0]; a[1] += c * q[1]; }
  // Backward on per-term differences (no cancellation of large sums, A22):
  // q = [a2, b2, QPa, QPb] (query Beta and its psi(a2) - psi(a2+b2), psi(b2) - psi(a2+b2)),
  // e = [Pa, Pb, A, B] (the same for the entity):  dKL/da2 = QPa - Pa, dKL/db2 = QPb - Pb;
  // dv accumulates sum C (A - a2), sum C (B - b2) (trigamma epilogue in the combine kernel).
  static constexpr int BF = 4, BOFF = 0, BQF = 4;
  __device__ static void grad(const float *q, const float *e, float c, float, float *dq, float *dv) {
    dq[0] = fmaf(c, q[2] - e[0], dq[0]);
    dq[1] = fmaf(c, q[3] - e[1], dq[1]);
    dv[0] = fmaf(c, e[2] - q[0], dv[0]);
    dv[1] = fmaf(c, e[3] - q[1], dv[1]);
  }
};
// MUFU.RSQ without the denormal-input fixup of rsqrtf (4 extra instructions per call); every
// caller passes s >= 1e-30 (normal) or discards the result for s <= 1e-30, where |z| < 1e-15 --
// not reachable by differences of non-equal floats of the embeddings' magnitude (~0.1)
__device__ __forceinline__ float rsqrt_n(float s) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s));
  return r;
}
struct MRot {  // RotatE: sum_k |q_k - t_k| (A3)
  static constexpr bool kRowAlpha = false;
  static constexpr int QF = 2, EF = 2, EOFF = 0, BQ_EF = 2, BQ_EOFF = 0, BV_EF = 2, BV_EOFF = 0, AV = 2, OUTF = 2;
  static constexpr bool kL2 = false, kBeta = false;
  // |z| = s * rsqrt(s), s = |z|^2 (MUFU.RSQ, <= 2 ulp: ~3e-7 relative per unit, far inside the
  // 1e-5 bar; the IEEE sqrtf / division sequences made RotatE's pair kernels 3x more instructions)
  __device__ static float acc(const float *q, const float *e, float) {
    const float a = q[0] - e[0], b = q[1] - e[1], s = fmaf(a, a, b * b);
    return s * rsqrt_n(fmaxf(s, 1e-30f));
  }
  __device__ static float fin(float s, float, float) { return s; }
  __device__ static void bq(const float *q, const float *e, float c, float, float *dq) {
    const float a = q[0] - e[0], b = q[1] - e[1], n = sqrtf(a * a + b * b);
    if (n > 0.f) { const float w = c / n; dq[0] += w * a; dq[1] += w * b; }
  }
  __device__ static void bv(const float *q, const float *e, float c, float, float *acc_) {
    const float a = q[0] - e[0], b = q[1] - e[1], n = sqrtf(a * a + b * b);
    if (n > 0.f) { const float w = c / n; acc_[0] -= w * a; acc_[1] -= w * b; }
  }
  static constexpr int BF = 2, BOFF = 0, BQF = QF;
  __device__ static void grad(const float *q, const float *e, float c, float, float *dq, float *dv) {
    const float a = q[0] - e[0], b = q[1] - e[1], s = fmaf(a, a, b * b);
    const float w = s > 1e-30f ? c * rsqrt_n(s) : 0.f;              // c / |z| (A19: 0 at z = 0)
    dq[0] += w * a; dq[1] += w * b;
    dv[0] -= w * a; dv[1] -= w * b;
  }
};
struct MDot {  // DistMult: -<q, t> (A13)
  static constexpr bool kRowAlpha = false;
  static constexpr int QF = 1, EF = 1, EOFF = 0, BQ_EF = 1, BQ_EOFF = 0, BV_EF = 1, BV_EOFF = 0, AV = 1, OUTF = 1;
  static constexpr bool kL2 = false, kBeta = false;
  __device__ static float acc(const float *q, const float *e, float) { return q[0] * e[0]; }
  __device__ static float fin(float s, float, float) { return -s; }
  __device__ static void bq(const float *, const float *e, float c, float, float *dq) { dq[0] -= c * e[0]; }
  __device__ static void bv(const float *q, const float *, float c, float, float *a) { a[0] -= c * q[0]; }
  static constexpr int BF = 1, BOFF = 0, BQF = QF;
  __device__ static void grad(const float *q, const float *e, float c, float, float *dq, float *dv) {
    dq[0] -= c * e[0];
    dv[0] -= c * q[0];
  }
};
struct MCpx {  // ComplEx: -Re<q, conj(t)> = -sum(q_re t_re + q_im t_im) (A13)
  static constexpr bool kRowAlpha = false;
  static constexpr int QF = 2, EF = 2, EOFF = 0, BQ_EF = 2, BQ_EOFF = 0, BV_EF = 2, BV_EOFF = 0, AV = 2, OUTF = 2;
  static constexpr bool kL2 = false, kBeta = false;
  __device__ static float acc(const float *q, const float *e, float) { return q[0] * e[0] + q[1] * e[1]; }
  __device__ static float fin(float s, float, float) { return -s; }
  __device__ static void bq(const float *, const float *e, float c, float, float *dq) { dq[0] -= c * e[0]; dq[1] -= c * e[1]; }
  __device__ static void bv(const float *q, const float *, float c, float, float *a) { a[0] -= c * q[0]; a[1] -= c * q[1]; }
  static constexpr int BF = 2, BOFF = 0, BQF = QF;
  __device__ static void grad(const float *q, const float *e, float c, float, float *dq, float *dv) {
    dq[0] -= c * e[0]; dq[1] -= c * e[1];
    dv[0] -= c * q[0]; dv[1] -= c * q[1];
  }
};

__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }

// ---------------------------------------------------------------- pair_fwd (partial)
// Tile 64 queries x 64 candidates, 256 threads (4x4 pairs each), units in chunks of
// 16 staged in shared memory.  blockIdx.z selects a contiguous range of units
// (split reduction: more CTAs than the 148 SMs even at B = 512); the raw partial
// sums go to Dpart[z][t][i][j] and pair_epi_kernel adds them in the fixed order z.
// (A balanced one-wave schedule -- each CTA an equal run of (tile, chunk) items, a tile's
// partials in a variable number of slots -- measured slower: C5-q2b 40 -> 47 us; likewise
// for pair_bwd_kernel, 0.142 -> 0.147 ms per step.)
// resident CTAs per SM of pair_fwd (KG_FWD_OCC4=1: 4 for the single-output Q2B box kernel, i.e.
// <= 64 registers: measured slower, C5-q2b scoring forward 57 -> 59 us, as was 3 per SM at 79
// registers, 54 -> 54.4 us; the default lets the compiler take 102 registers, 2 per SM)
#ifndef KG_FWD_OCC4
#define KG_FWD_OCC4 0
#endif
template <class Mdl, int NOUT> struct kFwdOcc {
  // (the two-output DNF-union kernel at 2 per SM, <= 128 registers: neutral, 92.6 vs 92.4 us)
  static constexpr int v = (KG_FWD_OCC4 && NOUT == 1 && std::is_same<Mdl, MBox>::value) ? 4 : 1;
};
template <class Mdl, int NOUT>
__global__ void __launch_bounds__(256, kFwdOcc<Mdl, NOUT>::v) pair_fwd_kernel(ScoreArgs a) {
  KG_GRID_DEP_WAIT();
  // thread (tx, ty) owns queries i0 + 4*ty + x and candidates j0 + 4*tx + b (x, b < 4):
  // one 128-bit shared load per operand row per unit.
  constexpr int BI = 64, BJ = 64, KC = 16, PAD = 4;
  // double-buffered staging (the small 1-output models): chunk c + 1 is loaded into registers
  // while chunk c is computed; otherwise one buffer and a barrier after the compute
  constexpr bool DB = NOUT == 1 && Mdl::QF * (BI + PAD) + Mdl::EF * (BJ + PAD) <= 3 * 68;
  constexpr int NB = DB ? 2 : 1;
  __shared__ __align__(16) float sQ2[NB][NOUT][Mdl::QF][KC][BI + PAD];
  __shared__ __align__(16) float sE2[NB][Mdl::EF][KC][BJ + PAD];
  __shared__ int64_t sRow[BJ];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int i0 = blockIdx.y * BI, j0 = blockIdx.x * BJ;
  const int M = a.M, K = a.K, U = a.U;
  const int qstride = Mdl::QF * U;
  const int ku0 = blockIdx.z * a.ups, ku1 = min(U, ku0 + a.ups);
  if (t < BJ) {
    const int j = j0 + t;
    sRow[t] = (j < K) ? (a.eidx ? a.eidx[j] : (int64_t)j) : 0;
  }
  float acc[NOUT][4][4];
#pragma unroll
  for (int tt = 0; tt < NOUT; ++tt)
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[tt][x][y] = 0.f;
  float2 s1[NOUT][4][2], s2[NOUT][4][2];   // Q2B: sum |t| and sum min(|t|, o) per candidate pair
#pragma unroll
  for (int tt = 0; tt < NOUT; ++tt)
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) s1[tt][x][y] = s2[tt][x][y] = make_float2(0.f, 0.f);
  __syncthreads();

  constexpr int NQ4 = NOUT * Mdl::QF * BI * (KC / 4), NE4 = Mdl::EF * BJ * (KC / 4);
  constexpr int RQ = (NQ4 + 255) / 256, RE = (NE4 + 255) / 256;
  float4 rq[RQ], re[RE];
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int r = 0; r < RQ; ++r) {
      const int e = t + 256 * r;
      rq[r] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e >= NQ4) continue;
      const int q4 = e % (KC / 4);
      int rest = e / (KC / 4);
      const int row = rest % BI; rest /= BI;
      const int f = rest % Mdl::QF, tt = rest / Mdl::QF;
      const int i = i0 + row, k = k0 + q4 * 4;
      if (i < M && k < ku1) rq[r] = ld4(a.Q + (size_t)(tt * M + i) * qstride + f * U + k);
    }
#pragma unroll
    for (int r = 0; r < RE; ++r) {
      const int e = t + 256 * r;
      re[r] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e >= NE4) continue;
      const int q4 = e % (KC / 4);
      const int rest = e / (KC / 4);
      const int row = rest % BJ, f = rest / BJ;
      const int j = j0 + row, k = k0 + q4 * 4;
      if (j < K && k < ku1) re[r] = ld4(a.E + sRow[row] * a.estride + (Mdl::EOFF + f) * U + k);
    }
  };
  auto store_chunk = [&](int buf) {
#pragma unroll
    for (int r = 0; r < RQ; ++r) {
      const int e = t + 256 * r;
      if (e >= NQ4) continue;
      const int q4 = e % (KC / 4);
      int rest = e / (KC / 4);
      const int row = rest % BI; rest /= BI;
      const int f = rest % Mdl::QF, tt = rest / Mdl::QF;
      sQ2[buf][tt][f][q4 * 4 + 0][row] = rq[r].x; sQ2[buf][tt][f][q4 * 4 + 1][row] = rq[r].y;
      sQ2[buf][tt][f][q4 * 4 + 2][row] = rq[r].z; sQ2[buf][tt][f][q4 * 4 + 3][row] = rq[r].w;
    }
#pragma unroll
    for (int r = 0; r < RE; ++r) {
      const int e = t + 256 * r;
      if (e >= NE4) continue;
      const int q4 = e % (KC / 4);
      const int rest = e / (KC / 4);
      const int row = rest % BJ, f = rest / BJ;
      sE2[buf][f][q4 * 4 + 0][row] = re[r].x; sE2[buf][f][q4 * 4 + 1][row] = re[r].y;
      sE2[buf][f][q4 * 4 + 2][row] = re[r].z; sE2[buf][f][q4 * 4 + 3][row] = re[r].w;
    }
  };
  if (DB && ku0 < ku1) load_chunk(ku0);
  int buf = 0;
  for (int k0 = ku0; k0 < ku1; k0 += KC, buf = DB ? buf ^ 1 : 0) {
    if (!DB) load_chunk(k0);
    store_chunk(buf);
    __syncthreads();   // chunk visible; (DB) every thread is past the compute of chunk - 2
    if (DB && k0 + KC < ku1) load_chunk(k0 + KC);
    auto &sQ = sQ2[buf];
    auto &sE = sE2[buf];
    if constexpr (std::is_same<Mdl, MBox>::value) {
      // Q2B: D = sum |t| + (alpha - 1) sum min(|t|, o), t = v - c, on packed f32x2 pairs of
      // candidates (FADD2 with |.| operands): 2.5 instructions per (query, candidate, unit)
#pragma unroll 4
      for (int kk = 0; kk < KC; ++kk) {
        const float4 v = *reinterpret_cast<const float4 *>(&sE[0][kk][4 * tx]);
        const float2 e01 = make_float2(v.x, v.y), e23 = make_float2(v.z, v.w);
#pragma unroll
        for (int tt = 0; tt < NOUT; ++tt) {
          const float4 cq = *reinterpret_cast<const float4 *>(&sQ[tt][0][kk][4 * ty]);
          const float4 oq = *reinterpret_cast<const float4 *>(&sQ[tt][1][kk][4 * ty]);
          const float cs[4] = {cq.x, cq.y, cq.z, cq.w}, os[4] = {oq.x, oq.y, oq.z, oq.w};
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const float2 cc = make_float2(-cs[x], -cs[x]);
            const float2 t0 = __fadd2_rn(e01, cc), t1 = __fadd2_rn(e23, cc);
            const float2 a0 = make_float2(fabsf(t0.x), fabsf(t0.y)), a1 = make_float2(fabsf(t1.x), fabsf(t1.y));
            s1[tt][x][0] = __fadd2_rn(s1[tt][x][0], a0);
            s1[tt][x][1] = __fadd2_rn(s1[tt][x][1], a1);
            s2[tt][x][0] = __fadd2_rn(s2[tt][x][0], make_float2(fminf(a0.x, os[x]), fminf(a0.y, os[x])));
            s2[tt][x][1] = __fadd2_rn(s2[tt][x][1], make_float2(fminf(a1.x, os[x]), fminf(a1.y, os[x])));
          }
        }
      }
    } else if constexpr (std::is_same<Mdl, MRot>::value) {
      // RotatE on packed f32x2 pairs of candidates: |q - t| = s rsqrt(s), s = a^2 + b^2 (the
      // generic path's arithmetic, two candidates per instruction; the MUFU.RSQ bounds it)
#pragma unroll 4
      for (int kk = 0; kk < KC; ++kk) {
        const float4 er = *reinterpret_cast<const float4 *>(&sE[0][kk][4 * tx]);
        const float4 ei = *reinterpret_cast<const float4 *>(&sE[1][kk][4 * tx]);
        const float2 er01 = make_float2(-er.x, -er.y), er23 = make_float2(-er.z, -er.w);
        const float2 ei01 = make_float2(-ei.x, -ei.y), ei23 = make_float2(-ei.z, -ei.w);
#pragma unroll
        for (int tt = 0; tt < NOUT; ++tt) {
          const float4 qr = *reinterpret_cast<const float4 *>(&sQ[tt][0][kk][4 * ty]);
          const float4 qi = *reinterpret_cast<const float4 *>(&sQ[tt][1][kk][4 * ty]);
          const float qrs[4] = {qr.x, qr.y, qr.z, qr.w}, qis[4] = {qi.x, qi.y, qi.z, qi.w};
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const float2 qre = make_float2(qrs[x], qrs[x]), qim = make_float2(qis[x], qis[x]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const float2 a2 = __fadd2_rn(qre, h ? er23 : er01), b2 = __fadd2_rn(qim, h ? ei23 : ei01);
              const float2 s2 = __ffma2_rn(a2, a2, __fmul2_rn(b2, b2));
              const float2 r2 = make_float2(rsqrt_n(fmaxf(s2.x, 1e-30f)), rsqrt_n(fmaxf(s2.y, 1e-30f)));
              const float2 d2 = __fmul2_rn(s2, r2);
              const float2 o = __fadd2_rn(make_float2(acc[tt][x][2 * h], acc[tt][x][2 * h + 1]), d2);
              acc[tt][x][2 * h] = o.x;
              acc[tt][x][2 * h + 1] = o.y;
            }
          }
        }
      }
    } else {
#pragma unroll 4
      for (int kk = 0; kk < KC; ++kk) {
        float ev[4][Mdl::EF];
#pragma unroll
        for (int f = 0; f < Mdl::EF; ++f) {
          const float4 v = *reinterpret_cast<const float4 *>(&sE[f][kk][4 * tx]);
          ev[0][f] = v.x; ev[1][f] = v.y; ev[2][f] = v.z; ev[3][f] = v.w;
        }
#pragma unroll
        for (int tt = 0; tt < NOUT; ++tt) {
          float qv[4][Mdl::QF];
#pragma unroll
          for (int f = 0; f < Mdl::QF; ++f) {
            const float4 v = *reinterpret_cast<const float4 *>(&sQ[tt][f][kk][4 * ty]);
            qv[0][f] = v.x; qv[1][f] = v.y; qv[2][f] = v.z; qv[3][f] = v.w;
          }
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[tt][x][b] += Mdl::acc(qv[x], ev[b], a.alpha);
        }
      }
    }
    if (!DB) __syncthreads();
  }
  if constexpr (std::is_same<Mdl, MBox>::value) {
#pragma unroll
    for (int tt = 0; tt < NOUT; ++tt)
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        acc[tt][x][0] = fmaf(a.alpha - 1.f, s2[tt][x][0].x, s1[tt][x][0].x);
        acc[tt][x][1] = fmaf(a.alpha - 1.f, s2[tt][x][0].y, s1[tt][x][0].y);
        acc[tt][x][2] = fmaf(a.alpha - 1.f, s2[tt][x][1].x, s1[tt][x][1].x);
        acc[tt][x][3] = fmaf(a.alpha - 1.f, s2[tt][x][1].y, s1[tt][x][1].y);
      }
  }
  float *out = a.Dpart + (size_t)blockIdx.z * NOUT * M * a.Kp;
  const int jb = j0 + 4 * tx;
#pragma unroll
  for (int tt = 0; tt < NOUT; ++tt)
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int i = i0 + 4 * ty + x;
      if (i >= M) continue;
      float *o = out + (size_t)(tt * M + i) * a.Kp + jb;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (jb + b < K) o[b] = acc[tt][x][b];
    }
}

// ---------------------------------------------------------------- pair epilogue
// One CTA per query i: D_t = fin(sum_z Dpart), DNF min (A11), Eq. 1 adjoint
// coefficients C[t][i][j] (train) or distances (score), the row's negative loss
// term and sum_j C (BetaE), all reduced in a fixed order.
template <class Mdl, int NOUT, bool TRAIN>
__global__ void __launch_bounds__(256) pair_epi_kernel(ScoreArgs a) {
  KG_GRID_DEP_WAIT();
  __shared__ float red[32];
  const int i = blockIdx.x, M = a.M, K = a.K;
  const size_t zs = (size_t)NOUT * M * a.Kp;
  float inv_n = 0.f;
  if (TRAIN) {
    float n = 0.f;
    for (int w = threadIdx.x; w < a.W; w += blockDim.x) {
      uint32_t bits = a.mask[(size_t)i * a.W + w];
      if (w == a.W - 1 && (K & 31)) bits &= (1u << (K & 31)) - 1u;   // padding bits j >= K are not negatives
      n += (float)__popc(bits);
    }
    n = block_sum(n, red);
    inv_n = n > 0.f ? 1.f / n : 0.f;
  }
  float lsum = 0.f, csum[NOUT];
#pragma unroll
  for (int tt = 0; tt < NOUT; ++tt) csum[tt] = 0.f;
  const int jend = TRAIN ? a.Kp : K;
  if (TRAIN && !(K & 3) && !(a.Kp & 3) && (a.Dmin == nullptr)) {
    // 4 consecutive candidates per thread (float4 loads of the partials and stores of C); the
    // per-pair arithmetic is the scalar loop's below
    const float4 *Dp = reinterpret_cast<const float4 *>(a.Dpart);
    for (int j4 = threadIdx.x; j4 * 4 < jend; j4 += blockDim.x) {
      const int j0 = j4 * 4;
      float4 D4[NOUT];
#pragma unroll
      for (int tt = 0; tt < NOUT; ++tt) {
        const size_t base = ((size_t)(tt * M + i) * a.Kp + j0) / 4;
        float4 s4 = Dp[base];
        for (int z = 1; z < a.KS; ++z) {
          const float4 q = Dp[z * zs / 4 + base];
          s4.x += q.x; s4.y += q.y; s4.z += q.z; s4.w += q.w;
        }
        const float cq = Mdl::kBeta ? a.Cq[tt * M + i] : 0.f;
        float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
        if (Mdl::kBeta && j0 < K) cv = *reinterpret_cast<const float4 *>(a.Cv + j0);   // K % 4 == 0
        D4[tt] = make_float4(Mdl::fin(s4.x, cq, cv.x), Mdl::fin(s4.y, cq, cv.y), Mdl::fin(s4.z, cq, cv.z),
                             Mdl::fin(s4.w, cq, cv.w));
      }
      const uint32_t word = j0 < K ? a.mask[(size_t)i * a.W + (j0 >> 5)] : 0u;
      float cf[NOUT][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u;
        float D[NOUT];
#pragma unroll
        for (int tt = 0; tt < NOUT; ++tt) D[tt] = u == 0 ? D4[tt].x : u == 1 ? D4[tt].y : u == 2 ? D4[tt].z : D4[tt].w;
        int tm = 0;
        float Dm = D[0];
        if (NOUT == 2 && D[1] < D[0]) { tm = 1; Dm = D[1]; }   // DNF min, ties -> lowest (A11)
        float c = 0.f;
        if (j < K && ((word >> (j & 31)) & 1u)) {
          c = -sigm_(a.gamma - Dm) * inv_n * a.scale;         // dl/dD_ij of Eq. 1 (A12)
          lsum += softplusf_(a.gamma - Dm) * inv_n;
        }
#pragma unroll
        for (int tt = 0; tt < NOUT; ++tt) {
          float coef = (tt == tm) ? c : 0.f;
          csum[tt] += coef;
          if (Mdl::kL2) coef = (coef != 0.f && D[tt] > 0.f) ? coef / D[tt] : 0.f;
          cf[tt][u] = coef;
        }
      }
#pragma unroll
      for (int tt = 0; tt < NOUT; ++tt)
        *reinterpret_cast<float4 *>(a.C + (size_t)(tt * M + i) * a.Kp + j0) = make_float4(cf[tt][0], cf[tt][1], cf[tt][2], cf[tt][3]);
    }
  } else
  for (int j = threadIdx.x; j < jend; j += blockDim.x) {
    if (j >= K) {
#pragma unroll
      for (int tt = 0; tt < NOUT; ++tt) a.C[(size_t)(tt * M + i) * a.Kp + j] = 0.f;
      continue;
    }
    float D[NOUT];
#pragma unroll
    for (int tt = 0; tt < NOUT; ++tt) {
      float s = 0.f;
      for (int z = 0; z < a.KS; ++z) s += a.Dpart[z * zs + (size_t)(tt * M + i) * a.Kp + j];
      D[tt] = Mdl::fin(s, Mdl::kBeta ? a.Cq[tt * M + i] : 0.f, Mdl::kBeta ? a.Cv[j] : 0.f);
    }
    int tm = 0;
    float Dm = D[0];
    if (NOUT == 2 && D[1] < D[0]) { tm = 1; Dm = D[1]; }   // DNF min, ties -> lowest (A11)
    if (TRAIN) {
      const bool bit = (a.mask[(size_t)i * a.W + (j >> 5)] >> (j & 31)) & 1u;
      float c = 0.f;
      if (bit) {
        c = -sigm_(a.gamma - Dm) * inv_n * a.scale;         // dl/dD_ij of Eq. 1 (A12)
        lsum += softplusf_(a.gamma - Dm) * inv_n;
      }
#pragma unroll
      for (int tt = 0; tt < NOUT; ++tt) {
        float coef = (tt == tm) ? c : 0.f;
        csum[tt] += coef;
        if (Mdl::kL2) coef = (coef != 0.f && D[tt] > 0.f) ? coef / D[tt] : 0.f;
        a.C[(size_t)(tt * M + i) * a.Kp + j] = coef;
      }
      if (a.Dmin) a.Dmin[(size_t)i * K + j] = Dm;
    } else {
      a.Dmin[(size_t)i * a.ldo + j] = Dm;
    }
  }
  if (TRAIN) {
    lsum = block_sum(lsum, red);
    if (threadIdx.x == 0) a.loss_part[i] = lsum;
    if (Mdl::kBeta || Mdl::kRowAlpha) {   // row sums of C: BetaE psi terms, Q2B alpha * sum_j c (dD/do)
#pragma unroll
      for (int tt = 0; tt < NOUT; ++tt) {
        const float s = block_sum(csum[tt], red);
        if (threadIdx.x == 0) a.Csum[tt * M + i] = s;
      }
    }
  }
}

// ---------------------------------------------------------------- fused scoring backward
// One pass over the (query row r, pool entry j, unit k) terms computes both
// reductions: dQ[r][k] = sum_j C_rj dD/dq and dV[j][k] = sum_r C_rj dD/dv.
// Lanes = 32 consecutive units k; warp w of the CTA owns JW = 16 pool entries
// (their entity features and their dV accumulators live in registers for the
// whole row range); each row's dQ partial over the warp's entries is combined
// across the NW warps in shared memory in a fixed order and written once per
// (row, j-block of NW*JW).  blockIdx.z splits the rows; all partial sums are
// added by the combine kernels in a fixed order (deterministic, no atomics).
constexpr int kBW = 8, kJW = 16, kIC = 16;
// the t = 0 factor of the box backward from the FMA pipe (sat(|t| 2^126)) instead of a compare:
// fewer instructions (80.6 -> 73.9 M per launch) but the FMA pipe becomes the limiter, C5-q2b
// pair_bwd 120 -> 130 us, so off for the single-disjunct kernel; KG_UNION_NZ_SAT for the union one
#ifndef KG_BOX_NZ_SAT
#define KG_BOX_NZ_SAT 0
#endif
#ifndef KG_UNION_NZ_SAT
#define KG_UNION_NZ_SAT 1
#endif
// resident CTAs per SM for the fused backward: 4 where the per-term state fits 64 registers
// without spills (measured +4 % C5-q2b q/s over 2), 2 for the 2- / 4-feature models
template <class Mdl> struct BwdOcc { static constexpr int v = (Mdl::BF == 1 && Mdl::AV == 1) ? 4 : 2; };

template <class Mdl>
__global__ void __launch_bounds__(kBW * 32, BwdOcc<Mdl>::v) pair_bwd_kernel(ScoreArgs a) {
  KG_GRID_DEP_WAIT();
  constexpr int QF = Mdl::QF, BQF = Mdl::BQF, BF = Mdl::BF, AV = Mdl::AV, JB = kBW * kJW;
  extern __shared__ __align__(16) float smem[];
  float *sC = smem;                                   // [kIC][JB]
  float *sQ = sC + kIC * JB;                          // [kIC][BQF][32]: Q features (+ BetaE QP)
  float *sDQ = sQ + kIC * BQF * 32;                   // [kBW][kIC][QF][32]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int U = a.U, K = a.K, NQ = a.NQ, qstride = QF * U;
  const int k = blockIdx.x * 32 + lane;
  const bool kval = k < U;
  const int jb0 = blockIdx.y * JB, jw0 = jb0 + w * kJW;
  const int rb = blockIdx.z * a.rps, re = min(NQ, rb + a.rps);
  float ev[kJW][BF], dv[kJW][AV];
#pragma unroll
  for (int jj = 0; jj < kJW; ++jj) {
    const int j = jw0 + jj;
    const int64_t er = (j < K) ? (a.eidx ? a.eidx[j] : (int64_t)j) : 0;
#pragma unroll
    for (int f = 0; f < BF; ++f) ev[jj][f] = (j < K && kval) ? a.E[er * a.estride + (Mdl::BOFF + f) * U + k] : 0.f;
#pragma unroll
    for (int f = 0; f < AV; ++f) dv[jj][f] = 0.f;
  }
  for (int r0 = rb; r0 < re; r0 += kIC) {
    // stage C[r0 .. r0+kIC][jb0 .. jb0+JB) and the query features of the chunk
    for (int e = threadIdx.x; e < kIC * JB / 4; e += blockDim.x) {
      const int ii = e / (JB / 4), c4 = e - ii * (JB / 4);
      const int r = r0 + ii, j = jb0 + c4 * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < re && j < a.Kp) v = ld4(a.C + (size_t)r * a.Kp + j);   // Kp % 64 == 0, padding is 0
      *reinterpret_cast<float4 *>(sC + ii * JB + c4 * 4) = v;
    }
    for (int e = threadIdx.x; e < kIC * BQF * 32; e += blockDim.x) {
      const int ii = e / (BQF * 32), f = (e / 32) % BQF, l = e & 31;
      const int r = r0 + ii, kk = blockIdx.x * 32 + l;
      float v = 0.f;
      if (r < re && kk < U)
        v = f < QF ? a.Q[(size_t)r * qstride + f * U + kk] : a.QP[(size_t)r * (BQF - QF) * U + (f - QF) * U + kk];
      sQ[e] = v;
    }
    __syncthreads();
#pragma unroll 1
    for (int ii = 0; ii < kIC; ++ii) {
      float q[BQF], dq[QF], dq2[QF];
#pragma unroll
      for (int f = 0; f < BQF; ++f) q[f] = sQ[(ii * BQF + f) * 32 + lane];
#pragma unroll
      for (int f = 0; f < QF; ++f) { dq[f] = 0.f; dq2[f] = 0.f; }
      const float4 *crow = reinterpret_cast<const float4 *>(sC + ii * JB + w * kJW);
      if constexpr (std::is_same<Mdl, MBox>::value) {
        // Q2B on packed f32x2 pairs of pool entries: t = v - c, a = |t|, W = [a > o] + alpha [a < o],
        // cw = C W, cg = sign(t) cw (0 at t = 0, A19): dq_c -= cg, dv += cg, dq_o -= cw
        const float2 cc = make_float2(-q[0], -q[0]);
        const float o = q[1];
        float2 gq0 = make_float2(0.f, 0.f), gq1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int j4 = 0; j4 < kJW / 4; ++j4) {
          const float4 c4 = crow[j4];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int jp = j4 * 2 + h2;
            const float2 cf = h2 ? make_float2(c4.z, c4.w) : make_float2(c4.x, c4.y);
            const float2 t = __fadd2_rn(make_float2(ev[2 * jp][0], ev[2 * jp + 1][0]), cc);
            const float ax = fabsf(t.x), ay = fabsf(t.y);
            const float2 W = make_float2(fmaf(a.alpha, ax < o ? 1.f : 0.f, ax > o ? 1.f : 0.f),
                                         fmaf(a.alpha, ay < o ? 1.f : 0.f, ay > o ? 1.f : 0.f));
            const float2 cw = __fmul2_rn(cf, W);
#if KG_BOX_NZ_SAT
            // sign(t) cw, 0 at t = 0 (A19): unconditional sign transfer (LOP3) times a 0 / 1
            // factor from the FMA pipe, sat(|t| 2^126) (1 for every normal |t|, 0 at t = 0),
            // instead of a compare + predicated LOP3 on the ALU pipe (this loop's limiter)
            const float2 csg = make_float2(__int_as_float(__float_as_int(cw.x) ^ (__float_as_int(t.x) & 0x80000000)),
                                           __int_as_float(__float_as_int(cw.y) ^ (__float_as_int(t.y) & 0x80000000)));
            const float2 cg = __fmul2_rn(csg, make_float2(__saturatef(ax * 0x1p126f), __saturatef(ay * 0x1p126f)));
#else
            const float2 cg = make_float2(
                t.x == 0.f ? 0.f : __int_as_float(__float_as_int(cw.x) ^ (__float_as_int(t.x) & 0x80000000)),
                t.y == 0.f ? 0.f : __int_as_float(__float_as_int(cw.y) ^ (__float_as_int(t.y) & 0x80000000)));
#endif
            gq0 = __fadd2_rn(gq0, cg);
            gq1 = __fadd2_rn(gq1, cw);
            const float2 dvp = __fadd2_rn(make_float2(dv[2 * jp][0], dv[2 * jp + 1][0]), cg);
            dv[2 * jp][0] = dvp.x;
            dv[2 * jp + 1][0] = dvp.y;
          }
        }
        dq[0] = -(gq0.x + gq0.y);
        dq[1] = -(gq1.x + gq1.y);
      } else if constexpr (std::is_same<Mdl, MRot>::value) {
        // RotatE on packed f32x2 pairs of pool entries (even j -> .x, odd j -> .y: the generic
        // path's dq / dq2 split, so the sums are the same): a = q - t, w = C / |z| (0 at z = 0,
        // A19); dq += w (a, b), dv -= w (a, b).  The FMA pipe was the limiter at 8 unpacked
        // instructions per term; packed, the MUFU.RSQ is.
        const float2 qre = make_float2(q[0], q[0]), qim = make_float2(q[1], q[1]);
        float2 g0 = make_float2(0.f, 0.f), g1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int j4 = 0; j4 < kJW / 4; ++j4) {
          const float4 c4 = crow[j4];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int jp = j4 * 2 + h2;
            const float2 cf = h2 ? make_float2(c4.z, c4.w) : make_float2(c4.x, c4.y);
            const float2 a2 = __fadd2_rn(qre, make_float2(-ev[2 * jp][0], -ev[2 * jp + 1][0]));
            const float2 b2 = __fadd2_rn(qim, make_float2(-ev[2 * jp][1], -ev[2 * jp + 1][1]));
            const float2 s2 = __ffma2_rn(a2, a2, __fmul2_rn(b2, b2));
            float2 w2 = __fmul2_rn(cf, make_float2(rsqrt_n(s2.x), rsqrt_n(s2.y)));
            w2.x = s2.x > 1e-30f ? w2.x : 0.f;
            w2.y = s2.y > 1e-30f ? w2.y : 0.f;
            g0 = __ffma2_rn(w2, a2, g0);
            g1 = __ffma2_rn(w2, b2, g1);
            const float2 nw = make_float2(-w2.x, -w2.y);
            const float2 dre = __ffma2_rn(nw, a2, make_float2(dv[2 * jp][0], dv[2 * jp + 1][0]));
            const float2 dim = __ffma2_rn(nw, b2, make_float2(dv[2 * jp][1], dv[2 * jp + 1][1]));
            dv[2 * jp][0] = dre.x; dv[2 * jp + 1][0] = dre.y;
            dv[2 * jp][1] = dim.x; dv[2 * jp + 1][1] = dim.y;
          }
        }
        dq[0] = g0.x; dq2[0] = g0.y;
        dq[1] = g1.x; dq2[1] = g1.y;
      } else if constexpr (std::is_same<Mdl, MBeta>::value) {
        // BetaE (MBeta::grad) on packed f32x2 pairs of pool entries, element for element the
        // same fmaf / subtraction sequence (even j -> .x = dq, odd j -> .y = dq2)
        const float2 a2 = make_float2(q[0], q[0]), b2 = make_float2(q[1], q[1]);
        const float2 qa = make_float2(q[2], q[2]), qb = make_float2(q[3], q[3]);
        float2 g0 = make_float2(0.f, 0.f), g1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int j4 = 0; j4 < kJW / 4; ++j4) {
          const float4 c4 = crow[j4];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int jp = j4 * 2 + h2, j0 = 2 * jp, j1 = 2 * jp + 1;
            const float2 cf = h2 ? make_float2(c4.z, c4.w) : make_float2(c4.x, c4.y);
            g0 = __ffma2_rn(cf, __fadd2_rn(qa, make_float2(-ev[j0][0], -ev[j1][0])), g0);
            g1 = __ffma2_rn(cf, __fadd2_rn(qb, make_float2(-ev[j0][1], -ev[j1][1])), g1);
            const float2 v0 = __ffma2_rn(cf, __fadd2_rn(make_float2(ev[j0][2], ev[j1][2]), make_float2(-a2.x, -a2.y)),
                                         make_float2(dv[j0][0], dv[j1][0]));
            const float2 v1 = __ffma2_rn(cf, __fadd2_rn(make_float2(ev[j0][3], ev[j1][3]), make_float2(-b2.x, -b2.y)),
                                         make_float2(dv[j0][1], dv[j1][1]));
            dv[j0][0] = v0.x; dv[j1][0] = v0.y;
            dv[j0][1] = v1.x; dv[j1][1] = v1.y;
          }
        }
        dq[0] = g0.x; dq2[0] = g0.y;
        dq[1] = g1.x; dq2[1] = g1.y;
      } else {
#pragma unroll
        for (int j4 = 0; j4 < kJW / 4; ++j4) {
          const float4 c4 = crow[j4];
          Mdl::grad(q, ev[j4 * 4 + 0], c4.x, a.alpha, dq, dv[j4 * 4 + 0]);
          Mdl::grad(q, ev[j4 * 4 + 1], c4.y, a.alpha, dq2, dv[j4 * 4 + 1]);
          Mdl::grad(q, ev[j4 * 4 + 2], c4.z, a.alpha, dq, dv[j4 * 4 + 2]);
          Mdl::grad(q, ev[j4 * 4 + 3], c4.w, a.alpha, dq2, dv[j4 * 4 + 3]);
        }
      }
#pragma unroll
      for (int f = 0; f < QF; ++f) sDQ[((w * kIC + ii) * QF + f) * 32 + lane] = dq[f] + dq2[f];
    }
    __syncthreads();
    // fixed-order combine over the warps; one partial per (row, j-block)
    for (int e = threadIdx.x; e < kIC * QF * 32; e += blockDim.x) {
      const int ii = e / (QF * 32), f = (e / 32) % QF, l = e & 31;
      const int r = r0 + ii, kk = blockIdx.x * 32 + l;
      float s = 0.f;
#pragma unroll
      for (int ww = 0; ww < kBW; ++ww) s += sDQ[ww * kIC * QF * 32 + e];
      if (r < re && kk < U) a.partQ[((size_t)blockIdx.y * NQ + r) * qstride + f * U + kk] = s;
    }
    __syncthreads();
  }
  const size_t zs = (size_t)K * AV * U;
#pragma unroll
  for (int jj = 0; jj < kJW; ++jj) {
    const int j = jw0 + jj;
    if (j >= K || !kval) continue;
#pragma unroll
    for (int f = 0; f < AV; ++f) a.partV[blockIdx.z * zs + (size_t)j * AV * U + f * U + k] = dv[jj][f];
  }
}

// Q2B unions (NOUT = 2, A11): C[t][i][j] is non-zero only for the argmin disjunct t of the
// pair (i, j) (or for neither), so one pass per QUERY covers both disjunct rows instead of one
// pass per disjunct row: t(i, j) = [C[1][i][j] != 0] picks the disjunct's box (bit-mask
// selects) and its dQ accumulators (x {0, 1} products, exact); c = C[0] + C[1] (one is 0,
// exact).  The terms and their fp32 arithmetic are those of pair_bwd_kernel<MBox>; it writes
// the same partials (rows t M + i), so the combines are shared.
constexpr int kICU = 8;   // query rows per staged chunk (two disjunct rows each; 52 KB of shared memory)
#ifndef KG_UNION_OCC
#define KG_UNION_OCC 3
#endif
// resident CTAs per SM (4, at 64 registers with a small spill, measured slower: C5-q2b 2u scoring
// backward 0.207 -> 0.232 ms)
constexpr int kUnionOcc = KG_UNION_OCC;
__global__ void __launch_bounds__(kBW * 32, kUnionOcc) pair_bwd_union_box_kernel(ScoreArgs a) {
  KG_GRID_DEP_WAIT();
  constexpr int JB = kBW * kJW;
  extern __shared__ __align__(16) float smem[];
  float *sC = smem;                                             // [kICU][JB] C[0] + C[1]
  float *sT = sC + kICU * JB;                                    // [kICU][JB] t as 0 / 1
  float *sN = sT + kICU * JB;                                    // [kICU][JB] 1 - t
  int *sMk = reinterpret_cast<int *>(sN + kICU * JB);            // [kICU][JB] -t (bit mask)
  float *sQ = reinterpret_cast<float *>(sMk + kICU * JB);        // [kICU][4][32] cA oA cB oB
  float *sDQ = sQ + kICU * 4 * 32;                               // [kBW][kICU][4][32]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int U = a.U, K = a.K, M = a.M, qstride = 2 * U;
  const int k = blockIdx.x * 32 + lane;
  const bool kval = k < U;
  const int jb0 = blockIdx.y * JB, jw0 = jb0 + w * kJW;
  const int rb = blockIdx.z * a.rps, re = min(M, rb + a.rps);
  float ev[kJW], dv[kJW];
#pragma unroll
  for (int jj = 0; jj < kJW; ++jj) {
    const int j = jw0 + jj;
    const int64_t er = (j < K) ? (a.eidx ? a.eidx[j] : (int64_t)j) : 0;
    ev[jj] = (j < K && kval) ? a.E[er * a.estride + k] : 0.f;
    dv[jj] = 0.f;
  }
  for (int r0 = rb; r0 < re; r0 += kICU) {
    for (int e = threadIdx.x; e < kICU * JB / 4; e += blockDim.x) {
      const int ii = e / (JB / 4), c4 = e - ii * (JB / 4);
      const int i = r0 + ii, j = jb0 + c4 * 4;
      float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
      if (i < re && j < a.Kp) {
        v0 = ld4(a.C + (size_t)i * a.Kp + j);
        v1 = ld4(a.C + (size_t)(M + i) * a.Kp + j);
      }
      *reinterpret_cast<float4 *>(sC + ii * JB + c4 * 4) = make_float4(v0.x + v1.x, v0.y + v1.y, v0.z + v1.z, v0.w + v1.w);
      const int4 mk = make_int4(-(int)(v1.x != 0.f), -(int)(v1.y != 0.f), -(int)(v1.z != 0.f), -(int)(v1.w != 0.f));
      *reinterpret_cast<float4 *>(sT + ii * JB + c4 * 4) = make_float4(-mk.x, -mk.y, -mk.z, -mk.w);
      *reinterpret_cast<float4 *>(sN + ii * JB + c4 * 4) = make_float4(1 + mk.x, 1 + mk.y, 1 + mk.z, 1 + mk.w);
      *reinterpret_cast<int4 *>(sMk + ii * JB + c4 * 4) = mk;
    }
    for (int e = threadIdx.x; e < kICU * 4 * 32; e += blockDim.x) {
      const int ii = e / 128, f = (e / 32) & 3, l = e & 31;
      const int i = r0 + ii, kk = blockIdx.x * 32 + l;
      float v = 0.f;
      if (i < re && kk < U) v = a.Q[(size_t)((f >> 1) * M + i) * qstride + (f & 1) * U + kk];
      sQ[e] = v;
    }
    __syncthreads();
#pragma unroll 1
    for (int ii = 0; ii < kICU; ++ii) {
      const float cA = sQ[(ii * 4 + 0) * 32 + lane], oA = sQ[(ii * 4 + 1) * 32 + lane];
      const float cB = sQ[(ii * 4 + 2) * 32 + lane], oB = sQ[(ii * 4 + 3) * 32 + lane];
      const int icA = __float_as_int(cA), icB = __float_as_int(cB), ioA = __float_as_int(oA), ioB = __float_as_int(oB);
      float2 gA0 = make_float2(0.f, 0.f), gA1 = gA0, gB0 = gA0, gB1 = gA0;
      const float4 *crow = reinterpret_cast<const float4 *>(sC + ii * JB + w * kJW);
      const float4 *trow = reinterpret_cast<const float4 *>(sT + ii * JB + w * kJW);
      const float4 *nrow = reinterpret_cast<const float4 *>(sN + ii * JB + w * kJW);
      const int4 *mrow = reinterpret_cast<const int4 *>(sMk + ii * JB + w * kJW);
#pragma unroll
      for (int j4 = 0; j4 < kJW / 4; ++j4) {
        const float4 c4 = crow[j4], t4 = trow[j4], n4 = nrow[j4];
        const int4 m4 = mrow[j4];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int jp = j4 * 2 + h2;
          const float2 cf = h2 ? make_float2(c4.z, c4.w) : make_float2(c4.x, c4.y);
          const float2 tf = h2 ? make_float2(t4.z, t4.w) : make_float2(t4.x, t4.y);
          const float2 nt = h2 ? make_float2(n4.z, n4.w) : make_float2(n4.x, n4.y);
          const int mx = h2 ? m4.z : m4.x, my = h2 ? m4.w : m4.y;   // all ones <=> disjunct 1
          const float2 cs = make_float2(__int_as_float((icA & ~mx) | (icB & mx)), __int_as_float((icA & ~my) | (icB & my)));
          const float ox = __int_as_float((ioA & ~mx) | (ioB & mx)), oy = __int_as_float((ioA & ~my) | (ioB & my));
          const float2 t = __fadd2_rn(make_float2(ev[2 * jp], ev[2 * jp + 1]), make_float2(-cs.x, -cs.y));
          const float ax = fabsf(t.x), ay = fabsf(t.y);
          const float2 W = make_float2(fmaf(a.alpha, ax < ox ? 1.f : 0.f, ax > ox ? 1.f : 0.f),
                                       fmaf(a.alpha, ay < oy ? 1.f : 0.f, ay > oy ? 1.f : 0.f));
          const float2 cw = __fmul2_rn(cf, W);
          // sign(t) cw with 0 at t = 0 (A19): sign transfer (LOP3) x a 0/1 factor on the FMA
          // pipe instead of a select (this loop's ALU pipe also carries the disjunct selects)
          const float2 csg = make_float2(__int_as_float(__float_as_int(cw.x) ^ (__float_as_int(t.x) & 0x80000000)),
                                         __int_as_float(__float_as_int(cw.y) ^ (__float_as_int(t.y) & 0x80000000)));
#if KG_UNION_NZ_SAT
          // the 0 / 1 factor from the FMA pipe: sat(|t| 2^126) (1 for every normal |t|, 0 at t = 0)
          const float2 cg = __fmul2_rn(csg, make_float2(__saturatef(ax * 0x1p126f), __saturatef(ay * 0x1p126f)));
#else
          const float2 cg = __fmul2_rn(csg, make_float2(t.x != 0.f ? 1.f : 0.f, t.y != 0.f ? 1.f : 0.f));
#endif
          gA0 = __ffma2_rn(cg, nt, gA0);
          gB0 = __ffma2_rn(cg, tf, gB0);
          gA1 = __ffma2_rn(cw, nt, gA1);
          gB1 = __ffma2_rn(cw, tf, gB1);
          const float2 dvp = __fadd2_rn(make_float2(dv[2 * jp], dv[2 * jp + 1]), cg);
          dv[2 * jp] = dvp.x;
          dv[2 * jp + 1] = dvp.y;
        }
      }
      float *o = sDQ + ((w * kICU + ii) * 4) * 32 + lane;
      o[0] = -(gA0.x + gA0.y);
      o[32] = -(gA1.x + gA1.y);
      o[64] = -(gB0.x + gB0.y);
      o[96] = -(gB1.x + gB1.y);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kICU * 4 * 32; e += blockDim.x) {
      const int ii = e / 128, f = (e / 32) & 3, l = e & 31;
      const int i = r0 + ii, kk = blockIdx.x * 32 + l;
      float sum = 0.f;
#pragma unroll
      for (int ww = 0; ww < kBW; ++ww) sum += sDQ[ww * kICU * 4 * 32 + e];
      if (i < re && kk < U)
        a.partQ[((size_t)blockIdx.y * a.NQ + (size_t)(f >> 1) * M + i) * qstride + (f & 1) * U + kk] = sum;
    }
    __syncthreads();
  }
  const size_t zs = (size_t)K * U;
#pragma unroll
  for (int jj = 0; jj < kJW; ++jj) {
    const int j = jw0 + jj;
    if (j >= K || !kval) continue;
    a.partV[blockIdx.z * zs + (size_t)j * U + k] = dv[jj];
  }
}

// dQ[r][f*U + k] += sum_z partQ[z] (+ Q2B offset: alpha * Csum[r]); dQ already holds the
// positive term.  (BetaE's partials already hold sum_j C (QP - P), see MBeta::grad.)
template <bool BETA, bool BOX>
__device__ __forceinline__ void bwd_q_combine(const ScoreArgs &a, int qstride, int64_t e) {
  const int64_t n = (int64_t)a.NQ * qstride;
  if (e >= n) return;
  float v = 0.f;
  for (int z = 0; z < a.JS; ++z) v += a.partQ[z * n + e];
  v *= a.gsign;
  if (BOX && (e % qstride) >= a.U) v = fmaf(a.alpha, a.Csum[e / qstride], v);
  a.dQ[e] += v;
}

// Raw-row gradient of pool entry j: sum_z partials (+ BetaE epilogue with the
// entity features [A, B, TA, TB, TAB, GA, GB] = F planes 2..8).
template <class Mdl>
__device__ __forceinline__ void bwd_v_combine(const ScoreArgs &a, int64_t e) {
  constexpr int AV = Mdl::AV;
  const int U = a.U, K = a.K;
  if (e >= (int64_t)K * U) return;
  const int j = (int)(e / U), k = (int)(e - (int64_t)j * U);
  const size_t zs = (size_t)K * AV * U;
  float acc[AV];
#pragma unroll
  for (int f = 0; f < AV; ++f) {
    float s = 0.f;
    for (int z = 0; z < a.RS; ++z) s += a.partV[z * zs + (size_t)j * AV * U + f * U + k];
    acc[f] = s * a.gsign;
  }
  float *out = a.dV + (size_t)j * a.d;
  if (Mdl::kBeta) {
    // S1 = sum_i C (A - a2), S2 = sum_i C (B - b2) (MBeta::grad):
    // dKL/dA = (A - a2) psi'(A) - ((A - a2) + (B - b2)) psi'(A + B), likewise for B
    const float *Fr = a.E + (size_t)j * a.estride;
    const float TA = Fr[4 * U + k], TB = Fr[5 * U + k], TAB = Fr[6 * U + k], GA = Fr[7 * U + k],
                GB = Fr[8 * U + k];
    const float S1 = acc[0], S2 = acc[AV - 1];
    const float S = S1 + S2;
    out[k] = (TA * S1 - TAB * S) * GA;
    out[U + k] = (TB * S2 - TAB * S) * GB;
  } else {
#pragma unroll
    for (int f = 0; f < Mdl::OUTF; ++f) out[f * U + k] = acc[f];
  }
}

// Both combines in one launch: blocks [0, nqb) sum the dQ partials, the rest the dV partials.
template <class Mdl>
__global__ void bwd_combine_kernel(ScoreArgs a, int qstride, int nqb) {
  KG_GRID_DEP_WAIT();
  if ((int)blockIdx.x < nqb)
    bwd_q_combine<Mdl::kBeta, Mdl::kRowAlpha>(a, qstride, blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  else
    bwd_v_combine<Mdl>(a, (blockIdx.x - nqb) * (int64_t)blockDim.x + threadIdx.x);
}
// The same sums on 4 consecutive units per thread (U % 4 == 0): float4 loads of the partials,
// a quarter of the threads and instructions; every element's sum is the scalar kernel's.
__device__ __forceinline__ void add4v(float4 &a, const float4 b) { a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w; }
template <bool BOX>
__device__ __forceinline__ void bwd_q_combine4(const ScoreArgs &a, int qstride, int64_t e4) {
  const int64_t n4 = (int64_t)a.NQ * qstride / 4;
  if (e4 >= n4) return;
  const float4 *P = reinterpret_cast<const float4 *>(a.partQ);
  float4 v = P[e4];
  for (int z = 1; z < a.JS; ++z) add4v(v, P[z * n4 + e4]);
  v.x *= a.gsign; v.y *= a.gsign; v.z *= a.gsign; v.w *= a.gsign;
  const int64_t e = e4 * 4;
  if (BOX && (e % qstride) >= a.U) {
    const float cs = a.Csum[e / qstride];
    v.x = fmaf(a.alpha, cs, v.x); v.y = fmaf(a.alpha, cs, v.y); v.z = fmaf(a.alpha, cs, v.z); v.w = fmaf(a.alpha, cs, v.w);
  }
  float4 *d = reinterpret_cast<float4 *>(a.dQ) + e4;
  float4 o = *d;
  o.x += v.x; o.y += v.y; o.z += v.z; o.w += v.w;
  *d = o;
}
template <class Mdl>
__device__ __forceinline__ void bwd_v_combine4(const ScoreArgs &a, int64_t e4) {
  constexpr int AV = Mdl::AV;
  const int U = a.U, K = a.K, U4 = U / 4;
  if (e4 >= (int64_t)K * U4) return;
  const int j = (int)(e4 / U4), k = (int)(e4 - (int64_t)j * U4) * 4;
  const size_t zs = (size_t)K * AV * U;
  float4 acc[AV];
#pragma unroll
  for (int f = 0; f < AV; ++f) {
    const float4 *P = reinterpret_cast<const float4 *>(a.partV + (size_t)j * AV * U + f * U + k);
    float4 s4 = P[0];
    for (int z = 1; z < a.RS; ++z) add4v(s4, P[z * zs / 4]);
    acc[f] = make_float4(s4.x * a.gsign, s4.y * a.gsign, s4.z * a.gsign, s4.w * a.gsign);
  }
  float *out = a.dV + (size_t)j * a.d;
  if (Mdl::kBeta) {
    const float *Fr = a.E + (size_t)j * a.estride;
    const float4 TA = *reinterpret_cast<const float4 *>(Fr + 4 * U + k), TB = *reinterpret_cast<const float4 *>(Fr + 5 * U + k),
                 TAB = *reinterpret_cast<const float4 *>(Fr + 6 * U + k), GA = *reinterpret_cast<const float4 *>(Fr + 7 * U + k),
                 GB = *reinterpret_cast<const float4 *>(Fr + 8 * U + k);
    const float4 S1 = acc[0], S2 = acc[AV - 1];
    float4 oa, ob;
#define KG_BETA_V(c)                                   \
    {                                                  \
      const float S = S1.c + S2.c;                     \
      oa.c = (TA.c * S1.c - TAB.c * S) * GA.c;         \
      ob.c = (TB.c * S2.c - TAB.c * S) * GB.c;         \
    }
    KG_BETA_V(x) KG_BETA_V(y) KG_BETA_V(z) KG_BETA_V(w)
#undef KG_BETA_V
    *reinterpret_cast<float4 *>(out + k) = oa;
    *reinterpret_cast<float4 *>(out + U + k) = ob;
  } else {
#pragma unroll
    for (int f = 0; f < Mdl::OUTF; ++f) *reinterpret_cast<float4 *>(out + f * U + k) = acc[f];
  }
}
template <class Mdl>
__global__ void bwd_combine4_kernel(ScoreArgs a, int qstride, int nqb) {
  KG_GRID_DEP_WAIT();
  if ((int)blockIdx.x < nqb)
    bwd_q_combine4<Mdl::kRowAlpha>(a, qstride, blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  else
    bwd_v_combine4<Mdl>(a, (blockIdx.x - nqb) * (int64_t)blockDim.x + threadIdx.x);
}
template <class Mdl>
static void launch_combine(const ScoreArgs &a, int qstride, cudaStream_t st) {
  const int64_t nq = (int64_t)a.NQ * qstride, nv = (int64_t)a.K * a.U;
  const bool vec = (a.U % 4 == 0) && (a.d % 4 == 0) && (a.estride % 4 == 0) &&
                   !(reinterpret_cast<uintptr_t>(a.dQ) & 15) && !(reinterpret_cast<uintptr_t>(a.dV) & 15) &&
                   !(reinterpret_cast<uintptr_t>(a.partQ) & 15) && !(reinterpret_cast<uintptr_t>(a.partV) & 15) &&
                   !(reinterpret_cast<uintptr_t>(a.E) & 15);
  if (vec) {
    const int nqb = (int)((nq / 4 + 255) / 256), nvb = (int)((nv / 4 + 255) / 256);
    if (nqb + nvb > 0) { bwd_combine4_kernel<Mdl><<<nqb + nvb, 256, 0, st>>>(a, qstride, nqb); ++g_launches; }
    return;
  }
  const int nqb = (int)((nq + 255) / 256), nvb = (int)((nv + 255) / 256);
  if (nqb + nvb > 0) { bwd_combine_kernel<Mdl><<<nqb + nvb, 256, 0, st>>>(a, qstride, nqb); ++g_launches; }
}

// ---------------------------------------------------------------- positives
// One CTA per query i: D+ for each disjunct, DNF min, Eq. 1 positive term and
// its adjoint sigma(D+ - gamma)/(M G); initialises dQ (all disjuncts) and
// writes the raw-row gradient of the answer occurrence.
template <int KIND, int NOUT>
__global__ void __launch_bounds__(128) pos_kernel(PosArgs p) {
  KG_GRID_DEP_WAIT();
  __shared__ float red[32];
  const int i = blockIdx.x, M = p.M, U = p.U, d = p.d;
  constexpr int QF = (KIND == GQE || KIND == TRANSE || KIND == DISTMULT) ? 1 : 2;
  const float *x = p.ent + p.ans_rows[i] * (int64_t)d;
  float part[NOUT + 1];
#pragma unroll
  for (int tt = 0; tt <= NOUT; ++tt) part[tt] = 0.f;
  for (int k = threadIdx.x; k < U; k += blockDim.x) {
    float A = 0.f, B = 0.f, Pa = 0.f, Pb = 0.f;
    if (KIND == BETAE) {
      A = beta_act(x[k]); B = beta_act(x[U + k]);
      const float pab = digammaf_(A + B);
      Pa = digammaf_(A) - pab; Pb = digammaf_(B) - pab;
      part[NOUT] += lnbetaf_(A, B);
    }
#pragma unroll
    for (int tt = 0; tt < NOUT; ++tt) {
      const float *q = p.Q + (size_t)(tt * M + i) * QF * U;
      float v;
      if (KIND == GQE || KIND == TRANSE) { const float z = q[k] - x[k]; v = z * z; }
      else if (KIND == Q2B) { const float dl = fabsf(x[k] - q[k]); v = fmaxf(dl - q[U + k], 0.f) + p.alpha * fminf(dl, q[U + k]); }
      else if (KIND == BETAE) { v = (A - q[k]) * Pa + (B - q[U + k]) * Pb; }
      else if (KIND == ROTATE) { const float a = q[k] - x[k], b = q[U + k] - x[U + k]; v = sqrtf(a * a + b * b); }
      else if (KIND == DISTMULT) { v = q[k] * x[k]; }
      else { v = q[k] * x[k] + q[U + k] * x[U + k]; }
      part[tt] += v;
    }
  }
  float D[NOUT], cv = 0.f;
  if (KIND == BETAE) cv = block_sum(part[NOUT], red);
#pragma unroll
  for (int tt = 0; tt < NOUT; ++tt) {
    const float s = block_sum(part[tt], red);
    if (KIND == GQE || KIND == TRANSE) D[tt] = sqrtf(s);
    else if (KIND == BETAE) D[tt] = s + p.Cq[tt * M + i] - cv;
    else if (KIND == DISTMULT || KIND == COMPLEX) D[tt] = -s;
    else D[tt] = s;
  }
  int tm = 0;
  float Dm = D[0];
  if (NOUT == 2 && D[1] < D[0]) { tm = 1; Dm = D[1]; }
  const float c = sigm_(Dm - p.gamma) * p.scale;                  // dl/dD+ (Eq. 1)
  if (threadIdx.x == 0) {
    p.loss_pos[i] = softplusf_(Dm - p.gamma);
    if (p.Dpos) p.Dpos[i] = Dm;
  }
  const float *q = p.Q + (size_t)(tm * M + i) * QF * U;
  float *og = p.dV + (size_t)i * d;
  const float invD = (Dm > 0.f) ? 1.f / Dm : 0.f;
  for (int k = threadIdx.x; k < U; k += blockDim.x) {
    float gq[2] = {0.f, 0.f}, gv[2] = {0.f, 0.f};
    if (KIND == GQE || KIND == TRANSE) {
      const float z = (q[k] - x[k]) * invD * c; gq[0] = z; gv[0] = -z;
    } else if (KIND == Q2B) {
      const float dl = x[k] - q[k], a = fabsf(dl), o = q[U + k];
      const float s = (dl > 0.f) ? 1.f : ((dl < 0.f) ? -1.f : 0.f);
      const float outb = a > o ? 1.f : 0.f, inb = a < o ? 1.f : 0.f;
      gq[0] = -c * s * (outb + p.alpha * inb);
      gq[1] = c * (-outb + p.alpha * (a >= o ? 1.f : 0.f));
      gv[0] = c * s * (outb + p.alpha * inb);
    } else if (KIND == BETAE) {
      const float A = beta_act(x[k]), B = beta_act(x[U + k]);
      const float pab = digammaf_(A + B), Pa = digammaf_(A) - pab, Pb = digammaf_(B) - pab;
      const float a2 = q[k], b2 = q[U + k];
      gq[0] = c * (-Pa + p.QP[(size_t)(tm * M + i) * 2 * U + k]);
      gq[1] = c * (-Pb + p.QP[(size_t)(tm * M + i) * 2 * U + U + k]);
      const float tab = trigammaf_(A + B), S = A + B - a2 - b2;
      gv[0] = c * ((A - a2) * trigammaf_(A) - S * tab) * beta_act_grad(x[k]);
      gv[1] = c * ((B - b2) * trigammaf_(B) - S * tab) * beta_act_grad(x[U + k]);
    } else if (KIND == ROTATE) {
      const float a = q[k] - x[k], b = q[U + k] - x[U + k], n = sqrtf(a * a + b * b);
      if (n > 0.f) { gq[0] = c * a / n; gq[1] = c * b / n; gv[0] = -gq[0]; gv[1] = -gq[1]; }
    } else if (KIND == DISTMULT) {
      gq[0] = -c * x[k]; gv[0] = -c * q[k];
    } else {
      gq[0] = -c * x[k]; gq[1] = -c * x[U + k]; gv[0] = -c * q[k]; gv[1] = -c * q[U + k];
    }
#pragma unroll
    for (int tt = 0; tt < NOUT; ++tt) {
      float *dq = p.dQ + (size_t)(tt * M + i) * QF * U;
#pragma unroll
      for (int f = 0; f < QF; ++f) dq[f * U + k] = (tt == tm) ? gq[f] : 0.f;
    }
    og[k] = gv[0];
    if (QF == 2 && KIND != Q2B) og[U + k] = gv[1];
  }
}

// ---------------------------------------------------------------- BetaE precompute
// Entity features of the pool (9 planes of m, layout above) and Cv_j = sum_k lnB(A, B).
__global__ void __launch_bounds__(128) beta_entity_kernel(const float *ent, const int64_t *rows, int K, int m,
                                                          float *F, float *Cv) {
  KG_GRID_DEP_WAIT();
  __shared__ float red[32];
  const int j = blockIdx.x;
  const float *x = ent + rows[j] * (int64_t)(2 * m);
  float *f = F + (size_t)j * 9 * m;
  float s = 0.f;
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    const float xa = x[k], xb = x[m + k];
    const float A = beta_act(xa), B = beta_act(xb);
    const float pab = digammaf_(A + B);
    f[k] = digammaf_(A) - pab;
    f[m + k] = digammaf_(B) - pab;
    f[2 * m + k] = A;
    f[3 * m + k] = B;
    f[4 * m + k] = trigammaf_(A);
    f[5 * m + k] = trigammaf_(B);
    f[6 * m + k] = trigammaf_(A + B);
    f[7 * m + k] = beta_act_grad(xa);
    f[8 * m + k] = beta_act_grad(xb);
    s += lnbetaf_(A, B);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) Cv[j] = s;
}

// Query features: QP[r] = [psi(a2) - psi(a2+b2) | psi(b2) - psi(a2+b2)], Cq[r] = sum_k lnB(a2, b2).
__global__ void __launch_bounds__(128) beta_query_kernel(const float *Q, int NQ, int m, float *QP, float *Cq) {
  KG_GRID_DEP_WAIT();
  __shared__ float red[32];
  const int r = blockIdx.x;
  const float *q = Q + (size_t)r * 2 * m;
  float s = 0.f;
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    const float a2 = q[k], b2 = q[m + k], pab = digammaf_(a2 + b2);
    QP[(size_t)r * 2 * m + k] = digammaf_(a2) - pab;
    QP[(size_t)r * 2 * m + m + k] = digammaf_(b2) - pab;
    s += lnbetaf_(a2, b2);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) Cq[r] = s;
}

// ---------------------------------------------------------------- loss
// Deterministic sum of the per-query terms; finite check; Adam step counter and
// bias corrections on device (so a step needs no host round trip).
__global__ void __launch_bounds__(256) loss_finalize_kernel(const float *loss_pos, const float *loss_part, int M,
                                                            int njt, double scale, double *loss_out,
                                                            int *flags, int64_t *t_dev, float *bc,
                                                            double beta1, double beta2, int apply, int check) {
  KG_GRID_DEP_WAIT();
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < M; i += 256) {
    double v = loss_pos[i];
    for (int jt = 0; jt < njt; ++jt) v += loss_part[(size_t)jt * M + i];
    s += v;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0 && !check) *loss_out = red[0] * scale;   // world > 1: summed over ranks, then loss_check
  if (threadIdx.x == 0 && check) {
    const double loss = red[0] * scale;
    // flags[1]: an input id / relation was out of range (device-side validation);
    // flags[0]: skip every update of this step (non-finite loss or bad input).
    const int bad = !isfinite(loss) || flags[1];
    *loss_out = loss;
    flags[0] = bad;
    if (!bad && apply) {
      const int64_t t = *t_dev + 1;
      *t_dev = t;
      bc[0] = (float)(1.0 / (1.0 - pow(beta1, (double)t)));   // reciprocal bias corrections (A15)
      bc[1] = (float)(1.0 / (1.0 - pow(beta2, (double)t)));
    }
  }
}

// ---------------------------------------------------------------- launchers
// Split counts: enough CTAs for ~4 per SM (148 SMs), bounded by the partial
// buffers and by whole chunks per split.
// Unit-range split of the forward: the count minimising (waves of resident CTAs) x (chunks per
// CTA), ties to fewer parts -- e.g. Q2B unions (114 registers, 2 CTAs per SM): 5 parts were
// 2.16 waves, 2 parts fit one.  `slots` = resident CTAs of the kernel on the whole GPU.
static int split_for(int tiles, int chunks, int slots, int64_t cap_floats, int64_t per_split_floats) {
  if (tiles >= slots) return 1;   // already a full wave: partials would only add traffic (B = K = 4096)
  int best = 1;
  int64_t best_cost = INT64_MAX;
  for (int s = 1; s <= std::min(8, chunks); ++s) {
    const int per = (chunks + s - 1) / s, parts = (chunks + per - 1) / per;
    if ((int64_t)parts * per_split_floats > cap_floats) break;
    const int64_t cost = (((int64_t)tiles * parts + slots - 1) / slots) * per;
    if (cost < best_cost) { best_cost = cost; best = parts; }
  }
  return best;
}
template <class F> static int gpu_slots(F kernel, int threads) {
  int dev = 0, sms = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, 0);
  return std::max(1, per) * std::max(1, sms);
}

template <class Mdl>
static void launch_pair(ScoreArgs a, int nout, bool train, cudaStream_t st, const std::function<void()> &between) {
  const int tiles = ((a.K + 63) / 64) * ((a.M + 63) / 64);
  const int chunks = (a.U + 15) / 16;
  static const int slots1 = gpu_slots(pair_fwd_kernel<Mdl, 1>, 256), slots2 = gpu_slots(pair_fwd_kernel<Mdl, 2>, 256);
  a.KS = split_for(tiles, chunks, nout == 1 ? slots1 : slots2, a.cap_D, (int64_t)nout * a.M * a.Kp);
  a.ups = ((chunks + a.KS - 1) / a.KS) * 16;
  a.KS = (a.U + a.ups - 1) / a.ups;
  dim3 gf((a.K + 63) / 64, (a.M + 63) / 64, a.KS);
  if (nout == 1) {
    { pair_fwd_kernel<Mdl, 1><<<gf, 256, 0, st>>>(a); ++g_launches; }
    if (between) between();
    if (train) { pair_epi_kernel<Mdl, 1, true><<<a.M, 256, 0, st>>>(a); ++g_launches; }
    else { pair_epi_kernel<Mdl, 1, false><<<a.M, 256, 0, st>>>(a); ++g_launches; }
  } else {
    { pair_fwd_kernel<Mdl, 2><<<gf, 256, 0, st>>>(a); ++g_launches; }
    if (between) between();
    if (train) { pair_epi_kernel<Mdl, 2, true><<<a.M, 256, 0, st>>>(a); ++g_launches; }
    else { pair_epi_kernel<Mdl, 2, false><<<a.M, 256, 0, st>>>(a); ++g_launches; }
  }
}

void launch_pair_fwd(int kind, const ScoreArgs &a, int nout, bool train, cudaStream_t st,
                     const std::function<void()> &between) {
  switch (kind) {
    case GQE: case TRANSE: launch_pair<ML2>(a, nout, train, st, between); break;
    case Q2B: launch_pair<MBox>(a, nout, train, st, between); break;
    case BETAE: launch_pair<MBeta>(a, nout, train, st, between); break;
    case ROTATE: launch_pair<MRot>(a, nout, train, st, between); break;
    case DISTMULT: launch_pair<MDot>(a, nout, train, st, between); break;
    case COMPLEX: launch_pair<MCpx>(a, nout, train, st, between); break;
  }
}

template <class Mdl>
static void launch_bwd(ScoreArgs a, cudaStream_t st, cudaStream_t st2) {
  (void)st2;
  constexpr int JB = kBW * kJW;
  const int qstride = Mdl::QF * a.U;
  const int kt = (a.U + 31) / 32, jt = (a.K + JB - 1) / JB;
  a.JS = jt;                                   // dQ partials: one per j-block
  // Q2B unions: one pass per query over both disjunct rows (pair_bwd_union_box_kernel)
  const bool union_box = std::is_same<Mdl, MBox>::value && a.NQ == 2 * a.M;
  if (union_box) {
    const int chunks = (a.M + kICU - 1) / kICU;
    int is = (kUnionOcc * 148) / (kt * jt);   // one wave of the resident CTAs (ncu: 5 splits at 3 per SM were 1.17 waves)
    is = std::max(1, std::min(is, std::min(16, chunks)));
    while (is > 1 && (int64_t)is * a.K * a.U > a.cap_V) --is;
    a.rps = ((chunks + is - 1) / is) * kICU;
    a.RS = (a.M + a.rps - 1) / a.rps;
    const size_t smem = sizeof(float) * (4 * kICU * JB + kICU * 4 * 32 + kBW * kICU * 4 * 32);
    static const bool configured =
        cudaFuncSetAttribute(pair_bwd_union_box_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
        cudaSuccess;
    (void)configured;
    dim3 g(kt, jt, a.RS);
    { pair_bwd_union_box_kernel<<<g, kBW * 32, smem, st>>>(a); ++g_launches; }
    launch_combine<Mdl>(a, qstride, st);
    return;
  }
  const int chunks = (a.NQ + kIC - 1) / kIC;
  // row splits: one wave of resident CTAs (floor) unless that leaves > 15 % of the slots idle,
  // then the next count up (C5: 5 splits = 520 of 592 slots; B = K = 4096: 416 tiles -> 2)
  const int slots = BwdOcc<Mdl>::v * 148;
  int is = std::max(1, slots / (kt * jt));
  if ((int64_t)is * kt * jt * 100 < 85LL * slots) is = (slots + kt * jt - 1) / (kt * jt);
  // (measured at C5-q2b: 5 splits 0.136 ms, 8: 0.136, 11: 0.146, 16: 0.150 -- the finer splits'
  // extra dV partials cost more than the better balance of 3 vs 4 CTAs per SM saves)
  is = std::max(1, std::min(is, std::min(16, chunks)));
  while (is > 1 && (int64_t)is * a.K * Mdl::AV * a.U > a.cap_V) --is;
  a.rps = ((chunks + is - 1) / is) * kIC;
  a.RS = (a.NQ + a.rps - 1) / a.rps;
  const size_t smem = sizeof(float) * (kIC * JB + kIC * Mdl::BQF * 32 + kBW * kIC * Mdl::QF * 32);
  static const bool configured =   // thread-safe one-time attribute (concurrent host threads)
      cudaFuncSetAttribute(pair_bwd_kernel<Mdl>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess;
  (void)configured;
  dim3 g(kt, jt, a.RS);
  { pair_bwd_kernel<Mdl><<<g, kBW * 32, smem, st>>>(a); ++g_launches; }
  launch_combine<Mdl>(a, qstride, st);
}

template <class Mdl>
static void launch_epi_only(const ScoreArgs &a, int nout, bool train, cudaStream_t st) {
  if (nout == 1) {
    if (train) { pair_epi_kernel<Mdl, 1, true><<<a.M, 256, 0, st>>>(a); ++g_launches; }
    else { pair_epi_kernel<Mdl, 1, false><<<a.M, 256, 0, st>>>(a); ++g_launches; }
  } else {
    if (train) { pair_epi_kernel<Mdl, 2, true><<<a.M, 256, 0, st>>>(a); ++g_launches; }
    else { pair_epi_kernel<Mdl, 2, false><<<a.M, 256, 0, st>>>(a); ++g_launches; }
  }
}
void launch_pair_epi(int kind, const ScoreArgs &a, int nout, bool train, cudaStream_t st) {
  if (kind == DISTMULT) launch_epi_only<MDot>(a, nout, train, st);
  else if (kind == COMPLEX) launch_epi_only<MCpx>(a, nout, train, st);
}

void launch_pair_bwd(int kind, const ScoreArgs &a, cudaStream_t st, cudaStream_t st2) {
  switch (kind) {
    case GQE: case TRANSE: launch_bwd<ML2>(a, st, st2); break;
    case Q2B: launch_bwd<MBox>(a, st, st2); break;
    case BETAE: launch_bwd<MBeta>(a, st, st2); break;
    case ROTATE: launch_bwd<MRot>(a, st, st2); break;
    case DISTMULT: launch_bwd<MDot>(a, st, st2); break;
    case COMPLEX: launch_bwd<MCpx>(a, st, st2); break;
  }
}

template <int KIND>
static void launch_pos_k(const PosArgs &p, int nout, cudaStream_t st) {
  if (nout == 1) { pos_kernel<KIND, 1><<<p.M, 128, 0, st>>>(p); ++g_launches; }
  else { pos_kernel<KIND, 2><<<p.M, 128, 0, st>>>(p); ++g_launches; }
}

void launch_pos(int kind, const PosArgs &p, int nout, cudaStream_t st) {
  switch (kind) {
    case GQE: launch_pos_k<GQE>(p, nout, st); break;
    case TRANSE: launch_pos_k<TRANSE>(p, nout, st); break;
    case Q2B: launch_pos_k<Q2B>(p, nout, st); break;
    case BETAE: launch_pos_k<BETAE>(p, nout, st); break;
    case ROTATE: launch_pos_k<ROTATE>(p, nout, st); break;
    case DISTMULT: launch_pos_k<DISTMULT>(p, nout, st); break;
    case COMPLEX: launch_pos_k<COMPLEX>(p, nout, st); break;
  }
}

void launch_beta_entity(const float *ent, const int64_t *rows, int K, int m, float *F, float *Cv, cudaStream_t st) {
  if (K > 0) { beta_entity_kernel<<<K, 128, 0, st>>>(ent, rows, K, m, F, Cv); ++g_launches; }
}
void launch_beta_query(const float *Q, int NQ, int m, float *QP, float *Cq, cudaStream_t st) {
  { beta_query_kernel<<<NQ, 128, 0, st>>>(Q, NQ, m, QP, Cq); ++g_launches; }
}
void launch_loss_finalize(const float *loss_pos, const float *loss_part, int M, int njt, double scale,
                          double *loss_out, int *flags, int64_t *t_dev, float *bc, double beta1, double beta2,
                          int apply, cudaStream_t st, int check) {
  { loss_finalize_kernel<<<1, 256, 0, st>>>(loss_pos, loss_part, M, njt, scale, loss_out, flags, t_dev, bc,
                                          beta1, beta2, apply, check); ++g_launches; }
}

// After the cross-rank sum of the loss and max of the input flags (world > 1).
__global__ void loss_check_kernel(double *loss_out, int *flags, int64_t *t_dev, float *bc, double beta1, double beta2,
                                  int apply) {
  KG_GRID_DEP_WAIT();
  const double loss = *loss_out;
  const int bad = !isfinite(loss) || flags[1];
  flags[0] = bad;
  if (!bad && apply) {
    const int64_t t = *t_dev + 1;
    *t_dev = t;
    bc[0] = (float)(1.0 / (1.0 - pow(beta1, (double)t)));
    bc[1] = (float)(1.0 / (1.0 - pow(beta2, (double)t)));
  }
}
void launch_loss_check(double *loss_out, int *flags, int64_t *t_dev, float *bc, double beta1, double beta2, int apply,
                       cudaStream_t st) {
  { loss_check_kernel<<<1, 1, 0, st>>>(loss_out, flags, t_dev, bc, beta1, beta2, apply); ++g_launches; }
}

}  // namespace kg
