// k_eval.cu -- the evaluation path: filtered ranks and MRR / Hit@k.
//
// PAPER.md App. F: each missing answer v of a test query q is ranked
// against n_neg negatives sampled per query from V \ A_q^{G_test} (the caller's
// sampler filters them); Metrics(q) = mean_v f(Rank(v)), f = 1/x (MRR), 1[x <= k]
// (Hit@k).  Reading A26: Rank(v) = 1 + #{j : D(q, v_j) <= D(q, v)} (ties count
// against v), D = the model distance with the DNF min over the disjuncts (A11).
//
// One CTA per query: its warps compute the distances of the query to its answers and
// its negatives (lanes over the embedding units, a fixed-order warp reduction), into
// shared memory; then each thread ranks answers against the negatives held in shared
// memory (broadcast reads) and the CTA reduces the per-query metrics in a fixed
// order.  Per-query candidates share nothing across queries, so the kernel is a
// row gather (n_cand x 4d bytes per query) plus the distance arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kg.h"
#include "kg_common.cuh"
#include "kg_launch.h"

namespace kg {

// distance of disjunct row q ([QF][U]) to the raw entity row e ([d]), warp-wide
template <int KIND>
__device__ __forceinline__ float warp_dist(const float *__restrict__ q, const float *__restrict__ e, int U,
                                           float alpha, int lane) {
  float acc = 0.f;
  for (int k = lane; k < U; k += 32) {
    if (KIND == KG_GQE || KIND == KG_TRANSE) {           // ||q - v||_2 (A2)
      const float t = q[k] - e[k];
      acc = fmaf(t, t, acc);
    } else if (KIND == KG_Q2B) {                         // sum ReLU(|v-c|-o) + alpha min(|v-c|, o) (A7)
      const float t = fabsf(e[k] - q[k]);
      acc += fmaf(alpha - 1.f, fminf(t, q[U + k]), t);
    } else if (KIND == KG_BETAE) {                       // KL(Beta(e(v)) || Beta(q)) (A10)
      const float a1 = beta_act(e[k]), b1 = beta_act(e[U + k]), a2 = q[k], b2 = q[U + k];
      acc += lnbetaf_(a2, b2) - lnbetaf_(a1, b1) + (a1 - a2) * digammaf_(a1) + (b1 - b2) * digammaf_(b1) +
             (a2 - a1 + b2 - b1) * digammaf_(a1 + b1);
    } else if (KIND == KG_ROTATE) {                      // sum |q_k - t_k| (A3)
      const float x = q[k] - e[k], y = q[U + k] - e[U + k];
      acc += sqrtf(fmaf(x, x, y * y));
    } else if (KIND == KG_DISTMULT) {                    // -<h o r, t> (A13)
      acc = fmaf(-q[k], e[k], acc);
    } else {                                             // ComplEx: -Re<h o r, conj(t)> (A13)
      acc -= fmaf(q[k], e[k], q[U + k] * e[U + k]);
    }
  }
  acc = warp_sum(acc);
  if (KIND == KG_GQE || KIND == KG_TRANSE) acc = sqrtf(acc);
  return acc;
}

template <int KIND, int NOUT>
__global__ void __launch_bounds__(256) eval_rank_kernel(EvalArgs a) {
  KG_GRID_DEP_WAIT();
  extern __shared__ float sD[];   // [max_ans] answer distances, then [n_neg] negative distances
  __shared__ float red[32];
  const int i = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int64_t a0 = a.ans_off[i];
  const int na = (int)(a.ans_off[i + 1] - a0), nn = a.n_neg;
  float *dA = sD, *dN = sD + a.max_ans;
  const int qstride = (KIND == KG_Q2B ? 2 : 1) * a.d;
  for (int c = warp; c < na + nn; c += nw) {
    const int64_t id = c < na ? a.ans_ids[a0 + c] : a.negatives[(int64_t)i * nn + (c - na)];
    const float *e = a.ent + id * a.d;
    float D = warp_dist<KIND>(a.Q + (int64_t)i * qstride, e, a.U, a.alpha, lane);
#pragma unroll
    for (int t = 1; t < NOUT; ++t)   // DNF: min over the disjuncts (A11)
      D = fminf(D, warp_dist<KIND>(a.Q + ((int64_t)t * a.M + i) * qstride, e, a.U, a.alpha, lane));
    if (lane == 0) {
      if (c < na) dA[c] = D;
      else dN[c - na] = D;
    }
  }
  __syncthreads();
  float s_rr = 0.f, s_h1 = 0.f, s_h3 = 0.f, s_h10 = 0.f;
  for (int v = threadIdx.x; v < na; v += blockDim.x) {
    const float Dv = dA[v];
    int cnt = 0;
    for (int j = 0; j < nn; ++j) cnt += dN[j] <= Dv ? 1 : 0;   // ties count against v (A26)
    const int rank = 1 + cnt;
    a.ranks[a0 + v] = rank;
    s_rr += 1.f / (float)rank;
    s_h1 += rank <= 1 ? 1.f : 0.f;
    s_h3 += rank <= 3 ? 1.f : 0.f;
    s_h10 += rank <= 10 ? 1.f : 0.f;
  }
  s_rr = block_sum(s_rr, red);
  s_h1 = block_sum(s_h1, red);
  s_h3 = block_sum(s_h3, red);
  s_h10 = block_sum(s_h10, red);
  if (threadIdx.x == 0) {
    const float inv = 1.f / (float)na;
    a.metrics[4 * i + 0] = s_rr * inv;
    a.metrics[4 * i + 1] = s_h1 * inv;
    a.metrics[4 * i + 2] = s_h3 * inv;
    a.metrics[4 * i + 3] = s_h10 * inv;
  }
}

// kg_score_each: out[i][c] = D(q_i, v_cand[i][c]) (DNF min over the disjuncts, A11); one CTA per
// query, one warp per candidate (the distance of eval_rank_kernel)
template <int KIND, int NOUT>
__global__ void __launch_bounds__(256) score_each_kernel(EvalArgs a) {
  KG_GRID_DEP_WAIT();
  const int i = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nc = a.n_neg;
  const int qstride = (KIND == KG_Q2B ? 2 : 1) * a.d;
  for (int c = warp; c < nc; c += nw) {
    const float *e = a.ent + a.negatives[(int64_t)i * nc + c] * a.d;
    float D = warp_dist<KIND>(a.Q + (int64_t)i * qstride, e, a.U, a.alpha, lane);
#pragma unroll
    for (int t = 1; t < NOUT; ++t)
      D = fminf(D, warp_dist<KIND>(a.Q + ((int64_t)t * a.M + i) * qstride, e, a.U, a.alpha, lane));
    if (lane == 0) a.metrics[(int64_t)i * nc + c] = D;
  }
}
template <int KIND>
static void launch_score_each_k(const EvalArgs &a, int nout, cudaStream_t st) {
  if (nout == 2) score_each_kernel<KIND, 2><<<a.M, 256, 0, st>>>(a);
  else score_each_kernel<KIND, 1><<<a.M, 256, 0, st>>>(a);
  ++g_launches;
}
void launch_score_each(int kind, const EvalArgs &a, int nout, cudaStream_t st) {
  if (a.M <= 0 || a.n_neg <= 0) return;
  switch (kind) {
    case KG_GQE: launch_score_each_k<KG_GQE>(a, nout, st); break;
    case KG_Q2B: launch_score_each_k<KG_Q2B>(a, nout, st); break;
    case KG_BETAE: launch_score_each_k<KG_BETAE>(a, nout, st); break;
    case KG_TRANSE: launch_score_each_k<KG_TRANSE>(a, nout, st); break;
    case KG_ROTATE: launch_score_each_k<KG_ROTATE>(a, nout, st); break;
    case KG_DISTMULT: launch_score_each_k<KG_DISTMULT>(a, nout, st); break;
    default: launch_score_each_k<KG_COMPLEX>(a, nout, st); break;
  }
}

template <int KIND>
static void launch_eval_k(const EvalArgs &a, int nout, size_t smem, cudaStream_t st) {
  if (nout == 2) {
    cudaFuncSetAttribute(eval_rank_kernel<KIND, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    eval_rank_kernel<KIND, 2><<<a.M, 256, smem, st>>>(a);
  } else {
    cudaFuncSetAttribute(eval_rank_kernel<KIND, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    eval_rank_kernel<KIND, 1><<<a.M, 256, smem, st>>>(a);
  }
  ++g_launches;
}

void launch_eval(int kind, const EvalArgs &a, int nout, cudaStream_t st) {
  if (a.M <= 0) return;
  const size_t smem = sizeof(float) * ((size_t)a.max_ans + a.n_neg);
  switch (kind) {
    case KG_GQE: launch_eval_k<KG_GQE>(a, nout, smem, st); break;
    case KG_Q2B: launch_eval_k<KG_Q2B>(a, nout, smem, st); break;
    case KG_BETAE: launch_eval_k<KG_BETAE>(a, nout, smem, st); break;
    case KG_TRANSE: launch_eval_k<KG_TRANSE>(a, nout, smem, st); break;
    case KG_ROTATE: launch_eval_k<KG_ROTATE>(a, nout, smem, st); break;
    case KG_DISTMULT: launch_eval_k<KG_DISTMULT>(a, nout, smem, st); break;
    default: launch_eval_k<KG_COMPLEX>(a, nout, smem, st); break;
  }
}

}  // namespace kg
