// k_dag.cu -- query-DAG operators (SURVEY K-new-2/K-new-3): fused row gather +
// entity activation + relation projection, intersection elementwise parts
// (softmax attention, mean pooling, min offset), and their adjoints.
//
// Projection P (Table 1 'Relation Projection' P:L139-143, Table 2 P:L162-168,
// App. B; readings A3, A6, A8, A9); intersection I (Table 1
// 'Intersection', A4, A5).  The dense d x d / MLP contractions around these
// kernels run as GEMMs issued by kg_api.cu.
#include "kg_common.cuh"
#include "kg_launch.h"

namespace kg {

static inline int blocks(int64_t n, int t = 256) { return (int)((n + t - 1) / t); }

// ------------------------------------------------------------ projection fwd
// One thread per (query i, unit k).  `anchor_rows` != nullptr: the input is the
// raw theta_E row of the anchor (fused gather; anchors are points, A6).
template <int KIND>
__global__ void proj_fwd_kernel(int N, int d, const float *in, int64_t in_ld, const int64_t *anchor_rows,
                                const float *ent, const int32_t *rel, int rel_ld, const float *relA,
                                const float *relB, float *out) {
  KG_GRID_DEP_WAIT();
  const int U = (KIND == COMPLEX || KIND == ROTATE) ? d / 2 : d;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)N * U) return;
  const int i = (int)(e / U), k = (int)(e - (int64_t)i * U);
  const int r = rel[(int64_t)i * rel_ld];
  const float *h = anchor_rows ? ent + anchor_rows[i] * (int64_t)d : in + i * in_ld;
  if (KIND == GQE || KIND == TRANSE) {
    out[(int64_t)i * d + k] = h[k] + relA[(int64_t)r * d + k];
  } else if (KIND == Q2B) {
    const float c = h[k], o = anchor_rows ? 0.f : h[d + k];
    out[(int64_t)i * 2 * d + k] = c + relA[(int64_t)r * d + k];
    out[(int64_t)i * 2 * d + d + k] = o + fmaxf(relB[(int64_t)r * d + k], 0.f);
  } else if (KIND == DISTMULT) {
    out[(int64_t)i * d + k] = h[k] * relA[(int64_t)r * d + k];
  } else if (KIND == COMPLEX) {
    const float hr = h[k], hi = h[U + k], rr = relA[(int64_t)r * d + k], ri = relA[(int64_t)r * d + U + k];
    out[(int64_t)i * d + k] = hr * rr - hi * ri;
    out[(int64_t)i * d + U + k] = hr * ri + hi * rr;
  } else if (KIND == ROTATE) {
    float s, c;
    sincosf(relA[(int64_t)r * U + k], &s, &c);
    const float hr = h[k], hi = h[U + k];
    out[(int64_t)i * d + k] = hr * c - hi * s;
    out[(int64_t)i * d + U + k] = hr * s + hi * c;
  }
}

template <int KIND>
__global__ void proj_bwd_kernel(int N, int d, const float *dout, const float *in, int64_t in_ld,
                                const int64_t *anchor_rows, const float *ent, const int32_t *rel, int rel_ld,
                                const float *relA, const float *relB, const float *out, float *din, int64_t din_ld,
                                float *drel) {
  KG_GRID_DEP_WAIT();
  const int U = (KIND == COMPLEX || KIND == ROTATE) ? d / 2 : d;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)N * U) return;
  const int i = (int)(e / U), k = (int)(e - (int64_t)i * U);
  const int r = rel[(int64_t)i * rel_ld];
  const float *h = anchor_rows ? ent + anchor_rows[i] * (int64_t)d : in + i * in_ld;
  float *di = din + i * din_ld;
  if (KIND == GQE || KIND == TRANSE) {
    const float g = dout[(int64_t)i * d + k];
    di[k] = g;
    drel[(int64_t)i * d + k] = g;
  } else if (KIND == Q2B) {
    const float gc = dout[(int64_t)i * 2 * d + k], go = dout[(int64_t)i * 2 * d + d + k];
    di[k] = gc;
    if (!anchor_rows) di[d + k] = go;           // an anchor's offset is the constant 0 (A6)
    drel[(int64_t)i * 2 * d + k] = gc;
    drel[(int64_t)i * 2 * d + d + k] = relB[(int64_t)r * d + k] > 0.f ? go : 0.f;   // ReLU'(0) = 0 (A19)
  } else if (KIND == DISTMULT) {
    const float g = dout[(int64_t)i * d + k];
    di[k] = g * relA[(int64_t)r * d + k];
    drel[(int64_t)i * d + k] = g * h[k];
  } else if (KIND == COMPLEX) {
    const float gr = dout[(int64_t)i * d + k], gi = dout[(int64_t)i * d + U + k];
    const float hr = h[k], hi = h[U + k], rr = relA[(int64_t)r * d + k], ri = relA[(int64_t)r * d + U + k];
    di[k] = gr * rr + gi * ri;
    di[U + k] = -gr * ri + gi * rr;
    drel[(int64_t)i * d + k] = gr * hr + gi * hi;
    drel[(int64_t)i * d + U + k] = -gr * hi + gi * hr;
  } else if (KIND == ROTATE) {
    float s, c;
    sincosf(relA[(int64_t)r * U + k], &s, &c);
    const float gr = dout[(int64_t)i * d + k], gi = dout[(int64_t)i * d + U + k];
    di[k] = gr * c + gi * s;                     // inverse rotation
    di[U + k] = -gr * s + gi * c;
    const float qr = out[(int64_t)i * d + k], qi = out[(int64_t)i * d + U + k];
    drel[(int64_t)i * U + k] = -gr * qi + gi * qr;   // d q / d theta = i q
  }
}

void launch_proj_fwd(int kind, int N, int d, const float *in, int64_t in_ld, const int64_t *anchor_rows,
                     const float *ent, const int32_t *rel, int rel_ld, const float *relA, const float *relB,
                     float *out, cudaStream_t st) {
  const int U = (kind == COMPLEX || kind == ROTATE) ? d / 2 : d;
  const int g = blocks((int64_t)N * U);
#define ARGS N, d, in, in_ld, anchor_rows, ent, rel, rel_ld, relA, relB, out
  switch (kind) {
    case GQE: { proj_fwd_kernel<GQE><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    case TRANSE: { proj_fwd_kernel<TRANSE><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    case Q2B: { proj_fwd_kernel<Q2B><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    case DISTMULT: { proj_fwd_kernel<DISTMULT><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    case COMPLEX: { proj_fwd_kernel<COMPLEX><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    case ROTATE: { proj_fwd_kernel<ROTATE><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    default: break;
  }
#undef ARGS
}

void launch_proj_bwd(int kind, int N, int d, const float *dout, const float *in, int64_t in_ld,
                     const int64_t *anchor_rows, const float *ent, const int32_t *rel, int rel_ld, const float *relA,
                     const float *relB, const float *out, float *din, int64_t din_ld, float *drel, cudaStream_t st) {
  const int U = (kind == COMPLEX || kind == ROTATE) ? d / 2 : d;
  const int g = blocks((int64_t)N * U);
#define ARGS N, d, dout, in, in_ld, anchor_rows, ent, rel, rel_ld, relA, relB, out, din, din_ld, drel
  switch (kind) {
    case GQE: { proj_bwd_kernel<GQE><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    case TRANSE: { proj_bwd_kernel<TRANSE><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    case Q2B: { proj_bwd_kernel<Q2B><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    case DISTMULT: { proj_bwd_kernel<DISTMULT><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    case COMPLEX: { proj_bwd_kernel<COMPLEX><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    case ROTATE: { proj_bwd_kernel<ROTATE><<<g, 256, 0, st>>>(ARGS); ++g_launches; } break;
    default: break;
  }
#undef ARGS
}

// sum of the raw split-K partial products [S][..] at element e, in ascending split order
__device__ __forceinline__ float psum(const float *P, int S, int64_t zs, int64_t e) {
  float v = P[e];
  for (int z = 1; z < S; ++z) v += P[z * zs + e];
  return v;
}

// ------------------------------------------------------------ BetaE MLP glue
// X[i] = [e_q(i) ; y_r(i)]  (A9), e_q = node value or clamp(x_anchor + 1) (A8)
__global__ void betae_proj_in_kernel(int N, int d, const float *in, const int64_t *anchor_rows, const float *ent,
                                     const int32_t *rel, int rel_ld, const float *relT, float *X) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)N * d) return;
  const int i = (int)(e / d), k = (int)(e - (int64_t)i * d);
  const float q = anchor_rows ? beta_act(ent[anchor_rows[i] * (int64_t)d + k]) : in[(int64_t)i * d + k];
  X[(int64_t)i * 2 * d + k] = q;
  X[(int64_t)i * 2 * d + d + k] = relT[(int64_t)rel[(int64_t)i * rel_ld] * d + k];
}
void launch_betae_proj_in(int N, int d, const float *in, const int64_t *anchor_rows, const float *ent,
                          const int32_t *rel, int rel_ld, const float *relT, float *X, cudaStream_t st) {
  { betae_proj_in_kernel<<<blocks((int64_t)N * d), 256, 0, st>>>(N, d, in, anchor_rows, ent, rel, rel_ld, relT, X); ++g_launches; }
}

// Y = act(Y + b) row-wise; act 1 = ReLU, 0 = identity.
__global__ void bias_act_kernel(float *Y, const float *b, int rows, int cols, int act) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)rows * cols) return;
  const float v = Y[e] + b[e % cols];
  Y[e] = act ? fmaxf(v, 0.f) : v;
}
void launch_bias_act(float *Y, const float *b, int rows, int cols, int act, cudaStream_t st) {
  { bias_act_kernel<<<blocks((int64_t)rows * cols), 256, 0, st>>>(Y, b, rows, cols, act); ++g_launches; }
}

__global__ void betae_proj_out_kernel(const float *Z, const float *b0, int rows, int d, float *Zp1, float *out) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)rows * d) return;
  const float z = Z[e] + b0[e % d] + 1.f;
  Zp1[e] = z;
  out[e] = fminf(fmaxf(z, kBetaLo), kBetaHi);
}
void launch_betae_proj_out(const float *Z, const float *b0, int rows, int d, float *Zp1, float *out,
                           cudaStream_t st) {
  { betae_proj_out_kernel<<<blocks((int64_t)rows * d), 256, 0, st>>>(Z, b0, rows, d, Zp1, out); ++g_launches; }
}

// the same from the raw split-K partials of Z = H2 W0^T over the rows of a projection group
// (fused epilogue, k_dag.cu *_red): z = (sum_z P) + b0 + 1; projection g of the group (rows
// [g M, (g + 1) M)) writes its node value out.p[g]
__global__ void betae_proj_out_red_kernel(const float *P, int S, const float *b0, int rows, int M, int d, float *Zp1,
                                          OutPtrs out) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)rows * d;
  if (e >= n) return;
  const float z = psum(P, S, n, e) * 1.f + b0[e % d] + 1.f;
  Zp1[e] = z;
  const int64_t Md = (int64_t)M * d, g = e / Md;
  out.p[g][e - g * Md] = fminf(fmaxf(z, kBetaLo), kBetaHi);
}
void launch_betae_proj_out_red(const float *P, int S, const float *b0, int rows, int M, int d, float *Zp1,
                               const OutPtrs &out, cudaStream_t st) {
  { betae_proj_out_red_kernel<<<blocks((int64_t)rows * d), 256, 0, st>>>(P, S, b0, rows, M, d, Zp1, out); ++g_launches; }
}

__global__ void betae_proj_dz_kernel(const float *dout, const float *Zp1, int rows, int d, float *dZ) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)rows * d) return;
  const float z = Zp1[e];
  dZ[e] = (z >= kBetaLo && z <= kBetaHi) ? dout[e] : 0.f;
}
void launch_betae_proj_dz(const float *dout, const float *Zp1, int rows, int d, float *dZ, cudaStream_t st) {
  { betae_proj_dz_kernel<<<blocks((int64_t)rows * d), 256, 0, st>>>(dout, Zp1, rows, d, dZ); ++g_launches; }
}

__global__ void relu_mask_kernel(float *dY, const float *Y, int64_t n) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n && !(Y[e] > 0.f)) dY[e] = 0.f;
}
void launch_relu_mask(float *dY, const float *Y, int rows, int cols, cudaStream_t st) {
  { relu_mask_kernel<<<blocks((int64_t)rows * cols), 256, 0, st>>>(dY, Y, (int64_t)rows * cols); ++g_launches; }
}

// dX [N][2d] -> din (query part; raw-row gradient through the clamp for anchors) and drel.
__global__ void betae_split_kernel(const float *dX, int N, int d, const int64_t *anchor_rows, const float *ent,
                                   float *din, int64_t din_ld, float *drel) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)N * d) return;
  const int i = (int)(e / d), k = (int)(e - (int64_t)i * d);
  float g = dX[(int64_t)i * 2 * d + k];
  if (anchor_rows) g *= beta_act_grad(ent[anchor_rows[i] * (int64_t)d + k]);
  din[i * din_ld + k] = g;
  drel[(int64_t)i * d + k] = dX[(int64_t)i * 2 * d + d + k];
}
void launch_betae_split(const float *dX, int N, int d, const int64_t *anchor_rows, const float *ent, float *din,
                        int64_t din_ld, float *drel, cudaStream_t st) {
  { betae_split_kernel<<<blocks((int64_t)N * d), 256, 0, st>>>(dX, N, d, anchor_rows, ent, din, din_ld, drel); ++g_launches; }
}

// ------------------------------------------------------------ -m query normalisation (A27)
// App. B: DistMult-m q <- q / ||q||_2 (parts = 1); ComplEx-m Re and Im halves each to the
// unit sphere (parts = 2).  One warp per (row, part), in place; the norms are kept for the
// adjoint g <- (g - y (y . g)) / ||x|| (y the normalised value).
__global__ void qnorm_fwd_kernel(float *X, int M, int d, int parts, float *nrm) {
  KG_GRID_DEP_WAIT();
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (w >= M * parts) return;
  const int L = d / parts;
  float *x = X + (int64_t)(w / parts) * d + (w % parts) * L;
  float s = 0.f;
  for (int k = lane; k < L; k += 32) s = fmaf(x[k], x[k], s);
  const float n = sqrtf(warp_sum(s));
  const float inv = 1.f / n;
  for (int k = lane; k < L; k += 32) x[k] *= inv;
  if (lane == 0) nrm[2 * (w / parts) + (w % parts)] = n;
}
__global__ void qnorm_bwd_kernel(float *G, const float *Y, int M, int d, int parts, const float *nrm) {
  KG_GRID_DEP_WAIT();
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (w >= M * parts) return;
  const int L = d / parts;
  const int64_t o = (int64_t)(w / parts) * d + (w % parts) * L;
  float *g = G + o;
  const float *y = Y + o;
  float s = 0.f;
  for (int k = lane; k < L; k += 32) s = fmaf(y[k], g[k], s);
  s = warp_sum(s);
  const float inv = 1.f / nrm[2 * (w / parts) + (w % parts)];
  for (int k = lane; k < L; k += 32) g[k] = (g[k] - y[k] * s) * inv;
}
void launch_qnorm_fwd(float *X, int M, int d, int parts, float *nrm, cudaStream_t st) {
  const int64_t threads = (int64_t)M * parts * 32;
  { qnorm_fwd_kernel<<<blocks(threads), 256, 0, st>>>(X, M, d, parts, nrm); ++g_launches; }
}
void launch_qnorm_bwd(float *G, const float *Y, int M, int d, int parts, const float *nrm, cudaStream_t st) {
  const int64_t threads = (int64_t)M * parts * 32;
  { qnorm_bwd_kernel<<<blocks(threads), 256, 0, st>>>(G, Y, M, d, parts, nrm); ++g_launches; }
}

// ------------------------------------------------------------ negation (BetaE)
// N(q) = 1/q elementwise on (alpha, beta) (Table 1 'Negation' P:L143); adjoint -g/q^2.
__global__ void neg_fwd_kernel(const float *in, int64_t n, float *out) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) out[e] = 1.f / in[e];
}
__global__ void neg_bwd_kernel(const float *dout, const float *in, int64_t n, float *din) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) {
    const float x = in[e];
    din[e] = -dout[e] / (x * x);
  }
}
void launch_neg_fwd(const float *in, int64_t n, float *out, cudaStream_t st) {
  if (n > 0) { neg_fwd_kernel<<<blocks(n), 256, 0, st>>>(in, n, out); ++g_launches; }
}
void launch_neg_bwd(const float *dout, const float *in, int64_t n, float *din, cudaStream_t st) {
  if (n > 0) { neg_bwd_kernel<<<blocks(n), 256, 0, st>>>(dout, in, n, din); ++g_launches; }
}

// ------------------------------------------------------------ intersections
__global__ void mean_stack_kernel(const float *H, int n, int64_t rc, float *out) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= rc) return;
  float s = 0.f;
  for (int t = 0; t < n; ++t) s += H[t * rc + e];
  out[e] = s / (float)n;
}
void launch_mean_stack(const float *H, int n, int rows, int cols, float *out, cudaStream_t st) {
  const int64_t rc = (int64_t)rows * cols;
  { mean_stack_kernel<<<blocks(rc), 256, 0, st>>>(H, n, rc, out); ++g_launches; }
}

// dH_t = dMn / n * [H_t > 0]   (DeepSet mean pooling + ReLU adjoint, A4)
__global__ void gqe_inter_dh_kernel(const float *dMn, const float *H, int n, int64_t rc, float *dH) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= rc * n) return;
  dH[e] = H[e] > 0.f ? dMn[e % rc] / (float)n : 0.f;
}
void launch_gqe_inter_dh(const float *dMn, const float *H, int n, int rows, int cols, float *dH, cudaStream_t st) {
  const int64_t rc = (int64_t)rows * cols;
  { gqe_inter_dh_kernel<<<blocks(rc * n), 256, 0, st>>>(dMn, H, n, rc, dH); ++g_launches; }
}

// ---- the intersection MLPs' GEMM epilogues fused with their consumers.  P holds the raw
// split-K partial products [S][rows][d] of a GEMM (launch_gemm_tc_raw); each kernel sums them in
// ascending split order and adds the bias exactly as gemm_reduce_kernel does, then applies the
// node's pooling in the order of the kernels above it replaces (mean_stack, q2b_off_fwd,
// q2b_att_fwd): the values are bitwise those of the unfused chain.
// DeepSet layer 1 + mean pooling (A4): H_t = ReLU(P_t + b), Mn = (sum_t H_t) / n
__global__ void mean_red_kernel(const float *P, int S, const float *b, int n, int M, int d, float *H, float *Mn) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t Md = (int64_t)M * d;
  if (e >= Md) return;
  const int k = (int)(e % d);
  const int64_t zs = (int64_t)n * Md;
  float s = 0.f;
  for (int t = 0; t < n; ++t) {
    const float h = fmaxf(psum(P, S, zs, t * Md + e) * 1.f + b[k], 0.f);
    H[t * Md + e] = h;
    s += h;
  }
  Mn[e] = s / (float)n;
}
void launch_mean_red(const float *P, int S, const float *b, int n, int M, int d, float *H, float *Mn, cudaStream_t st) {
  { mean_red_kernel<<<blocks((int64_t)M * d), 256, 0, st>>>(P, S, b, n, M, d, H, Mn); ++g_launches; }
}
// Q2B offset: Z = P + b, o = min_t o_t * sigmoid(Z) (Table 1), argmin ties -> lowest t (A19)
__global__ void q2b_off_red_kernel(const float *P, int S, const float *b, const float *stack, int n, int M, int d,
                                   float *sig, int8_t *amin, float *out) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t Md = (int64_t)M * d;
  if (e >= Md) return;
  const int i = (int)(e / d), k = (int)(e - (int64_t)i * d);
  float mn = stack[(int64_t)i * 2 * d + d + k];
  int am = 0;
  for (int t = 1; t < n; ++t) {
    const float o = stack[((int64_t)t * M + i) * 2 * d + d + k];
    if (o < mn) { mn = o; am = t; }
  }
  const float s = sigm_(psum(P, S, Md, e) * 1.f + b[k]);
  sig[e] = s;
  amin[e] = (int8_t)am;
  out[(int64_t)i * 2 * d + d + k] = mn * s;
}
void launch_q2b_off_red(const float *P, int S, const float *b, const float *stack, int n, int M, int d, float *sig,
                        int8_t *amin, float *out, cudaStream_t st) {
  { q2b_off_red_kernel<<<blocks((int64_t)M * d), 256, 0, st>>>(P, S, b, stack, n, M, d, sig, amin, out); ++g_launches; }
}
// Q2B center attention: Lg_t = P_t + b, a_t = softmax_t(Lg_t) per (i, k), c = sum_t a_t c_t (A5)
__global__ void q2b_att_red_kernel(const float *P, int S, const float *b, const float *stack, int n, int M, int d,
                                   float *a, float *out) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t Md = (int64_t)M * d;
  if (e >= Md) return;
  const int i = (int)(e / d), k = (int)(e - (int64_t)i * d);
  const int64_t zs = (int64_t)n * Md;
  float lg[3], mx = -INFINITY;
  for (int t = 0; t < n; ++t) {
    lg[t] = psum(P, S, zs, t * Md + e) * 1.f + b[k];
    mx = fmaxf(mx, lg[t]);
  }
  float z = 0.f, ex[3];
  for (int t = 0; t < n; ++t) { ex[t] = expf(lg[t] - mx); z += ex[t]; }
  float c = 0.f;
  for (int t = 0; t < n; ++t) {
    const float at = ex[t] / z;
    a[t * Md + e] = at;
    c += at * stack[((int64_t)t * M + i) * 2 * d + k];
  }
  out[(int64_t)i * 2 * d + k] = c;
}
void launch_q2b_att_red(const float *P, int S, const float *b, const float *stack, int n, int M, int d, float *a,
                        float *out, cudaStream_t st) {
  { q2b_att_red_kernel<<<blocks((int64_t)M * d), 256, 0, st>>>(P, S, b, stack, n, M, d, a, out); ++g_launches; }
}
// BetaE attention: Lg_t = P_t + c2 (m per row), w = softmax_t(Lg_t), out = (sum w a_t, sum w b_t)
__global__ void beta_att_red_kernel(const float *P, int S, const float *b, const float *stack, int n, int M, int d,
                                    float *w, float *out) {
  KG_GRID_DEP_WAIT();
  const int m = d / 2;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t Mm = (int64_t)M * m;
  if (e >= Mm) return;
  const int i = (int)(e / m), k = (int)(e - (int64_t)i * m);
  const int64_t zs = (int64_t)n * Mm;
  float lg[3], mx = -INFINITY;
  for (int t = 0; t < n; ++t) {
    lg[t] = psum(P, S, zs, t * Mm + e) * 1.f + b[k];
    mx = fmaxf(mx, lg[t]);
  }
  float z = 0.f, ex[3];
  for (int t = 0; t < n; ++t) { ex[t] = expf(lg[t] - mx); z += ex[t]; }
  float sa = 0.f, sb = 0.f;
  for (int t = 0; t < n; ++t) {
    const float wt = ex[t] / z;
    w[t * Mm + e] = wt;
    const float *row = stack + ((int64_t)t * M + i) * d;
    sa += wt * row[k];
    sb += wt * row[m + k];
  }
  out[(int64_t)i * d + k] = sa;
  out[(int64_t)i * d + m + k] = sb;
}
void launch_beta_att_red(const float *P, int S, const float *b, const float *stack, int n, int M, int d, float *w,
                         float *out, cudaStream_t st) {
  { beta_att_red_kernel<<<blocks((int64_t)M * (d / 2)), 256, 0, st>>>(P, S, b, stack, n, M, d, w, out); ++g_launches; }
}

// Q2B center attention: a_t = softmax_t(Lg_t) per (i, k); c = sum_t a_t c_t (A5).
__global__ void q2b_att_fwd_kernel(const float *stack, const float *Lg, int n, int M, int d, float *a, float *out) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t Md = (int64_t)M * d;
  if (e >= Md) return;
  const int i = (int)(e / d), k = (int)(e - (int64_t)i * d);
  float mx = -INFINITY;
  for (int t = 0; t < n; ++t) mx = fmaxf(mx, Lg[t * Md + e]);
  float z = 0.f, ex[3];
  for (int t = 0; t < n; ++t) { ex[t] = expf(Lg[t * Md + e] - mx); z += ex[t]; }
  float c = 0.f;
  for (int t = 0; t < n; ++t) {
    const float at = ex[t] / z;
    a[t * Md + e] = at;
    c += at * stack[((int64_t)t * M + i) * 2 * d + k];
  }
  out[(int64_t)i * 2 * d + k] = c;
}
void launch_q2b_att_fwd(const float *stack, const float *Lg, int n, int M, int d, float *a, float *out,
                        cudaStream_t st) {
  { q2b_att_fwd_kernel<<<blocks((int64_t)M * d), 256, 0, st>>>(stack, Lg, n, M, d, a, out); ++g_launches; }
}

// Q2B offset: o = min_t o_t * sigmoid(Z)  (Table 1), argmin ties -> lowest t (A19).
__global__ void q2b_off_fwd_kernel(const float *stack, const float *Z, int n, int M, int d, float *sig, int8_t *amin,
                                   float *out) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * d) return;
  const int i = (int)(e / d), k = (int)(e - (int64_t)i * d);
  float mn = stack[(int64_t)i * 2 * d + d + k];
  int am = 0;
  for (int t = 1; t < n; ++t) {
    const float o = stack[((int64_t)t * M + i) * 2 * d + d + k];
    if (o < mn) { mn = o; am = t; }
  }
  const float s = sigm_(Z[e]);
  sig[e] = s;
  amin[e] = (int8_t)am;
  out[(int64_t)i * 2 * d + d + k] = mn * s;
}
void launch_q2b_off_fwd(const float *stack, const float *Z, int n, int M, int d, float *sig, int8_t *amin,
                        float *out, cudaStream_t st) {
  { q2b_off_fwd_kernel<<<blocks((int64_t)M * d), 256, 0, st>>>(stack, Z, n, M, d, sig, amin, out); ++g_launches; }
}

__global__ void q2b_att_bwd_kernel(const float *stack, const float *a, const float *dout, int n, int M, int d,
                                   float *dLg, float *dstack) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t Md = (int64_t)M * d;
  if (e >= Md) return;
  const int i = (int)(e / d), k = (int)(e - (int64_t)i * d);
  const float dc = dout[(int64_t)i * 2 * d + k];
  float g[3], s = 0.f;
  for (int t = 0; t < n; ++t) {
    g[t] = dc * stack[((int64_t)t * M + i) * 2 * d + k];
    s += a[t * Md + e] * g[t];
  }
  for (int t = 0; t < n; ++t) {
    const float at = a[t * Md + e];
    dLg[t * Md + e] = at * (g[t] - s);                        // softmax adjoint
    dstack[((int64_t)t * M + i) * 2 * d + k] = at * dc;       // direct term (GEMM adds the MLP term)
  }
}
void launch_q2b_att_bwd(const float *stack, const float *a, const float *dout, int n, int M, int d, float *dLg,
                        float *dstack, cudaStream_t st) {
  { q2b_att_bwd_kernel<<<blocks((int64_t)M * d), 256, 0, st>>>(stack, a, dout, n, M, d, dLg, dstack); ++g_launches; }
}

__global__ void q2b_off_bwd_kernel(const float *stack, const float *sig, const int8_t *amin, const float *dout, int n,
                                   int M, int d, float *dZ, float *dstack) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * d) return;
  const int i = (int)(e / d), k = (int)(e - (int64_t)i * d);
  const float go = dout[(int64_t)i * 2 * d + d + k], s = sig[e];
  const int am = amin[e];
  const float mn = stack[((int64_t)am * M + i) * 2 * d + d + k];
  dZ[e] = go * mn * s * (1.f - s);
  for (int t = 0; t < n; ++t) dstack[((int64_t)t * M + i) * 2 * d + d + k] = (t == am) ? go * s : 0.f;
}
void launch_q2b_off_bwd(const float *stack, const float *sig, const int8_t *amin, const float *dout, int n, int M,
                        int d, float *dZ, float *dstack, cudaStream_t st) {
  { q2b_off_bwd_kernel<<<blocks((int64_t)M * d), 256, 0, st>>>(stack, sig, amin, dout, n, M, d, dZ, dstack); ++g_launches; }
}

// BetaE attention: w = softmax_t(Lg_t) (m per row), out = (sum w a_t, sum w b_t) (Table 1, A5).
__global__ void beta_att_fwd_kernel(const float *stack, const float *Lg, int n, int M, int d, float *w, float *out) {
  KG_GRID_DEP_WAIT();
  const int m = d / 2;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t Mm = (int64_t)M * m;
  if (e >= Mm) return;
  const int i = (int)(e / m), k = (int)(e - (int64_t)i * m);
  float mx = -INFINITY;
  for (int t = 0; t < n; ++t) mx = fmaxf(mx, Lg[t * Mm + e]);
  float z = 0.f, ex[3];
  for (int t = 0; t < n; ++t) { ex[t] = expf(Lg[t * Mm + e] - mx); z += ex[t]; }
  float sa = 0.f, sb = 0.f;
  for (int t = 0; t < n; ++t) {
    const float wt = ex[t] / z;
    w[t * Mm + e] = wt;
    const float *row = stack + ((int64_t)t * M + i) * d;
    sa += wt * row[k];
    sb += wt * row[m + k];
  }
  out[(int64_t)i * d + k] = sa;
  out[(int64_t)i * d + m + k] = sb;
}
void launch_beta_att_fwd(const float *stack, const float *Lg, int n, int M, int d, float *w, float *out,
                         cudaStream_t st) {
  { beta_att_fwd_kernel<<<blocks((int64_t)M * (d / 2)), 256, 0, st>>>(stack, Lg, n, M, d, w, out); ++g_launches; }
}

__global__ void beta_att_bwd_kernel(const float *stack, const float *w, const float *dout, int n, int M, int d,
                                    float *dLg, float *dstack) {
  KG_GRID_DEP_WAIT();
  const int m = d / 2;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t Mm = (int64_t)M * m;
  if (e >= Mm) return;
  const int i = (int)(e / m), k = (int)(e - (int64_t)i * m);
  const float da = dout[(int64_t)i * d + k], db = dout[(int64_t)i * d + m + k];
  float g[3], s = 0.f;
  for (int t = 0; t < n; ++t) {
    const float *row = stack + ((int64_t)t * M + i) * d;
    g[t] = da * row[k] + db * row[m + k];
    s += w[t * Mm + e] * g[t];
  }
  for (int t = 0; t < n; ++t) {
    const float wt = w[t * Mm + e];
    dLg[t * Mm + e] = wt * (g[t] - s);
    float *drow = dstack + ((int64_t)t * M + i) * d;
    drow[k] = wt * da;
    drow[m + k] = wt * db;
  }
}
void launch_beta_att_bwd(const float *stack, const float *w, const float *dout, int n, int M, int d, float *dLg,
                         float *dstack, cudaStream_t st) {
  { beta_att_bwd_kernel<<<blocks((int64_t)M * (d / 2)), 256, 0, st>>>(stack, w, dout, n, M, d, dLg, dstack); ++g_launches; }
}

// ------------------------------------------------------------ misc
__global__ void scale_copy_kernel(float *dst, const float *src, int64_t n, float s) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) dst[e] = src[e] * s;
}
void launch_scale_copy(float *dst, const float *src, int64_t n, float s, cudaStream_t st) {
  if (n > 0) { scale_copy_kernel<<<blocks(n), 256, 0, st>>>(dst, src, n, s); ++g_launches; }
}

__global__ void gather_rows_kernel(float *dst, const float *src, const int64_t *rows, int n, int d) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * d) return;
  const int i = (int)(e / d), k = (int)(e - (int64_t)i * d);
  dst[e] = src[rows[i] * (int64_t)d + k];
}
void launch_gather_rows(float *dst, const float *src, const int64_t *rows, int n, int d, cudaStream_t st) {
  if (n > 0) { gather_rows_kernel<<<blocks((int64_t)n * d), 256, 0, st>>>(dst, src, rows, n, d); ++g_launches; }
}
__global__ void scatter_rows_kernel(float *dst, const float *src, const int64_t *rows, int n, int d) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * d) return;
  const int i = (int)(e / d), k = (int)(e - (int64_t)i * d);
  dst[rows[i] * (int64_t)d + k] = src[e];
}
void launch_scatter_rows(float *dst, const float *src, const int64_t *rows, int n, int d, cudaStream_t st) {
  if (n > 0) { scatter_rows_kernel<<<blocks((int64_t)n * d), 256, 0, st>>>(dst, src, rows, n, d); ++g_launches; }
}

// ids = concat(anchors (slot-major: position a*M + i), answers, negatives) -- the
// occurrence order of the merge (A16); rows_out = local row = id / world;
// out-of-range ids raise bad[0] (device-side validation of device inputs).
__global__ void ids_concat_kernel(const int64_t *anchors, int na, int M, const int64_t *answers, int n_ans,
                                  const int64_t *negs, int K, int world, int64_t *ids, int64_t *rows_out,
                                  int32_t *bad, int64_t n_entities) {
  KG_GRID_DEP_WAIT();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int nai = na * M, L = nai + n_ans + K;
  if (p >= L) return;
  int64_t id;
  if (p < nai) { const int a = p / M, i = p - a * M; id = anchors[(int64_t)i * na + a]; }
  else if (p < nai + n_ans) id = answers[p - nai];
  else id = negs[p - nai - n_ans];
  if (id < 0 || id >= n_entities) { bad[0] = 1; id = 0; }
  ids[p] = id;
  rows_out[p] = id / world;
}
void launch_ids_concat(const int64_t *anchors, int na, int M, const int64_t *answers, int n_ans, const int64_t *negs,
                       int K, int world, int64_t *ids, int64_t *rows_out, int32_t *bad, int64_t n_entities,
                       cudaStream_t st) {
  const int L = na * M + n_ans + K;
  if (L > 0)
    { ids_concat_kernel<<<blocks(L), 256, 0, st>>>(anchors, na, M, answers, n_ans, negs, K, world, ids, rows_out, bad,
                                                 n_entities); ++g_launches; }
}

// Both of the step's index kernels in one launch: threads [0, L) do ids_concat_kernel's work,
// threads [L, L + nproj M) rel_occ_kernel's (the same per-element code).
__global__ void ids_rel_kernel(const int64_t *anchors, int na, int M, const int64_t *answers, int n_ans,
                               const int64_t *negs, int K, int world, int64_t *ids, int64_t *rows_out,
                               int64_t n_entities, const int32_t *relations, int nr, Slots4 slots, int nproj,
                               int n_rel, int32_t *occ, int32_t *bad) {
  KG_GRID_DEP_WAIT();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int nai = na * M, L = nai + n_ans + K;
  if (p < L) {
    int64_t id;
    if (p < nai) { const int a = p / M, i = p - a * M; id = anchors[(int64_t)i * na + a]; }
    else if (p < nai + n_ans) id = answers[p - nai];
    else id = negs[p - nai - n_ans];
    if (id < 0 || id >= n_entities) { bad[0] = 1; id = 0; }
    ids[p] = id;
    rows_out[p] = id / world;
    return;
  }
  const int e = p - L;
  if (e >= nproj * M) return;
  const int u = e / M, i = e - u * M;
  int r = relations[(int64_t)i * nr + slots.s[u]];
  if (r < 0 || r >= n_rel) { bad[0] = 1; r = 0; }
  occ[e] = r;
}
void launch_ids_rel(const int64_t *anchors, int na, int M, const int64_t *answers, int n_ans, const int64_t *negs,
                    int K, int world, int64_t *ids, int64_t *rows_out, int64_t n_entities, const int32_t *relations,
                    int nr, Slots4 slots, int nproj, int n_rel, int32_t *occ, int32_t *bad, cudaStream_t st) {
  const int n = na * M + n_ans + K + nproj * M;
  if (n > 0)
    { ids_rel_kernel<<<blocks(n), 256, 0, st>>>(anchors, na, M, answers, n_ans, negs, K, world, ids, rows_out,
                                              n_entities, relations, nr, slots, nproj, n_rel, occ, bad); ++g_launches; }
}

// occ[u*M + i] = relations[i][slot_u] (one relation occurrence per projection use).
__global__ void rel_occ_kernel(const int32_t *relations, int M, int nr, Slots4 slots, int nproj, int n_rel,
                               int32_t *occ, int32_t *bad) {
  KG_GRID_DEP_WAIT();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nproj * M) return;
  const int u = e / M, i = e - u * M;
  int r = relations[(int64_t)i * nr + slots.s[u]];
  if (r < 0 || r >= n_rel) { bad[0] = 1; r = 0; }
  occ[e] = r;
}
void launch_rel_occ(const int32_t *relations, int M, int nr, Slots4 slots, int nproj, int n_rel, int32_t *occ,
                    int32_t *bad, cudaStream_t st) {
  { rel_occ_kernel<<<blocks((int64_t)nproj * M), 256, 0, st>>>(relations, M, nr, slots, nproj, n_rel, occ, bad); ++g_launches; }
}

}  // namespace kg
