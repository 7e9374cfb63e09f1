// kg_launch.h -- host-side launchers of the sm_100a kernels (internal to libkg.so).
#pragma once
#include <functional>
#include <cuda_runtime.h>
#include <stdint.h>

namespace kg {

struct Slots4 { int s[4]; };

constexpr int kMaxWorld = 8;   // ranks supported by the row-sharded exchange

extern int64_t g_launches;   // kernels of this library enqueued so far (per process)

struct ScoreArgs {
  const float *Q = nullptr;     // [NQ][QF*U] query features (NQ = nout*M)
  int NQ = 0, M = 0, K = 0, Kp = 0, U = 0, d = 0;
  const float *E = nullptr;     // entity rows (raw theta_E) or BetaE feature rows
  const int64_t *eidx = nullptr;  // [K] row index into E (nullptr: identity)
  int64_t estride = 0;
  const uint32_t *mask = nullptr;
  int W = 0;
  const float *Cq = nullptr, *Cv = nullptr, *QP = nullptr;
  float gamma = 0.f, alpha = 0.f, scale = 0.f;
  float *C = nullptr;           // [NQ][Kp] adjoint coefficients
  float *Dmin = nullptr;        // train: [M][K] (optional); score: [M][ldo]
  int ldo = 0;
  float *loss_part = nullptr;   // [M] negative-term sum of each query
  float *dQ = nullptr;          // [NQ][QF*U]
  float *dV = nullptr;          // raw-row gradients of the pool, [K][d]
  // split-reduction partials (see k_score.cu) and their capacities (floats)
  float *Dpart = nullptr, *partQ = nullptr, *partV = nullptr, *Cpart = nullptr, *Csum = nullptr;
  int64_t cap_D = 0, cap_Q = 0, cap_V = 0;
  int KS = 1, JS = 1, RS = 1, ups = 0, jps = 0, rps = 0;
  float gsign = 1.f;            // sign applied to the summed dQ / dV partials (GEMM-path scoring: -1)
};

struct PosArgs {
  int M = 0, U = 0, d = 0;
  const float *ent = nullptr;
  const int64_t *ans_rows = nullptr;
  const float *Q = nullptr;
  float alpha = 0.f, gamma = 0.f, scale = 0.f;
  const float *Cq = nullptr, *QP = nullptr;
  float *loss_pos = nullptr, *Dpos = nullptr, *dQ = nullptr, *dV = nullptr;
};

// k_score.cu
// between(): called after the pair kernel is enqueued and before its epilogue (kg_api.cu runs the
// positive term there, on a side stream beside the epilogue)
void launch_pair_fwd(int kind, const ScoreArgs &a, int nout, bool train, cudaStream_t st,
                     const std::function<void()> &between = {});
void launch_pair_bwd(int kind, const ScoreArgs &a, cudaStream_t st, cudaStream_t st2);
// The dot-product scorers on the tensor-core GEMM (kg_api.cu): the pair epilogue over
// Dpart (a.KS partials) and the dQ / dV combines over partQ / partV (a.JS / a.RS partials).
void launch_pair_epi(int kind, const ScoreArgs &a, int nout, bool train, cudaStream_t st);
void launch_pos(int kind, const PosArgs &p, int nout, cudaStream_t st);
void launch_beta_entity(const float *ent, const int64_t *rows, int K, int m, float *F, float *Cv, cudaStream_t st);
void launch_beta_query(const float *Q, int NQ, int m, float *QP, float *Cq, cudaStream_t st);
void launch_loss_finalize(const float *loss_pos, const float *loss_part, int M, int njt, double scale,
                          double *loss_out, int *flags, int64_t *t_dev, float *bc, double beta1, double beta2,
                          int apply, cudaStream_t st, int check = 1);

// k_dedup.cu: sort keys (ids < 2^end_bit) with their positions; outputs
// uniq[U] (ascending), inv[L] (position -> unique index), perm[L] (sorted
// positions), seg[U+1] (segment starts into perm), *U_out.
int dedup_capacity();
void launch_dedup(const int64_t *ids64, const int32_t *ids32, int L, int end_bit, int64_t *uniq, int32_t *inv,
                  int32_t *perm, int32_t *seg, int32_t *U_out, cudaStream_t st, int32_t *sinv = nullptr,
                  int32_t *hrow = nullptr);

// k_adam.cu
void launch_init_rows(float *p, int64_t rows, int d, int64_t row0, int64_t row_step, uint64_t seed, uint64_t stream,
                      float lo, float hi, cudaStream_t st);
void launch_init_flat(float *p, int64_t n, uint64_t seed, uint64_t stream, float lo, float hi, cudaStream_t st);
void launch_sparse_adam(const int64_t *uniq, const int32_t *seg, const int32_t *perm, const int32_t *sinv,
                        const int32_t *hrow,
                        const int32_t *U_dev, int L, const float *OG, float *PS, int32_t *cnt, int d, int world,
                        float *ent, float *m, float *v, float *grad_out, const float *lr, double beta1, double beta2,
                        double eps, const float *bc, const int *flags, int apply, cudaStream_t st,
                        int64_t skip_key = -1, int early = 0);
void launch_rel_reduce(const int32_t *seg, const int32_t *perm, const int32_t *inv, const int32_t *U_dev, int Lr,
                       const float *RG, float *PS, int dr, float *RGU, cudaStream_t st);
void launch_rel_stamp(const int64_t *uniq_rel, const int32_t *U_dev, int Lmax, int32_t *rel_seg, int64_t *rel_stamp,
                      const int64_t *stamp, cudaStream_t st);
void launch_dense_adam_rel(float *p, float *m, float *v, int R, int width, int nseg, const float *RGU,
                           const int32_t *rel_seg, const int64_t *rel_stamp, const int64_t *stamp, const float *lr,
                           double beta1, double beta2, double eps, const float *bc, const int *flags,
                           cudaStream_t st, int untouched_only = 0);
void launch_dense_adam_rel_touched(float *p, float *m, float *v, int R, int width, int nseg, const float *RGU,
                                   const int64_t *runiq, const int32_t *rU, int Lr, const float *lr, double beta1,
                                   double beta2, double eps, const float *bc, const int *flags, cudaStream_t st);
void launch_dense_adam(float *p, float *m, float *v, const float *g, int64_t n, const float *lr, double beta1,
                       double beta2, double eps, const float *bc, const int *flags, cudaStream_t st);
void launch_colsum(const float *X, int rows, int cols, int ld, float *out, cudaStream_t st);
struct ColsumJob { const float *X; int rows, cols, ld; float *out; };
struct ColsumJobs {
  ColsumJob j[6];
  int n = 0;
  void add(const float *X, int rows, int cols, int ld, float *out) { j[n++] = ColsumJob{X, rows, cols, ld, out}; }
};
void launch_colsum_multi(const ColsumJobs &J, cudaStream_t st);   // out_i[c] = sum_r X_i[r][c], one launch

// k_gemm.cu: C[M][N] = beta C + op(A) op(B)^T (+ bias) (ReLU), op(A) [M][K], op(B) [N][K];
// tcgen05 kind::tf32 with a 3xTF32 split; A stored [M][lda], B stored [N][ldb] (K-major).
struct GemmArgs {
  const float *A = nullptr, *B = nullptr;
  float *C = nullptr;
  const float *bias = nullptr;
  int M = 0, N = 0, K = 0, lda = 0, ldb = 0, ldc = 0, relu = 0;
  float beta = 0.f;
  float alpha = 1.f;    // C = beta C + alpha op(A) op(B)^T (+ bias) (ReLU)
  float *P = nullptr;   // split-K partials [splits][M][N] (set by launch_gemm_tc)
  bool a_mn = false;    // A stored [K][M] (lda) instead of [M][K]
  bool b_mn = false;    // B stored [K][N] (ldb) instead of [N][K]
  int kbs = 1 << 30;    // k-blocks per split
  bool drain = false;   // fp32-accurate accumulation: TMEM chunks of kDrainKB k-blocks summed in registers
  bool lowp = false;    // bf16 score mode: operands rounded to bf16, one MMA per K-step (no 3xTF32 split)
  int force = 0;        // tile experiments (kg_test_gemm): bit 0 no split-K; bits 1-2 BN 1:64 2:128 3:160
  // pre-split B (K-major only): B_lo = rna_tf32(B - trunc_tf32(B)) in B's layout; the kernel
  // loads it with TMA instead of splitting B in shared memory (weights: kg_api.cu wsplit)
  const float *B_lo = nullptr;
  // ReLU backward folded in: C = 0 where !(mask > 0); mask has C's shape and leading dimension
  // (ldc == N required).  Applied by the split-K combine, or by a mask pass after an unsplit GEMM.
  const float *mask = nullptr;
};
struct WSplitJob { const float *w; float *lo, *t, *tlo; int R, C; };
struct WSplitJobs { WSplitJob j[12]; int n = 0; };
void launch_wsplit(const WSplitJobs &J, int part, cudaStream_t st);   // pre-split weight planes: 0 lo, 1 t + tlo
bool gemm_tc_accepts(const GemmArgs &g);   // 16-byte aligned operands, ld % 4 == 0
bool launch_gemm_tc(const GemmArgs &g, float *part, int64_t part_cap, cudaStream_t st);   // false: not launched
int launch_gemm_tc_raw(const GemmArgs &g, float *part, int64_t part_cap, cudaStream_t st);   // splits, 0: not launched
// k_dag.cu: GEMM epilogues fused with the intersection's pooling (P = raw partials [S][rows][d])
void launch_mean_red(const float *P, int S, const float *b, int n, int M, int d, float *H, float *Mn, cudaStream_t st);
void launch_q2b_off_red(const float *P, int S, const float *b, const float *stack, int n, int M, int d, float *sig,
                        int8_t *amin, float *out, cudaStream_t st);
void launch_q2b_att_red(const float *P, int S, const float *b, const float *stack, int n, int M, int d, float *a,
                        float *out, cudaStream_t st);
struct OutPtrs { float *p[4]; };
void launch_betae_proj_out_red(const float *P, int S, const float *b0, int rows, int M, int d, float *Zp1,
                               const OutPtrs &out, cudaStream_t st);
void launch_beta_att_red(const float *P, int S, const float *b, const float *stack, int n, int M, int d, float *w,
                         float *out, cudaStream_t st);
void launch_transpose(const float *in, int R, int Cc, int ld_in, float *out, int ld_out, cudaStream_t st);

// k_eval.cu (evaluation path, App. F)
struct EvalArgs {
  const float *Q = nullptr;       // query embeddings [nout][M][qstride]
  const float *ent = nullptr;     // raw entity rows [n][d]
  const int64_t *ans_off = nullptr, *ans_ids = nullptr, *negatives = nullptr;
  int M = 0, d = 0, U = 0, n_neg = 0, max_ans = 0;
  float alpha = 0.f;
  int32_t *ranks = nullptr;
  float *metrics = nullptr;       // [M][4]
};
// per-query candidates (kg_score_each): a.negatives = cand [M][n_neg], a.metrics = out [M][n_neg]
void launch_score_each(int kind, const EvalArgs &a, int nout, cudaStream_t st);
void launch_eval(int kind, const EvalArgs &a, int nout, cudaStream_t st);

// k_dist.cu (world > 1)
void launch_owner_partition(const int64_t *uniq, const int32_t *U_dev, int G, int64_t *send_ids, int32_t *send_pos,
                            int32_t *counts, cudaStream_t st, int cap = 0, int *flags = nullptr);
void launch_occ_rows(const int32_t *inv, const int32_t *send_pos, int L, int64_t *rows, cudaStream_t st);
void launch_gather_owned(const float *ent, const int64_t *ids, int n, int G, int d, float *out, cudaStream_t st);
void launch_reorder_rows(const float *Gu, const int32_t *send_pos, const int32_t *U_dev, int Lmax, int d, float *out,
                         cudaStream_t st);
void launch_local_rows(const int64_t *ids, int n, int G, int64_t *keys, cudaStream_t st, int64_t empty = -1);
// peer-memory exchange (KG_XCHG=p2p, k_dist.cu): the ranks' buffers mapped into every rank
struct PeerPtrs {
  const float *ent[kMaxWorld];            // theta_E shards
  int64_t *rids[kMaxWorld];               // owner-side receive ids   [G][cap]
  float *grecv[kMaxWorld];                // owner-side receive rows  [G][cap][d]
  unsigned long long *flags[kMaxWorld];   // barrier flags            [kMaxWorld]
};
void launch_p2p_gather(const PeerPtrs *pp, const int64_t *uniq, const int32_t *U_dev, const int32_t *send_pos, int G,
                       int Lmax, int d, float *X, cudaStream_t st);
void launch_p2p_push(const PeerPtrs *pp, const int64_t *send_ids, const float *Gsend, int G, int me, int cap, int d,
                     cudaStream_t st);
void launch_p2p_barrier(const PeerPtrs *pp, unsigned long long *mine, unsigned long long *epoch, int G, int me,
                        int *flags, cudaStream_t st);
void launch_scatter_rel(const float *RGU, const int64_t *runiq, const int32_t *rU, int Lrmax, int R, int w, int nseg,
                        float *gfull, cudaStream_t st);
void launch_loss_check(double *loss_out, int *flags, int64_t *t_dev, float *bc, double beta1, double beta2, int apply,
                       cudaStream_t st);

// k_dag.cu
void launch_proj_fwd(int kind, int N, int d, const float *in, int64_t in_ld, const int64_t *anchor_rows,
                     const float *ent, const int32_t *rel, int rel_ld, const float *relA, const float *relB,
                     float *out, cudaStream_t st);
void launch_proj_bwd(int kind, int N, int d, const float *dout, const float *in, int64_t in_ld,
                     const int64_t *anchor_rows, const float *ent, const int32_t *rel, int rel_ld, const float *relA,
                     const float *relB, const float *out, float *din, int64_t din_ld, float *drel, cudaStream_t st);
void launch_betae_proj_in(int N, int d, const float *in, const int64_t *anchor_rows, const float *ent,
                          const int32_t *rel, int rel_ld, const float *relT, float *X, cudaStream_t st);
void launch_bias_act(float *Y, const float *b, int rows, int cols, int act, cudaStream_t st);
void launch_betae_proj_out(const float *Z, const float *b0, int rows, int d, float *Zp1, float *out, cudaStream_t st);
void launch_betae_proj_dz(const float *dout, const float *Zp1, int rows, int d, float *dZ, cudaStream_t st);
void launch_relu_mask(float *dY, const float *Y, int rows, int cols, cudaStream_t st);
void launch_betae_split(const float *dX, int N, int d, const int64_t *anchor_rows, const float *ent, float *din,
                        int64_t din_ld, float *drel, cudaStream_t st);
void launch_qnorm_fwd(float *X, int M, int d, int parts, float *nrm, cudaStream_t st);
void launch_qnorm_bwd(float *G, const float *Y, int M, int d, int parts, const float *nrm, cudaStream_t st);
void launch_neg_fwd(const float *in, int64_t n, float *out, cudaStream_t st);
void launch_neg_bwd(const float *dout, const float *in, int64_t n, float *din, cudaStream_t st);
void launch_mean_stack(const float *H, int n, int rows, int cols, float *out, cudaStream_t st);
void launch_gqe_inter_dh(const float *dMn, const float *H, int n, int rows, int cols, float *dH, cudaStream_t st);
void launch_q2b_att_fwd(const float *stack, const float *Lg, int n, int M, int d, float *a, float *out,
                        cudaStream_t st);
void launch_q2b_off_fwd(const float *stack, const float *Z, int n, int M, int d, float *sig, int8_t *amin,
                        float *out, cudaStream_t st);
void launch_q2b_att_bwd(const float *stack, const float *a, const float *dout, int n, int M, int d, float *dLg,
                        float *dstack, cudaStream_t st);
void launch_q2b_off_bwd(const float *stack, const float *sig, const int8_t *amin, const float *dout, int n, int M,
                        int d, float *dZ, float *dstack, cudaStream_t st);
void launch_beta_att_fwd(const float *stack, const float *Lg, int n, int M, int d, float *w, float *out,
                         cudaStream_t st);
void launch_beta_att_bwd(const float *stack, const float *w, const float *dout, int n, int M, int d, float *dLg,
                         float *dstack, cudaStream_t st);
void launch_scale_copy(float *dst, const float *src, int64_t n, float s, cudaStream_t st);
void launch_gather_rows(float *dst, const float *src, const int64_t *rows, int n, int d, cudaStream_t st);
void launch_scatter_rows(float *dst, const float *src, const int64_t *rows, int n, int d, cudaStream_t st);
// ids = [anchors slot-major (a*M + i) | answers (n_ans) | negatives (K)], rows = id / world
void launch_ids_concat(const int64_t *anchors, int na, int M, const int64_t *answers, int n_ans, const int64_t *negs,
                       int K, int world, int64_t *ids, int64_t *rows_out, int32_t *bad, int64_t n_entities,
                       cudaStream_t st);
void launch_ids_rel(const int64_t *anchors, int na, int M, const int64_t *answers, int n_ans, const int64_t *negs,
                    int K, int world, int64_t *ids, int64_t *rows_out, int64_t n_entities, const int32_t *relations,
                    int nr, Slots4 slots, int nproj, int n_rel, int32_t *occ, int32_t *bad, cudaStream_t st);
void launch_rel_occ(const int32_t *relations, int M, int nr, Slots4 slots, int nproj, int n_rel, int32_t *occ,
                    int32_t *bad, cudaStream_t st);

}  // namespace kg
