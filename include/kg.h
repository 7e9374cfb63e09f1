/*
 * kg.h -- C-ABI of libkg.so: one training step of batched multi-hop
 * query-embedding models on a B200 (sm_100a), after SMORE (arXiv 2110.14890).
 *
 * Citations: P:Lnnn = /root/reference/PAPER.md line nnn.  The readings A1-A24
 * referred to below are listed in DESIGN.md §3.
 *
 * Conventions for every call
 *   - Every call returns kg_status (KG_OK = 0).  No C++ exception crosses the
 *     ABI.  On error, kg_last_error(handle) returns a NUL-terminated message
 *     owned by the handle (valid until the next call on that handle).
 *   - Memory ownership: the CALLER owns all table memory (theta_E shard, its
 *     Adam moments, theta_D and its moments), allocated on the handle's device
 *     and bound with kg_bind; the library never frees it.  The library owns the
 *     handle, its device workspace, pinned staging buffers, cuBLAS handle and
 *     NCCL communicator, all released by kg_destroy.
 *   - Host input arrays need only stay valid until the call returns (they are
 *     staged before return).  Device input arrays (kg_batch.on_device = 1)
 *     must stay valid until the step has executed on the bound stream.
 *   - All device work is enqueued on the stream given to kg_bind, in order.
 *   - Transactional: on a validation error nothing is enqueued; when the loss
 *     of a step is non-finite, the update kernels see a device flag and leave
 *     every table untouched (KG_ENONFINITE is reported by the call that reads
 *     the loss: kg_step with info != NULL, or kg_sync).
 *   - A CUDA / NCCL failure moves the handle to a sticky error state: later
 *     calls return KG_ESTATE.
 *   - world > 1: kg_step, kg_score, kg_eval and kg_gather_rows are collective: every
 *     rank calls them together (kg_step with the same structure, M and K, P:L303,
 *     L397-398; the others with their own queries / ids, sizes may differ per rank).
 */
#ifndef KG_H_
#define KG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KG_OK = 0,
  KG_EINVAL = 1,        /* null pointer, out-of-range id / size / config value */
  KG_EUNSUPPORTED = 2,  /* e.g. a multi-hop structure for a single-hop model */
  KG_ENOMEM = 3,        /* device / pinned allocation failed */
  KG_ECUDA = 4,         /* CUDA runtime / cuBLAS error (handle -> sticky state) */
  KG_ENCCL = 5,         /* NCCL error (handle -> sticky state) */
  KG_ENONFINITE = 6,    /* the step's loss was not finite; the step was not applied */
  KG_ESTATE = 7         /* handle unusable (earlier CUDA/NCCL error, or not bound) */
} kg_status;

/* Models of Table 1 and Table 2. */
typedef enum {
  KG_GQE = 0, KG_Q2B = 1, KG_BETAE = 2,                  /* multi-hop, all 9 structures */
  KG_TRANSE = 3, KG_ROTATE = 4, KG_DISTMULT = 5, KG_COMPLEX = 6,  /* single-hop: 1p only */
  /* multi-hop extensions (App. B; reading A27), all 9 structures: projection and
   * distance of the base model, GQE's DeepSet intersection; DistMult-m / ComplEx-m normalise
   * the query (whole / Re and Im parts) after every projection and intersection */
  KG_ROTATE_M = 7, KG_DISTMULT_M = 8, KG_COMPLEX_M = 9
} kg_model_kind;

/* Query structures, DNF for unions. */
typedef enum {
  KG_1P = 0, KG_2P = 1, KG_3P = 2, KG_2I = 3, KG_3I = 4,
  KG_IP = 5, KG_PI = 6, KG_2U = 7, KG_UP = 8,
  /* negation structures (Table 10), BetaE only: N(q) = 1/q (Table 1) */
  KG_2IN = 9, KG_3IN = 10, KG_INP = 11, KG_PIN = 12, KG_PNI = 13
} kg_structure;

/* Number of anchor / relation slots of a structure (execution order, A21):
 * anchors 1p,2p,3p:1  2i:2  3i:3  ip,pi,2u,up:2   2in:2 3in:3 inp,pin,pni:2
 * relations 1p:1 2p:2 3p:3 2i:2 3i:3 ip:3 pi:3 2u:2 up:3   2in:2 3in:3 inp,pin,pni:3
 * 2in = I(P(a0,r0), N(P(a1,r1)))         3in = I(P(a0,r0), P(a1,r1), N(P(a2,r2)))
 * inp = P(I(P(a0,r0), N(P(a1,r1))), r2)   pin = I(P(P(a0,r0),r1), N(P(a1,r2)))
 * pni = I(N(P(P(a0,r0),r1)), P(a1,r2))                                               */

typedef struct {
  int32_t kind;          /* kg_model_kind */
  int32_t dim;           /* d: fp32 values per entity row (A1); must be a multiple of 8, <= 2048 */
  int64_t n_entities;    /* |V|: 1 <= n_entities < 2^31 */
  int32_t n_relations;   /* |R| >= 1 */
  int32_t hidden;        /* BetaE projection MLP width H (A9), multiple of 8; ignored otherwise */
  float gamma;           /* margin of Eq. 1 */
  float box_alpha;       /* Q2B in-box weight alpha (Table 1, A7) */
  double beta1, beta2, eps; /* Adam (A15); double so that 1 - beta2 keeps its digits */
  int32_t max_M;         /* workspace sizing: queries per step */
  int32_t max_K;         /* workspace sizing: shared negatives per step */
  int32_t max_cand;      /* workspace sizing: candidates per kg_score call */
  int32_t rank, world;   /* this process's rank in [0, world); theta_E is row-sharded, owner(id) = id % world */
  const void *nccl_id;   /* world > 1: pointer to a 128-byte ncclUniqueId shared by all ranks; NULL if world == 1 */
  int32_t score_precision; /* KG_SCORE_FP32 (0, default) or KG_SCORE_BF16 (1): the dot-product scorers'
                            * (DistMult / ComplEx and their -m variants; SURVEY §8(a) a8 "bf16 opt-in") three
                            * scoring contractions of kg_step with operands rounded to bf16 and fp32
                            * accumulation (tolerance 2e-2, §8(c)); kg_score / kg_eval stay fp32.
                            * EUNSUPPORTED for the other kinds, EINVAL for other values. */
} kg_config;
enum { KG_SCORE_FP32 = 0, KG_SCORE_BF16 = 1 };

/* Caller-owned device tables (fp32, row-major).
 * ent, ent_m, ent_v : [kg_shard_rows() x dim]  theta_E row shard + Adam moments
 *                     local row of global id g is g / world (owner g % world).
 * dense, dense_m, dense_v : [kg_dense_size()]  theta_D = relation tables + operator weights
 *                     (P:L300), layout of DESIGN.md §5 (= kggen.dense_layout).             */
typedef struct {
  float *ent, *ent_m, *ent_v;
  float *dense, *dense_m, *dense_v;
} kg_tables;

/* One mini-batch (N, {(q_i, V_qi, A_qi)}_{i=1..M}, Mask) of P:L389, one structure.
 * anchors   int64 [M][n_anchors(structure)]  anchor entity ids (leaves of the plan)
 * relations int32 [M][n_relations(structure)] relation ids in execution order (A21)
 * answers   int64 [M]                         the single positive a_q per query
 * negatives int64 [K]                         the shared pool N, duplicates allowed (A20)
 * mask      uint32 [M][ceil(K/32)]            bit (j%32) of word j/32 set <=> negatives[j] is a
 *                                             negative of query i (Mask_ij of P:L389); the padding
 *                                             bits j >= K of the last word are ignored
 * on_device 0: host pointers; 1: device pointers on the handle's device.
 * For kg_score only structure, M, anchors and relations are read.                               */
typedef struct {
  int32_t structure;
  int32_t M;
  int32_t K;
  const int64_t *anchors;
  const int32_t *relations;
  const int64_t *answers;
  const int64_t *negatives;
  const uint32_t *mask;
  int32_t on_device;
} kg_batch;

typedef struct {
  double loss;           /* global Eq. 1 loss of the step (mean over queries and ranks, A12, A18) */
  int32_t n_touched;     /* distinct entity ids touched by this rank's batch (A16) */
  int64_t step;          /* Adam step counter t after the step */
  int32_t kernels;       /* kernels of this library enqueued by the step */
  int32_t gemms;         /* tcgen05 tensor-core GEMM launches enqueued by the step (MLP layers, dot scores) */
  float stage_ms[10];    /* device time per stage when stage timing is on (kg_set_apply bit 2), else 0:
                            0 ingest + dedup, 1 DAG forward, 2 scoring forward + Eq. 1, 3 scoring backward,
                            4 DAG backward, 5 sparse update (segment reduce + sparse Adam), 6 what the dense
                            update adds after the sparse one, 7 whole step; world = 1 only (else 0):
                            8 the late dense path (relation reduce + Adam of the used relation rows and of
                            the operator weights, on a second stream concurrently with stage 5), 9 the early
                            dense path (Adam of the relation rows the step does not use, g = 0, on a third
                            stream from the end of stage 2, concurrently with stages 3-5).  With world > 1
                            stage 5 also holds the relation reduce and the row-gradient exchange, and 6
                            what the all-reduce + dense Adam (on a second stream and communicator,
                            overlapped with stage 5) add after it. */
} kg_step_info;

typedef struct kg_handle kg_handle;   /* opaque; one per (process, device) */

/* Create a handle on the current CUDA device: validates cfg, allocates the
 * workspace for (max_M, max_K, max_cand), creates cuBLAS (and NCCL when
 * world > 1).  EINVAL on a bad config (dim % 8 != 0, odd sizes, ...). */
kg_status kg_create(const kg_config *cfg, kg_handle **out);

/* Rows of the local theta_E shard: ceil(n_entities / world). */
int64_t kg_shard_rows(const kg_handle *h);

/* Floats in theta_D for this model (relation tables + operator weights). */
int64_t kg_dense_size(const kg_handle *h);
/* Device bytes of the library's own workspace (staged batch, dedup outputs, occurrence
 * gradients, DAG activations, scoring partials, exchange buffers), sized once at kg_create
 * from max_M / max_K / max_cand and the model; allocated and freed by the library (the
 * caller owns the tables of kg_bind, the library only this scratch).  -1 for a NULL handle. */
int64_t kg_workspace_size(const kg_handle *h);

/* Record the caller's table pointers and the CUDA stream (cudaStream_t, may be NULL).
 * Host tier (the paper keeps theta_E in CPU memory): each of
 * ent / ent_m / ent_v may be pinned host memory (cudaHostAlloc / cudaHostRegister) instead of
 * device memory; the kernels then gather and update its rows zero-copy over the host link.
 * theta_D must be device memory.  EINVAL for pageable or misaligned pointers. */
kg_status kg_bind(kg_handle *h, const kg_tables *tables, void *cuda_stream);

/* Parameter init (A23): counter-based U(lo, hi) of (seed, stream, index) into ent and dense,
 * zero Adam moments, t = 0.  Identical to kggen.counter_uniform. */
kg_status kg_init_params(kg_handle *h, uint64_t seed);

/* One training step (stages 2-4, synchronous; A18):
 * dedup -> fused gather + query DAG forward (Tables 1-2) -> DNF min (A11)
 * -> positive + shared-negative scoring with Eq. 1 -> backward
 * -> deterministic segment-reduce of row gradients + sparse Adam on touched rows
 * -> [world > 1: NCCL all-reduce of dL/dtheta_D] -> dense Adam on theta_D (A17).
 * lr > 0.  info == NULL: fully asynchronous (nothing waits on the GPU; read the loss
 * later with kg_sync).  info != NULL: waits for the step and fills info.
 * Errors: EINVAL (bad pointer/size/id/relation/structure), EUNSUPPORTED (multi-hop
 * structure for a single-hop kind), ENONFINITE (info != NULL and loss not finite). */
kg_status kg_step(kg_handle *h, const kg_batch *batch, float lr, kg_step_info *info);

/* Wait for the last enqueued step and report it (ENONFINITE if its loss was not finite). */
kg_status kg_sync(kg_handle *h, kg_step_info *info);
/* The OLDEST unread step result (waits for that step only) -- two steps' results are kept,
 * so a host loop can issue step s + 1 (info = NULL) before reading step s and the device
 * never idles on the host round trip; a third unread step drops the oldest.  KG_ESTATE if
 * nothing is unread.  kg_sync instead waits for everything and returns the latest step. */
kg_status kg_result(kg_handle *h, kg_step_info *info);

/* Dist(f(q_i), f(v_c)) for every query of `queries` (forward DAG only) and every
 * shared candidate cand[c] (n_cand <= max_cand): out_dist host [M][n_cand], lower = closer,
 * unions = DNF min (A11).  world > 1: collective (each rank its own queries and candidates;
 * the anchor and candidate rows are fetched from their owners first); the
 * distances are bit-identical to those of one rank holding the whole table. */
kg_status kg_score(kg_handle *h, const kg_batch *queries, const int64_t *cand, int32_t n_cand,
                   float *out_dist);

/* Per-query candidates (SURVEY §8(b) sketch, `shared = 0`): Dist(f(q_i), f(v)) of every
 * query of `queries` (forward DAG only) to ITS OWN candidates: cand host [M][n_cand] (row i =
 * query i's candidates, any ids in [0, n_entities), duplicates allowed), out_dist host
 * [M][n_cand], lower = closer, unions = DNF min (A11).  n_cand >= 1 and n_cand * M <= 2^31.
 * One CTA per query (k_eval.cu score_each_kernel: a row gather of n_cand rows per query plus
 * the distance arithmetic -- nothing is shared across queries, so no pair tiling); the
 * distances equal kg_score's up to fp32 summation order.  world > 1: collective as kg_score
 * (candidate rows fetched from their owners).  Errors: EINVAL (pointer / size / id),
 * EUNSUPPORTED (structure not valid for the kind).  Synchronises the stream. */
kg_status kg_score_each(kg_handle *h, const kg_batch *queries, const int64_t *cand, int32_t n_cand,
                        float *out_dist);

/* Evaluation path (App. F, reading A26): filtered rank of every missing
 * answer of every query and the per-query metrics.  queries: structure, M (<= max_M),
 * anchors, relations (host or device per on_device).  ans_off host [M+1] (ans_off[0] = 0,
 * every query >= 1 answer), ans_ids host [ans_off[M]]: the missing answers
 * A_q^{G_test} \ A_q^{G_valid}; negatives host [M][n_neg]: per-query negatives the caller
 * sampled from V \ A_q^{G_test} (already filtered; "1000 negative answers ... for each
 * query").  Rank(v) = 1 + #{j : D(q, v_j) <= D(q, v)} (ties count against v), D the model
 * distance with the DNF min over disjuncts.  Outputs (host): ranks [ans_off[M]] and
 * metrics [M][4] = MRR, Hit@1, Hit@3, Hit@10 of each query (mean over its answers).
 * Needs (max answers per query + n_neg) <= 51200.  world > 1: collective as kg_score (answer
 * and negative rows fetched from their owners).  Errors: EINVAL (pointer / size / id),
 * EUNSUPPORTED (structure not valid for the kind).  Synchronises the stream. */
kg_status kg_eval(kg_handle *h, const kg_batch *queries, const int64_t *ans_off, const int64_t *ans_ids,
                  int32_t n_neg, const int64_t *negatives, int32_t *ranks, float *metrics);

/* Test / checkpoint hooks.  which: 0 parameter, 1 Adam m, 2 Adam v.
 * Rows are global ids owned by this rank (world == 1: any id); out/in host [n][dim]. */
kg_status kg_read_rows(kg_handle *h, int32_t which, const int64_t *ids, int32_t n, float *out);
/* Collective read ("with G>1 it is collective, gathering rows from their owners"):
 * every rank calls it with its own n >= 0 global ids (any owner) and receives their rows of table
 * `which` in out host [n][dim].  Exact per-owner counts are all-gathered, ids and rows exchanged
 * over NCCL (not the captured step: a few host round trips).  world == 1: kg_read_rows. */
kg_status kg_gather_rows(kg_handle *h, int32_t which, const int64_t *ids, int32_t n, float *out);
kg_status kg_write_rows(kg_handle *h, int32_t which, const int64_t *ids, int32_t n, const float *in);
kg_status kg_read_dense(kg_handle *h, int32_t which, float *out);          /* out [kg_dense_size()] */
kg_status kg_write_dense(kg_handle *h, int32_t which, const float *in);

/* Gradients of the last step, before the optimizer (parity stage (i) of SURVEY §8(c)):
 * uniq host int64 [cap] = touched ids ascending (A16), grad_rows host [cap][dim] = merged
 * dL/dtheta_E rows, grad_dense host [kg_dense_size()] = dL/dtheta_D (relation rows
 * not used by the step are 0).  *n_uniq receives U; EINVAL if U > cap.
 * Also: if d_neg != NULL, host [M][K] distances D_ij (DNF min, unmasked) and d_pos host [M]. */
kg_status kg_last_grads(kg_handle *h, int64_t *uniq, float *grad_rows, float *grad_dense,
                        int32_t cap, int32_t *n_uniq, float *d_pos, float *d_neg);

/* Test hook.  flags bit 0 (default 1): apply the optimizers; 0 computes loss and
 * gradients but skips both optimizers and t.  bit 1 (default 0): keep the merged
 * theta_E gradient rows of each step for kg_last_grads (one extra U x dim write).
 * bit 2 (default 0): record CUDA events between the stages of kg_step (kg_step_info.stage_ms). */
kg_status kg_set_apply(kg_handle *h, int32_t flags);

/* Checkpoint / resume: the tables are the caller's (kg_bind), so a checkpoint is
 * the caller's copy of them plus the Adam step counter t (A15), read and restored here.
 * kg_set_step waits for pending work; t >= 0. */
kg_status kg_get_step(kg_handle *h, int64_t *t);
kg_status kg_set_step(kg_handle *h, int64_t t);

const char *kg_last_error(const kg_handle *h);

/* Test hook: the tensor-core GEMM of the query-DAG contractions on device pointers,
 * C[M][N] (ldc) = beta*C + op(A) op(B)^T (+ bias[n]) (ReLU if relu & 1), op(A) = [M][K], op(B) = [N][K];
 * relu & 2 selects the drained (fp32-accurate) accumulation used for BetaE;
 * ta: A stored [K][lda] (else [M][lda]); tb: B stored [K][ldb] (else [N][ldb]); both layouts are
 * read in place by TMA.  tcgen05 kind::tf32 with a 3xTF32 split (fp32-level accuracy).  Needs
 * K >= 1, 16-byte aligned A / B and lda % 4 == ldb % 4 == 0 (else EINVAL).  Synchronises the stream.
 * Tool bits: (relu >> 2) & 63 forces a tile / split-K variant, relu >> 8 = back-to-back repetitions. */
kg_status kg_test_gemm(int32_t ta, int32_t tb, int32_t M, int32_t N, int32_t K, const float *A, int32_t lda,
                       const float *B, int32_t ldb, float *C, int32_t ldc, const float *bias, int32_t relu, float beta,
                       void *stream);

/* world > 1: rank 0 creates the 128-byte NCCL unique id (written to out) and shares it with
 * the other ranks (e.g. torch.distributed broadcast) before every rank calls kg_create. */
kg_status kg_nccl_unique_id(void *out);

/* Release everything the library owns; never frees caller memory.  NULL is a no-op. */
void kg_destroy(kg_handle *h);

#ifdef __cplusplus
}
#endif
#endif /* KG_H_ */
