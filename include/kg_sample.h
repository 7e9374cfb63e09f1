/* kg_sample.h -- C-ABI of libkgsample.so: the online training-data sampler that feeds
 * kg_step (§3, App. C).
 *
 * Host-side native code (C++17, std::thread): the paper's sampler runs on CPU threads
 * and overlaps with the GPU step; here a pool of worker threads fills a
 * bounded ring of ready batches in exactly the kg_step input format (kg.h kg_batch,
 * P:L389), while the GPU trains on the previous one.
 *
 * What one batch is (§4.3, "share the negative answers among"):
 *   - one query structure per step (scheduled structure sampling);
 *   - M queries, each grounded by REVERSE DIRECTIONAL SAMPLING (§3.1 P:L207-209,
 *     App. C): the root (answer) is a uniform entity with an incoming edge,
 *     every projection edge takes a uniform incoming edge (h, r, e) of the entity e it
 *     leaves, intersection / union children share the entity, a negated branch is
 *     grounded from a fresh uniform entity and the query is kept only if the root is
 *     an answer (reading S4);
 *   - a shared pool of K negatives, uniform over V with replacement;
 *   - Mask[i][j] = 1 iff pool_j is NOT an answer of query i, decided exactly by
 *     BIDIRECTIONAL REJECTION SAMPLING (§3.2): forward caching from the
 *     anchors up to the optimal node cut (Eq. 2, found by the App. C
 *     dynamic program P:L667-686), backward verification from the candidate down to
 *     the cut; complements are delayed into set differences.
 * Random numbers are counter-based (reading S5): the batch of (seed, rank, step) is a
 * pure function of those numbers and the graph, independent of the thread count.
 *
 * Query structures and slot order are those of kg.h (kg_structure 0..13): anchors
 * left to right, relations in execution (post-)order (reading A21).
 *
 * Ownership: the caller owns every array it passes; the library copies the triples
 * into its own CSR indices at kgs_graph_create and never keeps a caller pointer.
 * Errors: every call returns kgs_status; kgs_last_error() gives the message of the
 * last failure on the calling thread.  No C++ exception crosses the ABI.
 */
#ifndef KG_SAMPLE_H
#define KG_SAMPLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KGS_OK = 0,
  KGS_EINVAL = 1,      /* null pointer, size out of range, id >= n_entities, relation >= n_relations */
  KGS_ENOMEM = 2,
  KGS_EEXHAUSTED = 3,  /* reverse sampling found no valid grounding within 64 attempts (reading S4) */
  KGS_ESTATE = 4       /* pipeline stopped after a worker failure */
} kgs_status;

typedef struct kgs_graph kgs_graph;
typedef struct kgs_pipeline kgs_pipeline;

/* Build the graph indices (in-edges sorted by (t, r, h), out-edges by (h, r, t), duplicate
 * triples dropped) from n_edges triples (h[i], r[i], t[i]).  Entity ids < 2^31.
 * n_threads >= 1 threads sort the adjacency lists.  *out is owned by the caller
 * (kgs_graph_destroy). */
kgs_status kgs_graph_create(int64_t n_entities, int32_t n_relations, int64_t n_edges, const int64_t *h,
                            const int32_t *r, const int64_t *t, int32_t n_threads, kgs_graph **out);
void kgs_graph_destroy(kgs_graph *g);
/* Number of distinct triples, and of entities with in-degree >= 1 (the root candidates). */
int64_t kgs_graph_edges(const kgs_graph *g);
int64_t kgs_graph_roots(const kgs_graph *g);

/* App. C plan of a structure: node count (preorder ids, root = 0), and per node the
 * DP values u, s, o and cut[v] = 1 iff v is in the optimal node cut
 * (top-down construction P:L684-686, ties cut at v: reading S2).  Arrays hold >= 16
 * entries; any of them may be NULL. */
kgs_status kgs_plan(int32_t structure, int32_t *n_nodes, int32_t *u, int32_t *s, int32_t *o, int32_t *cut);

/* One batch.  Outputs (caller-owned host arrays): anchors int64 [M][n_anchors],
 * relations int32 [M][n_rel], answers int64 [M], negatives int64 [K],
 * mask uint32 [M][ceil(K/32)] (bit j%32 of word j/32, LSB first), attempts int32 [M]
 * (may be NULL).  1 <= M <= 2^20, 0 <= K < 2^24.  Queries are split over n_threads. */
kgs_status kgs_sample(const kgs_graph *g, int32_t structure, int32_t M, int32_t K, uint64_t seed, int64_t step,
                      int32_t rank, int32_t n_threads, int64_t *anchors, int32_t *relations, int64_t *answers,
                      int64_t *negatives, uint32_t *mask, int32_t *attempts);

/* Exact membership of candidates in the answer sets of M given queries (bidirectional
 * search at the optimal cut): is_answer[i][j] = 1 iff cand is an answer of query i,
 * with cand = cand[j] (shared = 1, cand [n_cand]) or cand[i][j] (shared = 0,
 * cand [M][n_cand]).  Used to filter evaluation negatives (App. F). */
kgs_status kgs_verify(const kgs_graph *g, int32_t structure, int32_t M, const int64_t *anchors,
                      const int32_t *relations, int32_t n_cand, const int64_t *cand, int32_t shared,
                      uint8_t *is_answer, int32_t n_threads);

/* Answer sets of M given queries by full forward traversal (App. A set semantics; the
 * evaluation set of App. E, needs A_q on G_train / G_valid / G_test):
 * offsets [M + 1] (int64) and, when ids is not NULL, ids [offsets[M]] (ascending per query).
 * Call once with ids = NULL to size the output, then with ids of capacity cap >= offsets[M].
 * KGS_EINVAL if a query's answer set is a complement (a negation at the root: none of the 14
 * structures) or cap is too small. */
kgs_status kgs_answers(const kgs_graph *g, int32_t structure, int32_t M, const int64_t *anchors,
                       const int32_t *relations, int64_t *offsets, int64_t *ids, int64_t cap, int32_t n_threads);

/* Asynchronous pipeline: n_workers threads produce the batches of steps first_step,
 * first_step + 1, ... (structure of step s = structures[s % n_structures]) into a ring
 * of `depth` >= n_workers slots; the graph must outlive the pipeline. */
kgs_status kgs_pipeline_create(const kgs_graph *g, const int32_t *structures, int32_t n_structures, int32_t M,
                               int32_t K, uint64_t seed, int32_t rank, int64_t first_step, int32_t depth,
                               int32_t n_workers, kgs_pipeline **out);
/* Blocks until the next step's batch is ready and copies it into the caller's arrays
 * (sized for the largest structure: anchors [M][3], relations [M][3]); *structure and
 * *step receive its structure id and step number, *wait_ms the time spent blocked. */
kgs_status kgs_pipeline_next(kgs_pipeline *p, int32_t *structure, int64_t *step, int64_t *anchors,
                             int32_t *relations, int64_t *answers, int64_t *negatives, uint32_t *mask,
                             double *wait_ms);
void kgs_pipeline_destroy(kgs_pipeline *p);

const char *kgs_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* KG_SAMPLE_H */
