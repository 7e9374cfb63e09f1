// sampler.cpp -- libkgsample.so: the online training-data sampler (include/kg_sample.h).
//
// SURVEY §8(f) f3.  PAPER.md §3.1 P:L207-209 + App. C P:L643 (reverse directional
// sampling), §3.2 P:L221-233 (bidirectional rejection sampling: forward caching to the
// node cut, backward verification from the candidate), Eq. 2 P:L237-240 and the App. C
// dynamic program P:L667-686 (optimal node cut), P:L655-656 (delayed complement).
// Readings S1-S7 of DESIGN.md §3.  Host C++17 with std::thread: the paper's sampler is
// CPU work overlapped with the GPU step; a bounded ring of ready batches in
// the kg_step input format is filled by worker threads.
#include "kg_sample.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <tuple>
#include <climits>
#include <vector>

namespace {

thread_local std::string g_err;
kgs_status fail(kgs_status s, const std::string &m) {
  g_err = m;
  return s;
}

// ------------------------------------------------------------------ S1: structures
// kg.h kg_structure order; a = anchor, p = projection, i = intersection, u = union, n = negation
const char *kDSL[14] = {
    "(p (a))",                          // 1p
    "(p (p (a)))",                      // 2p
    "(p (p (p (a))))",                  // 3p
    "(i (p (a)) (p (a)))",              // 2i
    "(i (p (a)) (p (a)) (p (a)))",      // 3i
    "(p (i (p (a)) (p (a))))",          // ip
    "(i (p (p (a))) (p (a)))",          // pi
    "(u (p (a)) (p (a)))",              // 2u
    "(p (u (p (a)) (p (a))))",          // up
    "(i (p (a)) (n (p (a))))",          // 2in
    "(i (p (a)) (p (a)) (n (p (a))))",  // 3in
    "(p (i (p (a)) (n (p (a)))))",      // inp
    "(i (p (p (a))) (n (p (a))))",      // pin
    "(i (n (p (p (a)))) (p (a)))",      // pni
};
constexpr int kMaxNodes = 16;

struct PNode {
  char op;
  int nch, ch[3], slot, parent;
};
struct Plan {
  int n = 0, na = 0, nr = 0;
  bool has_neg = false;
  PNode node[kMaxNodes];
  int u[kMaxNodes], s[kMaxNodes], o[kMaxNodes];
  bool cut[kMaxNodes];
};

// Recursive descent; preorder ids, anchor slots left to right, relation slots post-order.
int parse_node(Plan &P, const char *&c, int parent) {
  while (*c == ' ') ++c;
  ++c;  // '('
  const int id = P.n++;
  PNode &v = P.node[id];
  v.op = *c++;
  v.nch = 0;
  v.parent = parent;
  v.slot = -1;
  if (v.op == 'a') v.slot = P.na++;
  if (v.op == 'n') P.has_neg = true;
  for (;;) {
    while (*c == ' ') ++c;
    if (*c == ')') { ++c; break; }
    const int ch = parse_node(P, c, id);
    P.node[id].ch[P.node[id].nch++] = ch;
  }
  if (P.node[id].op == 'p') P.node[id].slot = P.nr++;
  return id;
}

void cut_rec(Plan &P, int v) {
  const PNode &x = P.node[v];
  int mo = -1;
  for (int k = 0; k < x.nch; ++k) mo = std::max(mo, P.o[x.ch[k]]);
  if (x.op == 'a' || mo >= std::max(P.u[v], P.s[v])) { P.cut[v] = true; return; }
  for (int k = 0; k < x.nch; ++k) cut_rec(P, x.ch[k]);
}

Plan make_plan(const char *dsl) {
  Plan P;
  const char *c = dsl;
  parse_node(P, c, -1);
  // App. C: u top-down (parents precede children in preorder), s and o bottom-up
  for (int v = 0; v < P.n; ++v)
    P.u[v] = P.node[v].parent < 0 ? 0 : P.u[P.node[v].parent] + (P.node[P.node[v].parent].op == 'p' ? 1 : 0);
  for (int v = P.n - 1; v >= 0; --v) {
    const PNode &x = P.node[v];
    if (x.op == 'a') { P.s[v] = 0; P.o[v] = P.u[v]; continue; }
    int ms = 0, mo = 0;
    for (int k = 0; k < x.nch; ++k) { ms = std::max(ms, P.s[x.ch[k]]); mo = std::max(mo, P.o[x.ch[k]]); }
    P.s[v] = (x.op == 'i' || x.op == 'u') ? ms : ms + (x.op == 'n' ? 0 : 1);
    P.o[v] = std::min(mo, std::max(P.u[v], P.s[v]));
  }
  for (int v = 0; v < P.n; ++v) P.cut[v] = false;
  cut_rec(P, 0);
  return P;
}

const Plan &plan_of(int structure) {
  static const std::vector<Plan> plans = [] {
    std::vector<Plan> v;
    for (int s = 0; s < 14; ++s) v.push_back(make_plan(kDSL[s]));
    return v;
  }();
  return plans[structure];
}

// ------------------------------------------------------------------ S5: counter-based generator
constexpr uint64_t kG1 = 0x9E3779B97F4A7C15ull, kG2 = 0xD1B54A32D192ED03ull;
constexpr int kMaxAttempts = 64, kMaxDraws = 32;

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t stream_key(uint64_t seed, uint64_t stream) { return mix64(seed ^ (stream * kG1)); }
inline uint64_t draw(uint64_t key, uint64_t idx) { return mix64(key + idx * kG2); }
inline uint64_t below(uint64_t x, uint64_t n) { return (uint64_t)(((unsigned __int128)x * n) >> 64); }

// ------------------------------------------------------------------ graph
struct Graph {
  int64_t V = 0;
  int32_t R = 0;
  std::vector<int64_t> in_off, out_off;   // [V + 1]
  std::vector<int32_t> in_rel, in_src;    // in-edges of t sorted by (r, h)
  std::vector<int32_t> out_rel, out_dst;  // out-edges of h sorted by (r, t)
  std::vector<int32_t> roots;             // entities with in-degree >= 1, ascending
};

template <class F>
void parallel_for(int64_t n, int threads, F f) {
  threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n));
  if (threads == 1) { f(0, n); return; }
  std::vector<std::thread> th;
  for (int k = 0; k < threads; ++k) th.emplace_back(f, n * k / threads, n * (k + 1) / threads);
  for (auto &t : th) t.join();
}

// CSR of (key = rel << 32 | other) bucketed by `node`, lists sorted and deduplicated.
void build_csr(int64_t V, int64_t E, const int64_t *node, const int32_t *rel, const int64_t *other, int threads,
               std::vector<int64_t> &off, std::vector<int32_t> &orel, std::vector<int32_t> &oth) {
  std::vector<int64_t> cnt(V + 1, 0);
  for (int64_t e = 0; e < E; ++e) ++cnt[node[e] + 1];
  for (int64_t v = 0; v < V; ++v) cnt[v + 1] += cnt[v];
  std::vector<uint64_t> key(E);
  {
    std::vector<int64_t> cur(cnt.begin(), cnt.end() - 1);
    for (int64_t e = 0; e < E; ++e) key[cur[node[e]]++] = ((uint64_t)(uint32_t)rel[e] << 32) | (uint32_t)other[e];
  }
  std::vector<int64_t> len(V, 0);
  parallel_for(V, threads, [&](int64_t a, int64_t b) {
    for (int64_t v = a; v < b; ++v) {
      uint64_t *p = key.data() + cnt[v], *q = key.data() + cnt[v + 1];
      std::sort(p, q);
      len[v] = std::unique(p, q) - p;
    }
  });
  off.assign(V + 1, 0);
  for (int64_t v = 0; v < V; ++v) off[v + 1] = off[v] + len[v];
  orel.resize(off[V]);
  oth.resize(off[V]);
  parallel_for(V, threads, [&](int64_t a, int64_t b) {
    for (int64_t v = a; v < b; ++v)
      for (int64_t k = 0; k < len[v]; ++k) {
        const uint64_t x = key[cnt[v] + k];
        orel[off[v] + k] = (int32_t)(x >> 32);
        oth[off[v] + k] = (int32_t)(uint32_t)x;
      }
  });
}

// [lo, hi) of the edges of `v` with relation r (lists sorted by relation)
inline void rel_range(const std::vector<int64_t> &off, const std::vector<int32_t> &rel, int64_t v, int32_t r,
                      int64_t &lo, int64_t &hi) {
  const int32_t *b = rel.data() + off[v], *e = rel.data() + off[v + 1];
  const int32_t *l = std::lower_bound(b, e, r);
  const int32_t *h = std::upper_bound(l, e, r);
  lo = l - rel.data();
  hi = h - rel.data();
}

// ------------------------------------------------------------------ S7: bidirectional search
using Set = std::vector<int32_t>;
struct CSet {
  Set s;
  bool neg = false;
};

struct Query {
  const Graph &g;
  const Plan &P;
  const int64_t *anchors;
  const int32_t *rels;
  CSet cache[kMaxNodes];

  Query(const Graph &g_, const Plan &P_, const int64_t *a, const int32_t *r) : g(g_), P(P_), anchors(a), rels(r) {}

  void project(const Set &S, int32_t r, Set &out) const {
    out.clear();
    for (int32_t x : S) {
      int64_t lo, hi;
      rel_range(g.out_off, g.out_rel, x, r, lo, hi);
      out.insert(out.end(), g.out_dst.begin() + lo, g.out_dst.begin() + hi);
    }
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
  }

  // forward evaluation of node v with the complement delayed
  CSet eval(int v) const {
    const PNode &x = P.node[v];
    CSet R;
    if (x.op == 'a') { R.s.push_back((int32_t)anchors[x.slot]); return R; }
    if (x.op == 'p') {
      CSet c = eval(x.ch[0]);
      project(c.s, rels[x.slot], R.s);   // c.neg is false: no projection right after a negation
      return R;
    }
    if (x.op == 'n') { R = eval(x.ch[0]); R.neg = !R.neg; return R; }
    std::vector<CSet> parts;
    for (int k = 0; k < x.nch; ++k) parts.push_back(eval(x.ch[k]));
    std::vector<const Set *> pos, negs;
    for (auto &c : parts) (c.neg ? negs : pos).push_back(&c.s);
    Set tmp;
    auto inter = [&](const std::vector<const Set *> &v) {
      Set acc = *v[0];
      for (size_t k = 1; k < v.size(); ++k) {
        tmp.clear();
        std::set_intersection(acc.begin(), acc.end(), v[k]->begin(), v[k]->end(), std::back_inserter(tmp));
        acc.swap(tmp);
      }
      return acc;
    };
    auto uni = [&](const std::vector<const Set *> &v) {
      Set acc = *v[0];
      for (size_t k = 1; k < v.size(); ++k) {
        tmp.clear();
        std::set_union(acc.begin(), acc.end(), v[k]->begin(), v[k]->end(), std::back_inserter(tmp));
        acc.swap(tmp);
      }
      return acc;
    };
    auto minus = [&](Set acc, const std::vector<const Set *> &v) {
      for (auto *s : v) {
        tmp.clear();
        std::set_difference(acc.begin(), acc.end(), s->begin(), s->end(), std::back_inserter(tmp));
        acc.swap(tmp);
      }
      return acc;
    };
    if (x.op == 'i') {
      if (!pos.empty()) { R.s = minus(inter(pos), negs); return R; }   // (∩ pos) \ (∪ negs)
      R.s = uni(negs); R.neg = true; return R;                          // ∩ ¬S = ¬ ∪ S
    }
    // 'u'
    if (!negs.empty()) { R.s = minus(inter(negs), pos); R.neg = true; return R; }  // ¬(∩ S \ ∪ pos)
    R.s = uni(pos);
    return R;
  }

  void forward_cache() {
    for (int v = 0; v < P.n; ++v)
      if (P.cut[v]) cache[v] = eval(v);
  }

  // backward verification: is e admitted by node v?
  bool member(int v, int32_t e) const {
    if (P.cut[v]) return std::binary_search(cache[v].s.begin(), cache[v].s.end(), e) != cache[v].neg;
    const PNode &x = P.node[v];
    switch (x.op) {
      case 'p': {
        int64_t lo, hi;
        rel_range(g.in_off, g.in_rel, e, rels[x.slot], lo, hi);
        for (int64_t k = lo; k < hi; ++k)
          if (member(x.ch[0], g.in_src[k])) return true;
        return false;
      }
      case 'i':
        for (int k = 0; k < x.nch; ++k)
          if (!member(x.ch[k], e)) return false;
        return true;
      case 'u':
        for (int k = 0; k < x.nch; ++k)
          if (member(x.ch[k], e)) return true;
        return false;
      case 'n':
        return !member(x.ch[0], e);
    }
    return false;
  }
};

// ------------------------------------------------------------------ S4: reverse directional sampling
struct Grounder {
  const Graph &g;
  const Plan &P;
  uint64_t key, base;
  int k;
  int64_t *anchors;
  int32_t *rels;

  uint64_t next() { return draw(key, base + (uint64_t)(k++)); }
  bool visit(int v, int32_t e) {
    const PNode &x = P.node[v];
    switch (x.op) {
      case 'a': anchors[x.slot] = e; return true;
      case 'p': {
        const int64_t deg = g.in_off[e + 1] - g.in_off[e];
        if (deg == 0) return false;
        const int64_t j = g.in_off[e] + (int64_t)below(next(), (uint64_t)deg);
        rels[x.slot] = g.in_rel[j];
        return visit(x.ch[0], g.in_src[j]);
      }
      case 'i':
      case 'u':
        for (int c = 0; c < x.nch; ++c)
          if (!visit(x.ch[c], e)) return false;
        return true;
      case 'n': {
        const int32_t e2 = g.roots[below(next(), g.roots.size())];
        return visit(x.ch[0], e2);
      }
    }
    return false;
  }
};

inline uint64_t query_stream(int rank) { return ((uint64_t)rank << 16) | 0x51; }
inline uint64_t pool_stream(int rank) { return ((uint64_t)rank << 16) | 0x52; }

// Ground query i of (seed, rank, step); on success the forward cache of q is built.
bool instantiate(const Graph &g, const Plan &P, uint64_t seed, int64_t step, int i, int rank, int64_t *anchors,
                 int32_t *rels, int64_t *answer, int32_t *attempts, Query &q) {
  const uint64_t key = stream_key(seed, query_stream(rank));
  for (int a = 0; a < kMaxAttempts; ++a) {
    Grounder G{g, P, key, (((uint64_t)step * (1ull << 20) + (uint64_t)i) * kMaxAttempts + (uint64_t)a) * kMaxDraws,
               0, anchors, rels};
    const int32_t ans = g.roots[below(G.next(), g.roots.size())];
    if (!G.visit(0, ans)) continue;
    q.forward_cache();
    if (P.has_neg && !q.member(0, ans)) continue;
    *answer = ans;
    if (attempts) *attempts = a + 1;
    return true;
  }
  return false;
}

// Backward verification batched over the shared pool (§3.2 with §4.3's shared negatives,
// P:L388-391): every query of a batch verifies the same K candidates, so the backward
// step starts once per batch from the pool -- its entities sorted with their positions,
// and its incoming edges grouped by relation -- and each query walks only the pool
// edges of its own relations instead of probing K candidates one by one.  The result
// is the same exact membership as Query::member (tests compare both with the oracle).
struct PoolIndex {
  std::vector<std::pair<int32_t, int32_t>> ent;   // (entity, position) sorted
  std::vector<int32_t> e_rel, e_src, e_pos;       // pool in-edges sorted by (r, h, position)
  int K = 0;

  void build(const Graph &g, const int64_t *pool, int K_) {
    K = K_;
    ent.resize(K);
    for (int j = 0; j < K; ++j) ent[j] = {(int32_t)pool[j], j};
    std::sort(ent.begin(), ent.end());
    std::vector<std::tuple<int32_t, int32_t, int32_t>> e;
    for (int j = 0; j < K; ++j)
      for (int64_t k = g.in_off[pool[j]]; k < g.in_off[pool[j] + 1]; ++k) e.emplace_back(g.in_rel[k], g.in_src[k], j);
    std::sort(e.begin(), e.end());
    e_rel.resize(e.size()); e_src.resize(e.size()); e_pos.resize(e.size());
    for (size_t k = 0; k < e.size(); ++k) std::tie(e_rel[k], e_src[k], e_pos[k]) = e[k];
  }
};

struct PosSet {
  std::vector<int32_t> pos;   // sorted pool positions
  bool neg = false;           // complemented within [0, K)
};

// Pool positions admitted by node v of query q (with the complement delayed).
PosSet admitted(const Query &q, const PoolIndex &X, int v) {
  const Plan &P = q.P;
  const PNode &x = P.node[v];
  PosSet R;
  if (P.cut[v]) {
    const Set &S = q.cache[v].s;
    R.neg = q.cache[v].neg;
    if ((int64_t)S.size() * 8 < X.K) {      // few cached entities: look each up in the sorted pool
      for (int32_t e : S) {
        auto lo = std::lower_bound(X.ent.begin(), X.ent.end(), std::make_pair(e, INT32_MIN));
        for (; lo != X.ent.end() && lo->first == e; ++lo) R.pos.push_back(lo->second);
      }
      std::sort(R.pos.begin(), R.pos.end());
    } else {                                 // else probe every pool entity in the cache
      for (int j = 0; j < X.K; ++j)
        if (std::binary_search(S.begin(), S.end(), X.ent[j].first)) R.pos.push_back(X.ent[j].second);
      std::sort(R.pos.begin(), R.pos.end());
    }
    return R;
  }
  if (x.op == 'p') {                         // pool edges (h, r, pool_j) with h admitted by the child
    const int32_t r = q.rels[x.slot];
    auto lo = std::lower_bound(X.e_rel.begin(), X.e_rel.end(), r) - X.e_rel.begin();
    auto hi = std::upper_bound(X.e_rel.begin(), X.e_rel.end(), r) - X.e_rel.begin();
    for (auto k = lo; k < hi; ++k)
      if (q.member(x.ch[0], X.e_src[k])) R.pos.push_back(X.e_pos[k]);
    std::sort(R.pos.begin(), R.pos.end());
    R.pos.erase(std::unique(R.pos.begin(), R.pos.end()), R.pos.end());
    return R;
  }
  if (x.op == 'n') { R = admitted(q, X, x.ch[0]); R.neg = !R.neg; return R; }
  std::vector<PosSet> parts;
  for (int k = 0; k < x.nch; ++k) parts.push_back(admitted(q, X, x.ch[k]));
  std::vector<const std::vector<int32_t> *> pos, negs;
  for (auto &c : parts) (c.neg ? negs : pos).push_back(&c.pos);
  std::vector<int32_t> tmp;
  auto fold = [&](const std::vector<const std::vector<int32_t> *> &v, int how) {
    std::vector<int32_t> acc = *v[0];
    for (size_t k = 1; k < v.size(); ++k) {
      tmp.clear();
      if (how == 0) std::set_intersection(acc.begin(), acc.end(), v[k]->begin(), v[k]->end(), std::back_inserter(tmp));
      else std::set_union(acc.begin(), acc.end(), v[k]->begin(), v[k]->end(), std::back_inserter(tmp));
      acc.swap(tmp);
    }
    return acc;
  };
  auto minus = [&](std::vector<int32_t> acc, const std::vector<const std::vector<int32_t> *> &v) {
    for (auto *s : v) {
      tmp.clear();
      std::set_difference(acc.begin(), acc.end(), s->begin(), s->end(), std::back_inserter(tmp));
      acc.swap(tmp);
    }
    return acc;
  };
  if (x.op == 'i') {
    if (!pos.empty()) { R.pos = minus(fold(pos, 0), negs); return R; }
    R.pos = fold(negs, 1); R.neg = true; return R;
  }
  if (!negs.empty()) { R.pos = minus(fold(negs, 0), pos); R.neg = true; return R; }
  R.pos = fold(pos, 1);
  return R;
}

// Queries [i0, i1) of one batch (the pool and its index already built).
bool sample_range(const Graph &g, const Plan &P, int i0, int i1, int K, uint64_t seed, int64_t step, int rank,
                  const PoolIndex &X, int64_t *anchors, int32_t *relations, int64_t *answers, uint32_t *mask,
                  int32_t *attempts) {
  const int W = (K + 31) / 32;
  for (int i = i0; i < i1; ++i) {
    int64_t *a = anchors + (int64_t)i * P.na;
    int32_t *r = relations + (int64_t)i * P.nr;
    Query q(g, P, a, r);
    if (!instantiate(g, P, seed, step, i, rank, a, r, answers + i, attempts ? attempts + i : nullptr, q))
      return false;
    uint32_t *mrow = mask + (int64_t)i * W;
    if (K == 0) continue;
    // Mask bit j = 1 iff pool_j is not an answer
    const PosSet A = admitted(q, X, 0);
    const uint32_t fill = A.neg ? 0u : ~0u;
    for (int w = 0; w < W; ++w) mrow[w] = fill;
    if (K % 32) mrow[W - 1] &= (1u << (K % 32)) - 1u;
    for (int32_t j : A.pos) mrow[j >> 5] ^= 1u << (j & 31);
  }
  return true;
}

void draw_pool(const Graph &g, int K, uint64_t seed, int64_t step, int rank, int64_t *pool) {
  const uint64_t key = stream_key(seed, pool_stream(rank));
  for (int j = 0; j < K; ++j) pool[j] = (int64_t)below(draw(key, (uint64_t)step * (1ull << 24) + (uint64_t)j), g.V);
}

kgs_status check_sample_args(const Graph *g, int structure, int M, int K, int64_t step) {
  if (!g) return fail(KGS_EINVAL, "null graph");
  if (structure < 0 || structure >= 14) return fail(KGS_EINVAL, "structure out of range [0, 14)");
  if (M < 1 || M > (1 << 20)) return fail(KGS_EINVAL, "M out of range [1, 2^20]");
  if (K < 0 || K >= (1 << 24)) return fail(KGS_EINVAL, "K out of range [0, 2^24)");
  if (step < 0) return fail(KGS_EINVAL, "negative step");
  if (g->roots.empty()) return fail(KGS_EINVAL, "graph has no edges");
  return KGS_OK;
}

}  // namespace

struct kgs_graph : Graph {};

// ------------------------------------------------------------------ pipeline
namespace {
struct Slot {
  std::vector<int64_t> anchors, answers, negatives;
  std::vector<int32_t> rels;
  std::vector<uint32_t> mask;
  int32_t structure = 0;
  int64_t step = -1;
  bool ready = false;
  kgs_status st = KGS_OK;
};
}  // namespace

struct kgs_pipeline {
  const Graph *g;
  std::vector<int32_t> structures;
  int M, K, rank, depth;
  uint64_t seed;
  int64_t consume = 0, claim = 0;   // next step to hand out / to produce
  std::vector<Slot> slots;
  std::mutex mu;
  std::condition_variable cv;
  bool stop = false, failed = false;
  std::vector<std::thread> workers;

  void work() {
    for (;;) {
      int64_t s;
      Slot *sl;
      {
        std::unique_lock<std::mutex> lk(mu);
        s = claim++;
        cv.wait(lk, [&] { return stop || s < consume + depth; });
        if (stop) return;
        sl = &slots[s % depth];
      }
      const int st = structures[s % structures.size()];
      const Plan &P = plan_of(st);
      draw_pool(*g, K, seed, s, rank, sl->negatives.data());
      PoolIndex X;
      X.build(*g, sl->negatives.data(), K);
      const bool ok = sample_range(*g, P, 0, M, K, seed, s, rank, X, sl->anchors.data(),
                                   sl->rels.data(), sl->answers.data(), sl->mask.data(), nullptr);
      {
        std::lock_guard<std::mutex> lk(mu);
        sl->structure = st;
        sl->step = s;
        sl->st = ok ? KGS_OK : KGS_EEXHAUSTED;
        sl->ready = true;
      }
      cv.notify_all();
    }
  }
};

extern "C" {

kgs_status kgs_graph_create(int64_t n_entities, int32_t n_relations, int64_t n_edges, const int64_t *h,
                            const int32_t *r, const int64_t *t, int32_t n_threads, kgs_graph **out) {
  if (!out || (n_edges > 0 && (!h || !r || !t))) return fail(KGS_EINVAL, "null pointer");
  *out = nullptr;
  if (n_entities < 1 || n_entities >= (1ll << 31) || n_relations < 1 || n_edges < 0)
    return fail(KGS_EINVAL, "sizes out of range");
  for (int64_t e = 0; e < n_edges; ++e)
    if (h[e] < 0 || h[e] >= n_entities || t[e] < 0 || t[e] >= n_entities || r[e] < 0 || r[e] >= n_relations)
      return fail(KGS_EINVAL, "triple " + std::to_string(e) + " out of range");
  kgs_graph *g = new (std::nothrow) kgs_graph();
  if (!g) return fail(KGS_ENOMEM, "graph allocation");
  try {
    g->V = n_entities;
    g->R = n_relations;
    const int th = std::max(1, n_threads);
    build_csr(n_entities, n_edges, t, r, h, th, g->in_off, g->in_rel, g->in_src);
    build_csr(n_entities, n_edges, h, r, t, th, g->out_off, g->out_rel, g->out_dst);
    for (int64_t v = 0; v < n_entities; ++v)
      if (g->in_off[v + 1] > g->in_off[v]) g->roots.push_back((int32_t)v);
  } catch (const std::bad_alloc &) {
    delete g;
    return fail(KGS_ENOMEM, "graph indices");
  }
  *out = g;
  return KGS_OK;
}

void kgs_graph_destroy(kgs_graph *g) { delete g; }
int64_t kgs_graph_edges(const kgs_graph *g) { return g ? (int64_t)g->in_src.size() : 0; }
int64_t kgs_graph_roots(const kgs_graph *g) { return g ? (int64_t)g->roots.size() : 0; }

kgs_status kgs_plan(int32_t structure, int32_t *n_nodes, int32_t *u, int32_t *s, int32_t *o, int32_t *cut) {
  if (structure < 0 || structure >= 14) return fail(KGS_EINVAL, "structure out of range [0, 14)");
  const Plan &P = plan_of(structure);
  if (n_nodes) *n_nodes = P.n;
  for (int v = 0; v < P.n; ++v) {
    if (u) u[v] = P.u[v];
    if (s) s[v] = P.s[v];
    if (o) o[v] = P.o[v];
    if (cut) cut[v] = P.cut[v] ? 1 : 0;
  }
  return KGS_OK;
}

kgs_status kgs_sample(const kgs_graph *g, int32_t structure, int32_t M, int32_t K, uint64_t seed, int64_t step,
                      int32_t rank, int32_t n_threads, int64_t *anchors, int32_t *relations, int64_t *answers,
                      int64_t *negatives, uint32_t *mask, int32_t *attempts) {
  kgs_status st = check_sample_args(g, structure, M, K, step);
  if (st != KGS_OK) return st;
  if (!anchors || !relations || !answers || (K > 0 && (!negatives || !mask))) return fail(KGS_EINVAL, "null output");
  const Plan &P = plan_of(structure);
  try {
    draw_pool(*g, K, seed, step, rank, negatives);
    PoolIndex X;
    X.build(*g, negatives, K);
    std::atomic<bool> ok{true};
    parallel_for(M, std::max(1, n_threads), [&](int64_t a, int64_t b) {
      if (!sample_range(*g, P, (int)a, (int)b, K, seed, step, rank, X, anchors, relations, answers, mask,
                        attempts))
        ok = false;
    });
    if (!ok) return fail(KGS_EEXHAUSTED, "reverse sampling: attempt budget exhausted");
  } catch (const std::bad_alloc &) {
    return fail(KGS_ENOMEM, "sampler working sets");
  }
  return KGS_OK;
}

kgs_status kgs_verify(const kgs_graph *g, int32_t structure, int32_t M, const int64_t *anchors,
                      const int32_t *relations, int32_t n_cand, const int64_t *cand, int32_t shared,
                      uint8_t *is_answer, int32_t n_threads) {
  if (!g || !anchors || !relations || (n_cand > 0 && (!cand || !is_answer))) return fail(KGS_EINVAL, "null pointer");
  if (structure < 0 || structure >= 14) return fail(KGS_EINVAL, "structure out of range [0, 14)");
  if (M < 1 || n_cand < 0) return fail(KGS_EINVAL, "sizes out of range");
  const Plan &P = plan_of(structure);
  for (int64_t k = 0; k < (int64_t)M * P.na; ++k)
    if (anchors[k] < 0 || anchors[k] >= g->V) return fail(KGS_EINVAL, "anchor id out of range");
  for (int64_t k = 0; k < (int64_t)M * P.nr; ++k)
    if (relations[k] < 0 || relations[k] >= g->R) return fail(KGS_EINVAL, "relation out of range");
  const int64_t nc = shared ? n_cand : (int64_t)M * n_cand;
  for (int64_t k = 0; k < nc; ++k)
    if (cand[k] < 0 || cand[k] >= g->V) return fail(KGS_EINVAL, "candidate id out of range");
  try {
    parallel_for(M, std::max(1, n_threads), [&](int64_t a, int64_t b) {
      for (int64_t i = a; i < b; ++i) {
        Query q(*g, P, anchors + i * P.na, relations + i * P.nr);
        q.forward_cache();
        const int64_t *c = shared ? cand : cand + i * n_cand;
        for (int j = 0; j < n_cand; ++j) is_answer[i * n_cand + j] = q.member(0, (int32_t)c[j]) ? 1 : 0;
      }
    });
  } catch (const std::bad_alloc &) {
    return fail(KGS_ENOMEM, "sampler working sets");
  }
  return KGS_OK;
}

kgs_status kgs_answers(const kgs_graph *g, int32_t structure, int32_t M, const int64_t *anchors,
                       const int32_t *relations, int64_t *offsets, int64_t *ids, int64_t cap, int32_t n_threads) {
  if (!g || !anchors || !relations || !offsets) return fail(KGS_EINVAL, "null pointer");
  if (structure < 0 || structure >= 14) return fail(KGS_EINVAL, "structure out of range [0, 14)");
  if (M < 1) return fail(KGS_EINVAL, "M < 1");
  const Plan &P = plan_of(structure);
  for (int64_t k = 0; k < (int64_t)M * P.na; ++k)
    if (anchors[k] < 0 || anchors[k] >= g->V) return fail(KGS_EINVAL, "anchor id out of range");
  for (int64_t k = 0; k < (int64_t)M * P.nr; ++k)
    if (relations[k] < 0 || relations[k] >= g->R) return fail(KGS_EINVAL, "relation out of range");
  std::vector<Set> ans(M);
  std::atomic<bool> comp{false};
  try {
    parallel_for(M, std::max(1, n_threads), [&](int64_t a, int64_t b) {
      for (int64_t i = a; i < b; ++i) {
        Query q(*g, P, anchors + i * P.na, relations + i * P.nr);
        CSet r = q.eval(0);
        if (r.neg) comp = true;
        ans[i].swap(r.s);
      }
    });
  } catch (const std::bad_alloc &) {
    return fail(KGS_ENOMEM, "answer sets");
  }
  if (comp) return fail(KGS_EINVAL, "an answer set is a complement (negation at the root)");
  offsets[0] = 0;
  for (int i = 0; i < M; ++i) offsets[i + 1] = offsets[i] + (int64_t)ans[i].size();
  if (!ids) return KGS_OK;
  if (cap < offsets[M]) return fail(KGS_EINVAL, "ids capacity below offsets[M]");
  for (int i = 0; i < M; ++i)
    for (size_t k = 0; k < ans[i].size(); ++k) ids[offsets[i] + (int64_t)k] = ans[i][k];
  return KGS_OK;
}

kgs_status kgs_pipeline_create(const kgs_graph *g, const int32_t *structures, int32_t n_structures, int32_t M,
                               int32_t K, uint64_t seed, int32_t rank, int64_t first_step, int32_t depth,
                               int32_t n_workers, kgs_pipeline **out) {
  if (!out || !structures || n_structures < 1) return fail(KGS_EINVAL, "null pointer / no structures");
  *out = nullptr;
  for (int k = 0; k < n_structures; ++k) {
    kgs_status st = check_sample_args(g, structures[k], M, K, first_step);
    if (st != KGS_OK) return st;
  }
  if (n_workers < 1 || depth < n_workers) return fail(KGS_EINVAL, "need n_workers >= 1 and depth >= n_workers");
  kgs_pipeline *p = new (std::nothrow) kgs_pipeline();
  if (!p) return fail(KGS_ENOMEM, "pipeline");
  try {
    p->g = g;
    p->structures.assign(structures, structures + n_structures);
    p->M = M; p->K = K; p->rank = rank; p->depth = depth; p->seed = seed;
    p->consume = p->claim = first_step;
    p->slots.resize(depth);
    for (auto &s : p->slots) {
      s.anchors.resize((size_t)M * 3);
      s.rels.resize((size_t)M * 3);
      s.answers.resize(M);
      s.negatives.resize(std::max(K, 1));
      s.mask.resize((size_t)M * std::max(1, (K + 31) / 32));
    }
    for (int w = 0; w < n_workers; ++w) p->workers.emplace_back([p] { p->work(); });
  } catch (...) {
    kgs_pipeline_destroy(p);
    return fail(KGS_ENOMEM, "pipeline buffers / threads");
  }
  *out = p;
  return KGS_OK;
}

kgs_status kgs_pipeline_next(kgs_pipeline *p, int32_t *structure, int64_t *step, int64_t *anchors,
                             int32_t *relations, int64_t *answers, int64_t *negatives, uint32_t *mask,
                             double *wait_ms) {
  if (!p || !anchors || !relations || !answers || (p->K > 0 && (!negatives || !mask)))
    return fail(KGS_EINVAL, "null pointer");
  const auto t0 = std::chrono::steady_clock::now();
  std::unique_lock<std::mutex> lk(p->mu);
  if (p->failed) return fail(KGS_ESTATE, "pipeline stopped after a worker failure");
  Slot &sl = p->slots[p->consume % p->depth];
  p->cv.wait(lk, [&] { return sl.ready && sl.step == p->consume; });
  if (wait_ms) *wait_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (sl.st != KGS_OK) {
    p->failed = true;
    return fail(sl.st, "reverse sampling: attempt budget exhausted");
  }
  const Plan &P = plan_of(sl.structure);
  if (structure) *structure = sl.structure;
  if (step) *step = sl.step;
  std::memcpy(anchors, sl.anchors.data(), sizeof(int64_t) * p->M * P.na);
  std::memcpy(relations, sl.rels.data(), sizeof(int32_t) * p->M * P.nr);
  std::memcpy(answers, sl.answers.data(), sizeof(int64_t) * p->M);
  if (p->K > 0) {
    std::memcpy(negatives, sl.negatives.data(), sizeof(int64_t) * p->K);
    std::memcpy(mask, sl.mask.data(), sizeof(uint32_t) * p->M * ((p->K + 31) / 32));
  }
  sl.ready = false;
  ++p->consume;
  lk.unlock();
  p->cv.notify_all();
  return KGS_OK;
}

void kgs_pipeline_destroy(kgs_pipeline *p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(p->mu);
    p->stop = true;
  }
  p->cv.notify_all();
  for (auto &t : p->workers) t.join();
  delete p;
}

const char *kgs_last_error(void) { return g_err.c_str(); }

}  // extern "C"
