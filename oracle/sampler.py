"""Online training-data sampler, plain Python (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

SURVEY §8(f) f3: reverse directional sampling (§3.1, App. C),
bidirectional rejection sampling with forward caching and backward verification
(§3.2), the optimal node cut of Eq. 2 by the App. C dynamic program
 and the delayed complement.  Every function
follows the paper's text in its order and notation; sets are Python sets, one entity
at a time, no blocking or reordering.

Readings (S1-S7):
  S1 query structures are trees written as S-expressions (a = anchor leaf, p = relation
     projection, i = intersection, u = union, n = negation); node ids are preorder
     indices (root = 0); anchor slots are numbered left to right, relation slots in
     post-order (= the execution order A21 that kg_step consumes).
  S2 App. C functions on a node v: u(v) = u(p(v)) + [p(v) is a projection];
     s(v) = 0 at anchors, max over children at i / u nodes, s(child) + [v is not a
     negation] at p / n nodes; o(v) = u(v) at anchors, else
     min(max_z o(z), max(u(v), s(v))).  Cut construction top-down: v joins the cut when
     max_z o(z) >= max(u(v), s(v)) (ties cut at v: the §3.2 worked example puts the ip
     cut on the node after the intersection, where both sides cost 1); a leaf reached
     by the recursion joins the cut.
  S3 Eq. 2 per path = max(#projections between the anchor and the cut node,
     #projections between the cut node and the root), log scale.
  S4 Reverse sampling: the root is a uniform entity with in-degree >= 1; a projection
     edge at an entity e takes a uniform incoming edge (h, r, e) of e (relation r, child
     grounded to h); intersection / union children are grounded to the same entity
     (App. C walkthrough); a negation child is grounded to a fresh uniform
     entity with in-degree >= 1 and the grounding is kept only if the root entity is
     an answer (SPEC S:L244 decision; the paper samples only positive paths).  A
     projection at an entity without incoming edges, or a rejected negation, restarts
     the attempt; at most MAX_ATTEMPTS attempts.
  S5 Random numbers: a counter-based generator, draw(seed, stream, idx) =
     mix64(mix64(seed ^ stream*G1) + idx*G2) (splitmix64 finaliser), index choice in
     [0, n) = floor(draw * n / 2^64).  Query draws use stream (rank << 16) | 0x51 and
     idx = ((step * 2^20 + i) * 64 + attempt) * 32 + k (k = the k-th draw of the
     attempt, DFS preorder); pool draws use stream (rank << 16) | 0x52 and
     idx = step * 2^24 + j.  The C++ sampler implements the same generator.
  S6 Shared negative pool: K entities uniform over V with
     replacement; Mask[i][j] = 1 iff pool_j is not an answer of q_i (exact).
  S7 Forward caching stores, per cut node, the entity set with a complement flag
     (delayed complement); backward verification decides v in A_q by
     recursion from the root: a projection admits v iff some incoming (h, r, v) has h
     admitted by the child, i / u / n combine the children's answers by and / or /
     not, a cut node answers by a membership probe of its cache.
"""
from __future__ import annotations

import itertools

import numpy as np

import kggen

# ----------------------------------------------------------------------------------
# S1: structures
# ----------------------------------------------------------------------------------
STRUCTURE_DSL = {
    "1p": "(p (a))",
    "2p": "(p (p (a)))",
    "3p": "(p (p (p (a))))",
    "2i": "(i (p (a)) (p (a)))",
    "3i": "(i (p (a)) (p (a)) (p (a)))",
    "ip": "(p (i (p (a)) (p (a))))",
    "pi": "(i (p (p (a))) (p (a)))",
    "2u": "(u (p (a)) (p (a)))",
    "up": "(p (u (p (a)) (p (a))))",
    "2in": "(i (p (a)) (n (p (a))))",
    "3in": "(i (p (a)) (p (a)) (n (p (a))))",
    "inp": "(p (i (p (a)) (n (p (a)))))",
    "pin": "(i (p (p (a))) (n (p (a))))",
    "pni": "(i (n (p (p (a)))) (p (a)))",
}


class Node:
    def __init__(self, op, children):
        self.op = op                  # 'a' | 'p' | 'i' | 'u' | 'n'
        self.children = children
        self.id = -1                  # preorder index
        self.slot = -1                # anchor slot ('a') or relation slot ('p')
        self.parent = None


def parse(dsl: str) -> Node:
    """S-expression -> tree with preorder ids, anchor slots (left to right), relation slots (post-order)."""
    toks = dsl.replace("(", " ( ").replace(")", " ) ").split()
    pos = 0

    def rd():
        nonlocal pos
        assert toks[pos] == "("
        op = toks[pos + 1]
        pos += 2
        ch = []
        while toks[pos] != ")":
            ch.append(rd())
        pos += 1
        return Node(op, ch)

    root = rd()
    pre = []

    def walk(v, parent):
        v.id = len(pre)
        v.parent = parent
        pre.append(v)
        for c in v.children:
            walk(c, v)

    walk(root, None)
    na = 0
    for v in pre:
        if v.op == "a":
            v.slot = na
            na += 1
    nr = 0

    def post(v):
        nonlocal nr
        for c in v.children:
            post(c)
        if v.op == "p":
            v.slot = nr
            nr += 1

    post(root)
    return root


def nodes(root: Node):
    out = []

    def walk(v):
        out.append(v)
        for c in v.children:
            walk(c)

    walk(root)
    return out


def leaf_paths(root: Node):
    """Every anchor-to-root path as a list of nodes [anchor, ..., root]."""
    paths = []
    for v in nodes(root):
        if v.op == "a":
            p, x = [], v
            while x is not None:
                p.append(x)
                x = x.parent
            paths.append(p)
    return paths


# ----------------------------------------------------------------------------------
# S2 / S3: App. C dynamic program and Eq. 2
# ----------------------------------------------------------------------------------
def annotate(root: Node):
    """u, s, o of App. C as lists indexed by node id."""
    ns = nodes(root)
    u = [0] * len(ns)
    s = [0] * len(ns)
    o = [0] * len(ns)

    def down(v):
        # u(v) = u(p(v)) + IsRel(v -> p(v))
        if v.parent is not None:
            u[v.id] = u[v.parent.id] + (1 if v.parent.op == "p" else 0)
        for c in v.children:
            down(c)

    def up(v):
        for c in v.children:
            up(c)
        if v.op == "a":
            s[v.id] = 0
            o[v.id] = u[v.id]
            return
        if v.op in ("i", "u"):
            s[v.id] = max(s[c.id] for c in v.children)
        else:   # 'p' or 'n': one child; NotNeg(ch(v) -> v)
            s[v.id] = s[v.children[0].id] + (0 if v.op == "n" else 1)
        o[v.id] = min(max(o[c.id] for c in v.children), max(u[v.id], s[v.id]))

    down(root)
    up(root)
    return u, s, o


def optimal_cut(root: Node):
    """Node cut from o(.) top-down (App. C, tie reading S2): sorted node ids."""
    u, s, o = annotate(root)
    cut = []

    def rec(v):
        if v.op == "a" or max(o[c.id] for c in v.children) >= max(u[v.id], s[v.id]):
            cut.append(v.id)
            return
        for c in v.children:
            rec(c)

    rec(root)
    return sorted(cut)


def is_cut(root: Node, cut) -> bool:
    """Def. 2: every anchor-to-root path contains exactly one node of the cut."""
    cs = set(cut)
    return all(sum(1 for x in p if x.id in cs) == 1 for p in leaf_paths(root))


def cut_cost(root: Node, cut) -> int:
    """Eq. 2 objective in log scale (S3), evaluated path by path."""
    assert is_cut(root, cut)
    cs = set(cut)
    worst = 0
    for p in leaf_paths(root):
        i = next(k for k, x in enumerate(p) if x.id in cs)
        # projections below the cut node: the parents p[1..i] that are projections
        below = sum(1 for x in p[1:i + 1] if x.op == "p")
        above = sum(1 for x in p[i + 1:] if x.op == "p")
        worst = max(worst, below, above)
    return worst


def brute_force_cut(root: Node):
    """Minimum of Eq. 2 over every node cut, by enumeration (footnote P:L242): (cut, cost)."""
    ns = nodes(root)
    assert len(ns) <= 20
    best = None
    for r in range(1, len(ns) + 1):
        for sub in itertools.combinations(range(len(ns)), r):
            if is_cut(root, sub):
                c = cut_cost(root, sub)
                if best is None or c < best[1]:
                    best = (list(sub), c)
    return best


# ----------------------------------------------------------------------------------
# The KG as plain Python adjacency (read-only)
# ----------------------------------------------------------------------------------
class OracleKG:
    def __init__(self, kg: dict):
        self.V = kg["n_entities"]
        self.R = kg["n_relations"]
        trip = sorted(set(zip(kg["h"].tolist(), kg["r"].tolist(), kg["t"].tolist())))
        self.out = {}           # (h, r) -> set of t
        self.inn = {}           # (t, r) -> set of h
        in_edges = {}           # t -> list of (r, h)
        for h, r, t in trip:
            self.out.setdefault((h, r), set()).add(t)
            self.inn.setdefault((t, r), set()).add(h)
            in_edges.setdefault(t, []).append((r, h))
        # incoming edges of t in ascending (r, h) order: the order the uniform choice indexes
        self.in_edges = {t: sorted(e) for t, e in in_edges.items()}
        self.roots = sorted(self.in_edges)     # entities with in-degree >= 1

    def project(self, S, r):
        out = set()
        for x in S:
            out |= self.out.get((x, r), set())
        return out


def exhaustive_answers(kg: OracleKG, root: Node, anchors, relations) -> set:
    """A_q by bottom-up traversal (the definition; complement taken against V)."""
    def ev(v):
        if v.op == "a":
            return {int(anchors[v.slot])}
        if v.op == "p":
            return kg.project(ev(v.children[0]), int(relations[v.slot]))
        if v.op == "i":
            sets = [ev(c) for c in v.children]
            return set.intersection(*sets)
        if v.op == "u":
            return set.union(*[ev(c) for c in v.children])
        if v.op == "n":
            return set(range(kg.V)) - ev(v.children[0])
        raise ValueError(v.op)

    return ev(root)


# ----------------------------------------------------------------------------------
# S7: bidirectional search -- forward caching and backward verification (§3.2)
# ----------------------------------------------------------------------------------
def forward_cache(kg: OracleKG, root: Node, cut, anchors, relations) -> dict:
    """node id -> (set, complemented) at every cut node, from the anchors upward.

    The complement is delayed: a negation flips the flag and the consuming
    intersection / union combines the flagged sets by set difference / union rules.
    """
    def ev(v):
        if v.op == "a":
            return {int(anchors[v.slot])}, False
        if v.op == "p":
            S, neg = ev(v.children[0])
            assert not neg, "projection right after a negation is excluded (P:L657)"
            return kg.project(S, int(relations[v.slot])), False
        if v.op == "n":
            S, neg = ev(v.children[0])
            return S, not neg
        parts = [ev(c) for c in v.children]
        pos = [S for S, neg in parts if not neg]
        negs = [S for S, neg in parts if neg]
        if v.op == "i":
            if pos:      # (∩ pos) \ (∪ negs)
                out = set.intersection(*pos)
                for S in negs:
                    out = out - S
                return out, False
            return set.union(*negs), True          # ∩ ¬S_k = ¬ ∪ S_k
        if v.op == "u":
            if negs:     # (∪ pos) ∪ (∪ ¬S_k) = ¬ (∩ S_k \ ∪ pos)
                out = set.intersection(*negs)
                for S in pos:
                    out = out - S
                return out, True
            return set.union(*pos), False
        raise ValueError(v.op)

    by_id = {v.id: v for v in nodes(root)}
    return {c: ev(by_id[c]) for c in cut}


def verify(kg: OracleKG, root: Node, cache: dict, relations, v: int) -> bool:
    """Backward verification: is v an answer of q?  (recursion of reading S7)"""
    def member(x, e):
        if x.id in cache:
            S, neg = cache[x.id]
            return (e in S) != neg
        if x.op == "p":
            r = int(relations[x.slot])
            return any(member(x.children[0], h) for h in sorted(kg.inn.get((e, r), ())))
        if x.op == "i":
            return all(member(c, e) for c in x.children)
        if x.op == "u":
            return any(member(c, e) for c in x.children)
        if x.op == "n":
            return not member(x.children[0], e)
        raise AssertionError("recursion reached a leaf outside the cut")

    return member(root, int(v))


# ----------------------------------------------------------------------------------
# S5: counter-based generator (this module's own implementation)
# ----------------------------------------------------------------------------------
M64 = (1 << 64) - 1
G1 = 0x9E3779B97F4A7C15
G2 = 0xD1B54A32D192ED03
MAX_ATTEMPTS = 64
MAX_DRAWS = 32


def mix64(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def draw(seed: int, stream: int, idx: int) -> int:
    s = mix64((seed ^ (stream * G1)) & M64)
    return mix64((s + idx * G2) & M64)


def below(x: int, n: int) -> int:
    """Index in [0, n) from a 64-bit draw: floor(x * n / 2^64)."""
    return (x * n) >> 64


def query_stream(rank: int) -> int:
    return (rank << 16) | 0x51


def pool_stream(rank: int) -> int:
    return (rank << 16) | 0x52


# ----------------------------------------------------------------------------------
# S4: reverse directional sampling (§3.1, App. C)
# ----------------------------------------------------------------------------------
class SamplerError(RuntimeError):
    pass


def instantiate(kg: OracleKG, root: Node, seed: int, step: int, i: int, rank: int = 0):
    """Ground one query: (anchors, relations, answer, attempts used)."""
    ns = nodes(root)
    na = sum(1 for v in ns if v.op == "a")
    nr = sum(1 for v in ns if v.op == "p")
    has_neg = any(v.op == "n" for v in ns)
    stream = query_stream(rank)
    for attempt in range(MAX_ATTEMPTS):
        base = ((step * (1 << 20) + i) * MAX_ATTEMPTS + attempt) * MAX_DRAWS
        k = 0

        def nxt():
            nonlocal k
            x = draw(seed, stream, base + k)
            k += 1
            return x

        anchors = [0] * na
        relations = [0] * nr

        def visit(v, e):
            if v.op == "a":
                anchors[v.slot] = e
                return True
            if v.op == "p":
                inc = kg.in_edges.get(e, [])
                if not inc:
                    return False
                r, h = inc[below(nxt(), len(inc))]
                relations[v.slot] = r
                return visit(v.children[0], h)
            if v.op in ("i", "u"):
                return all(visit(c, e) for c in v.children)
            if v.op == "n":
                e2 = kg.roots[below(nxt(), len(kg.roots))]
                return visit(v.children[0], e2)
            raise ValueError(v.op)

        ans = kg.roots[below(nxt(), len(kg.roots))]
        if not visit(root, ans):
            continue
        if has_neg and ans not in exhaustive_answers(kg, root, anchors, relations):
            continue
        return anchors, relations, ans, attempt + 1
    raise SamplerError("reverse sampling: attempt budget exhausted")


def sample_pool(V: int, K: int, seed: int, step: int, rank: int = 0):
    """Shared negative pool (S6): K uniform entities with replacement."""
    st = pool_stream(rank)
    return [below(draw(seed, st, step * (1 << 24) + j), V) for j in range(K)]


def sample_batch(kg: OracleKG, structure: str, M: int, K: int, seed: int = 0, step: int = 0,
                 rank: int = 0, exact_mask: str = "exhaustive") -> dict:
    """One training mini-batch (N, {(q_i, V_qi, a_qi)}, Mask) in the P:L389 / kg_step format.

    exact_mask: "exhaustive" builds A_q by full traversal (the definition); "bidirectional"
    uses forward caching + backward verification at the optimal cut (§3.2).  Both are exact.
    """
    root = parse(STRUCTURE_DSL[structure])
    cut = optimal_cut(root)
    pool = sample_pool(kg.V, K, seed, step, rank)
    A, Rl, ans, att = [], [], [], []
    bits = np.zeros((M, K), dtype=bool)
    for i in range(M):
        a, r, e, n_att = instantiate(kg, root, seed, step, i, rank)
        A.append(a)
        Rl.append(r)
        ans.append(e)
        att.append(n_att)
        if exact_mask == "exhaustive":
            S = exhaustive_answers(kg, root, a, r)
            bits[i] = [p not in S for p in pool]
        else:
            cache = forward_cache(kg, root, cut, a, r)
            bits[i] = [not verify(kg, root, cache, r, p) for p in pool]
    return dict(structure=structure, M=M, K=K,
                anchors=np.array(A, dtype=np.int64).reshape(M, -1),
                relations=np.array(Rl, dtype=np.int32).reshape(M, -1),
                answers=np.array(ans, dtype=np.int64),
                negatives=np.array(pool, dtype=np.int64),
                mask=kggen.pack_mask(bits), attempts=np.array(att, dtype=np.int32))
