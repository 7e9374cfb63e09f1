"""Pins of the online-sampler oracle (oracle/sampler.py) against what the paper and
mathematics fix: the §3.2 worked example, hand-evaluated App. C recursions, brute-force
enumeration of node cuts (Eq. 2), exhaustive traversal on tiny KGs, the published
splitmix64 outputs, and the distribution reverse sampling defines (chi-square)."""
import json
import os
import random

import numpy as np
import pytest

import kggen
from oracle import sampler as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sampler_pins.json")))


def kg_from_triples(triples, V, R):
    h, r, t = (np.array(x, dtype=np.int64) for x in zip(*triples))
    return S.OracleKG(dict(h=h, r=r.astype(np.int32), t=t, n_entities=V, n_relations=R))


def ip_example():
    g = GOLD["ip_worked_example"]
    E = {n: i for i, n in enumerate(g["entities"])}
    Rl = {n: i for i, n in enumerate(g["relations"])}
    kg = kg_from_triples([(E[a], Rl[b], E[c]) for a, b, c in g["triples"]], len(E), len(Rl))
    return g, E, Rl, kg


# ------------------------------------------------------------------ DP / node cut
def test_ip_worked_example_cut_cache_answers():
    g, E, Rl, kg = ip_example()
    root = S.parse(S.STRUCTURE_DSL["ip"])
    cut = S.optimal_cut(root)
    assert cut == g["cut"]
    anchors = [E[a] for a in g["anchors"]]
    rels = [Rl[r] for r in g["query_relations"]]
    cache = S.forward_cache(kg, root, cut, anchors, rels)
    assert cache == {1: ({E[x] for x in g["cache_at_cut"]}, False)}
    assert S.exhaustive_answers(kg, root, anchors, rels) == {E[x] for x in g["answers"]}
    for x in g["answers"]:
        assert S.verify(kg, root, cache, rels, E[x])
    for x in g["non_answers_checked"]:
        assert not S.verify(kg, root, cache, rels, E[x])


@pytest.mark.parametrize("name,structure", [("dp_2p", "2p"), ("dp_1p", "1p")])
def test_dp_hand_values(name, structure):
    g = GOLD[name]
    root = S.parse(S.STRUCTURE_DSL[structure])
    u, s, o = S.annotate(root)
    assert (u, s, o) == (g["u"], g["s"], g["o"])
    cut = S.optimal_cut(root)
    assert cut == g["cut"] and S.cut_cost(root, cut) == g["cost"]


def test_3p_cost_is_two():
    root = S.parse(S.STRUCTURE_DSL["3p"])
    assert S.cut_cost(root, S.optimal_cut(root)) == GOLD["dp_3p_cost"]["cost"]
    assert S.brute_force_cut(root)[1] == GOLD["dp_3p_cost"]["cost"]


def random_tree(rng, budget):
    """Random computation plan (ops a / p / i / u / n, no projection right above a negation)."""
    def gen(b, parent_op):
        if b <= 1:
            return "(a)", 1
        ops = ["a", "p", "p", "i", "u", "n"]
        if parent_op == "n":
            ops = ["p", "i", "u"]
        op = rng.choice(ops)
        if op == "a":
            return "(a)", 1
        if op in ("p", "n"):
            if op == "n" and parent_op == "p":
                op = "p"
            s, used = gen(b - 1, op)
            return f"({op} {s})", used + 1
        k = rng.choice([2, 2, 3])
        parts, used = [], 1
        for _ in range(k):
            s, u_ = gen(max(1, (b - used) // k), op)
            parts.append(s)
            used += u_
        return f"({op} {' '.join(parts)})", used
    while True:
        s, n = gen(budget, None)
        if not s.startswith("(a") and n <= 12:
            return s


def test_dp_matches_brute_force_catalog_and_random_trees():
    for name, dsl in S.STRUCTURE_DSL.items():
        root = S.parse(dsl)
        cut = S.optimal_cut(root)
        assert S.is_cut(root, cut), name
        assert S.cut_cost(root, cut) == S.brute_force_cut(root)[1], name
        assert S.cut_cost(root, cut) == S.annotate(root)[2][0], name      # o(root) = the optimum
    rng = random.Random(7)
    for _ in range(300):
        dsl = random_tree(rng, rng.randint(3, 12))
        root = S.parse(dsl)
        cut = S.optimal_cut(root)
        assert S.is_cut(root, cut), dsl
        assert S.cut_cost(root, cut) == S.brute_force_cut(root)[1], dsl


def test_cut_validity_checker_rejects_non_cuts():
    root = S.parse(S.STRUCTURE_DSL["pi"])      # ids: 0 i, 1 p, 2 p, 3 a, 4 p, 5 a
    assert S.is_cut(root, [0]) and S.is_cut(root, [3, 5]) and S.is_cut(root, [1, 4])
    assert not S.is_cut(root, [1])             # misses the a1 path
    assert not S.is_cut(root, [0, 1])          # two nodes on one path


# ------------------------------------------------------------------ traversal semantics
def test_exhaustive_small_cases():
    g = GOLD["exhaustive_small"]
    kg = kg_from_triples(g["triples"], g["n_entities"], 2)
    for c in g["cases"]:
        root = S.parse(S.STRUCTURE_DSL[c["structure"]])
        assert S.exhaustive_answers(kg, root, c["anchors"], c["relations"]) == set(c["answers"]), c


def small_kg(seed, V=48, R=3, E=260):
    return S.OracleKG(kggen.make_kg(V, R, E, seed=seed, a=0.5))


@pytest.mark.parametrize("structure", kggen.ALL_STRUCTURES)
def test_bidirectional_equals_exhaustive(structure):
    """Backward verification at the optimal cut decides v in A_q exactly."""
    root = S.parse(S.STRUCTURE_DSL[structure])
    cut = S.optimal_cut(root)
    na = sum(1 for v in S.nodes(root) if v.op == "a")
    nr = sum(1 for v in S.nodes(root) if v.op == "p")
    rng = np.random.default_rng(1)
    for seed in range(3):
        kg = small_kg(seed)
        for q in range(12):
            if q % 2 == 0:
                a, r, _, _ = S.instantiate(kg, root, seed, 0, q)
            else:      # arbitrary groundings, including empty answer sets
                a = rng.integers(0, kg.V, na).tolist()
                r = rng.integers(0, kg.R, nr).tolist()
            A = S.exhaustive_answers(kg, root, a, r)
            cache = S.forward_cache(kg, root, cut, a, r)
            for v in range(kg.V):
                assert S.verify(kg, root, cache, r, v) == (v in A), (structure, a, r, v)
            # every cut node's cache is the exhaustive value of its sub-plan
            for c in cut:
                sub = next(x for x in S.nodes(root) if x.id == c)
                Sset, neg = cache[c]
                val = S.exhaustive_answers(kg, sub, a, r)
                assert (set(range(kg.V)) - Sset if neg else Sset) == val


# ------------------------------------------------------------------ generator
def test_splitmix64_published_outputs():
    g = GOLD["splitmix64"]
    for x, y in zip(g["inputs"], g["outputs"]):
        assert S.mix64(int(x, 16)) == int(y, 16)


def test_below_is_uniform():
    n, N = 7, 70000
    c = np.bincount([S.below(S.draw(3, 9, i), n) for i in range(N)], minlength=n)
    chi2 = float(((c - N / n) ** 2 / (N / n)).sum())
    assert chi2 < 22.5          # chi-square(6) 0.999 quantile
    assert S.below(S.M64, 10) == 9 and S.below(0, 10) == 0


# ------------------------------------------------------------------ reverse sampling
def test_single_edge_kg_1p():
    kg = kg_from_triples([(0, 0, 1)], 2, 1)
    root = S.parse(S.STRUCTURE_DSL["1p"])
    for i in range(5):
        a, r, e, att = S.instantiate(kg, root, 0, 0, i)
        assert (a, r, e, att) == ([0], [0], 1, 1)


def test_1p_reverse_sampling_distribution():
    """P(edge (h, r, t)) = 1 / (#roots * indeg(t)): uniform root, then uniform in-edge (§3.1)."""
    trip = [(0, 0, 1), (2, 0, 1), (3, 1, 1), (0, 1, 2), (1, 0, 3), (2, 1, 3)]
    kg = kg_from_triples(trip, 4, 2)
    root = S.parse(S.STRUCTURE_DSL["1p"])
    N = 6000
    cnt = {}
    for i in range(N):
        a, r, e, _ = S.instantiate(kg, root, 5, 0, i)
        cnt[(a[0], r[0], e)] = cnt.get((a[0], r[0], e), 0) + 1
    indeg = {1: 3, 2: 1, 3: 2}
    chi2 = 0.0
    for (h, r, t) in trip:
        exp = N / (3 * indeg[t])
        chi2 += (cnt.get((h, r, t), 0) - exp) ** 2 / exp
    assert set(cnt) <= set(trip)
    assert chi2 < 20.5          # chi-square(5) 0.999 quantile


@pytest.mark.parametrize("structure", kggen.ALL_STRUCTURES)
def test_positive_is_an_answer(structure):
    """Reverse sampling always yields a valid query whose root is an answer (§3.1)."""
    root = S.parse(S.STRUCTURE_DSL[structure])
    neg = next((x for x in S.nodes(root) if x.op == "n"), None)
    for seed in range(2):
        kg = small_kg(10 + seed)
        for i in range(25):
            a, r, e, att = S.instantiate(kg, root, seed, 3, i)
            assert e in S.exhaustive_answers(kg, root, a, r)
            assert 1 <= att <= S.MAX_ATTEMPTS
            if neg is not None:       # the answer is outside the negated branch's set
                assert e not in S.exhaustive_answers(kg, neg.children[0], a, r)


def test_sample_batch_masks_agree_and_are_exact():
    kg = small_kg(3)
    for structure in ("2p", "ip", "up", "pni"):
        b1 = S.sample_batch(kg, structure, 10, 40, seed=2, step=1)
        b2 = S.sample_batch(kg, structure, 10, 40, seed=2, step=1, exact_mask="bidirectional")
        for k in ("anchors", "relations", "answers", "negatives", "mask"):
            assert np.array_equal(b1[k], b2[k]), (structure, k)
        bits = kggen.unpack_mask(b1["mask"], 40)
        root = S.parse(S.STRUCTURE_DSL[structure])
        for i in range(10):
            A = S.exhaustive_answers(kg, root, b1["anchors"][i], b1["relations"][i])
            assert [p not in A for p in b1["negatives"]] == bits[i].tolist()
            # the positive is never a masked-in negative (A20)
            assert not any(bits[i][j] for j in range(40) if b1["negatives"][j] == b1["answers"][i])


def test_determinism_and_rank_streams():
    kg = small_kg(4)
    b0 = S.sample_batch(kg, "2i", 8, 16, seed=1, step=2, rank=0)
    b0b = S.sample_batch(kg, "2i", 8, 16, seed=1, step=2, rank=0)
    b1 = S.sample_batch(kg, "2i", 8, 16, seed=1, step=2, rank=1)
    assert all(np.array_equal(b0[k], b0b[k]) for k in ("anchors", "relations", "answers", "negatives", "mask"))
    assert not np.array_equal(b0["negatives"], b1["negatives"])
