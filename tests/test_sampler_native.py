"""Parity of the native sampler (libkgsample.so, include/kg_sample.h) with the sampler
oracle (oracle/sampler.py): the same counter-based draws must give bit-identical
batches (anchors, relations, answers, pool, mask) and identical App. C plans.  Host
code only: these run without a GPU."""
import os

import numpy as np
import pytest

import kggen
from oracle import sampler as S
from paper_2110_14890_b200 import sampler as N

KEYS = ("anchors", "relations", "answers", "negatives", "mask")


@pytest.fixture(scope="module")
def small():
    kg = kggen.make_kg(48, 3, 260, seed=0, a=0.5)
    return kg, S.OracleKG(kg), N.KGSampler(kg, n_threads=2)


@pytest.fixture(scope="module")
def fb15k():
    kg = kggen.make_kg(*kggen.KG_SHAPES["FB15k-237"], seed=1)
    return kg, S.OracleKG(kg), N.KGSampler(kg, n_threads=4)


@pytest.mark.parametrize("structure", kggen.ALL_STRUCTURES)
def test_plan_matches_oracle_dp(structure):
    root = S.parse(S.STRUCTURE_DSL[structure])
    u, s, o = S.annotate(root)
    assert N.plan(structure) == (u, s, o, S.optimal_cut(root))


def test_graph_dedup_and_roots(small):
    kg, okg, smp = small
    assert smp.n_edges == sum(len(v) for v in okg.in_edges.values()) == len(kg["h"])
    assert smp.n_roots == len(okg.roots)
    dup = dict(h=np.r_[kg["h"], kg["h"][:10]], r=np.r_[kg["r"], kg["r"][:10]], t=np.r_[kg["t"], kg["t"][:10]],
               n_entities=kg["n_entities"], n_relations=kg["n_relations"])
    assert N.KGSampler(dup, 1).n_edges == smp.n_edges


@pytest.mark.parametrize("structure", kggen.ALL_STRUCTURES)
def test_batch_bit_exact_vs_oracle_small(small, structure):
    kg, okg, smp = small
    for seed, step, rank in ((0, 0, 0), (3, 17, 1)):
        ref = S.sample_batch(okg, structure, 16, 40, seed=seed, step=step, rank=rank)
        got = smp.sample(structure, 16, 40, seed=seed, step=step, rank=rank)
        for k in KEYS + ("attempts",):
            assert np.array_equal(ref[k], got[k]), (structure, k)


@pytest.mark.parametrize("structure", ["1p", "3p", "ip", "pi", "up", "3in", "pni"])
def test_batch_bit_exact_vs_oracle_fb15k(fb15k, structure):
    """FB15k-237-shaped KG (Table 3): grounding bit-exact; mask vs the oracle's bidirectional search."""
    kg, okg, smp = fb15k
    M, K = 24, 300
    got = smp.sample(structure, M, K, seed=5, step=2)
    root = S.parse(S.STRUCTURE_DSL[structure])
    cut = S.optimal_cut(root)
    assert got["negatives"].tolist() == S.sample_pool(okg.V, K, 5, 2)
    bits = kggen.unpack_mask(got["mask"], K)
    for i in range(M):
        a, r, e, att = S.instantiate(okg, root, 5, 2, i)
        assert (got["anchors"][i].tolist(), got["relations"][i].tolist(), int(got["answers"][i]),
                int(got["attempts"][i])) == (a, r, e, att)
        cache = S.forward_cache(okg, root, cut, a, r)
        assert bits[i].tolist() == [not S.verify(okg, root, cache, r, p) for p in got["negatives"]]


def test_thread_count_does_not_change_the_batch(fb15k):
    kg, okg, smp = fb15k
    a = smp.sample("2i", 200, 256, seed=9, step=4, n_threads=1)
    b = smp.sample("2i", 200, 256, seed=9, step=4, n_threads=7)
    assert all(np.array_equal(a[k], b[k]) for k in KEYS)


@pytest.mark.parametrize("structure", ["2p", "2in", "inp", "up"])
def test_verify_matches_exhaustive(small, structure):
    kg, okg, smp = small
    root = S.parse(S.STRUCTURE_DSL[structure])
    rng = np.random.default_rng(4)
    M = 20
    a = rng.integers(0, okg.V, (M, N.N_ANCHORS[N.STRUCTS[structure]]))
    r = rng.integers(0, okg.R, (M, N.N_RELS[N.STRUCTS[structure]])).astype(np.int32)
    cand = np.arange(okg.V, dtype=np.int64)
    got = smp.verify(structure, a, r, cand)
    for i in range(M):
        A = S.exhaustive_answers(okg, root, a[i], r[i])
        assert got[i].tolist() == [v in A for v in range(okg.V)]
    per_query = np.tile(cand[::-1], (M, 1))
    assert np.array_equal(smp.verify(structure, a, r, per_query, shared=False), got[:, ::-1])


def test_pipeline_matches_direct_sampling(fb15k):
    kg, okg, smp = fb15k
    structs = ["1p", "2i", "pni"]
    for workers in (1, 3):
        p = N.Pipeline(smp, structs, 64, 128, seed=2, first_step=5, depth=4, n_workers=workers)
        for s in range(5, 12):
            b = p.next()
            assert b["step"] == s and b["structure"] == structs[s % 3]
            ref = smp.sample(b["structure"], 64, 128, seed=2, step=s)
            for k in KEYS:
                assert np.array_equal(b[k], ref[k]), (s, k)
        p.close()


def test_errors():
    kg = dict(h=np.array([0]), r=np.array([0], np.int32), t=np.array([1]), n_entities=2, n_relations=1)
    smp = N.KGSampler(kg, 1)
    assert smp.sample("1p", 3, 4)["answers"].tolist() == [1, 1, 1]
    with pytest.raises(N.KGSError) as e:          # no entity has an incoming edge to continue a 2p chain
        smp.sample("2p", 3, 4)
    assert e.value.status == 3
    with pytest.raises(S.SamplerError):
        S.instantiate(S.OracleKG(kg), S.parse(S.STRUCTURE_DSL["2p"]), 0, 0, 0)
    bad = dict(kg, t=np.array([5]))
    with pytest.raises(N.KGSError) as e:
        N.KGSampler(bad, 1)
    assert e.value.status == 1
    with pytest.raises(N.KGSError):
        smp.sample("1p", 0, 4)
    with pytest.raises(N.KGSError):
        smp.verify("1p", [[7]], [[0]], [0])
