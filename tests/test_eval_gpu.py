"""Parity of the evaluation path kg_eval (k_eval.cu) with oracle/eval.py (-m gpu).

Ranks are integers decided by fp32 distance comparisons on the GPU and by fp64 ones
in the oracle (reading A26): a rank must equal the oracle's exactly when no negative
lies within the fp32 resolution of the answer's distance, and lie between the strict
and the tie-inclusive counts otherwise.  Metrics must equal the App. F formula of the
GPU's own ranks (and the oracle's where all ranks are decided).
"""
import numpy as np
import pytest

import kggen
import oracle

pytestmark = pytest.mark.gpu

CASES = [("gqe", "1p"), ("gqe", "ip"), ("q2b", "2u"), ("q2b", "pi"), ("betae", "up"), ("betae", "pni"),
         ("betae", "3i"), ("transe", "1p"), ("rotate", "1p"), ("distmult", "1p"), ("complex", "1p"),
         ("rotate-m", "2i"), ("distmult-m", "ip"), ("complex-m", "2u")]


def _model(cfg, max_M):
    from paper_2110_14890_b200 import KGModel
    m = KGModel(cfg, max_M, 16, 0)
    m.init_params(5)
    return m


def _inputs(rng, M, n_ent, n_neg, max_ans=5):
    """Missing answers per query and n_neg negatives sampled from the non-answers (App. F)."""
    counts = rng.integers(1, max_ans + 1, size=M)
    ans_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    ans = [rng.choice(n_ent, size=c, replace=False) for c in counts]
    negatives = np.stack([rng.choice(np.setdiff1d(np.arange(n_ent), a), size=n_neg) for a in ans])
    return ans_off, np.concatenate(ans), negatives


@pytest.mark.parametrize("kind,structure", CASES)
def test_eval_parity(kind, structure):
    cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
    gm = _model(cfg, 40)
    table = oracle.SparseTable(cfg, 5)
    M, n_neg = 37, 150
    b = kggen.make_batch(cfg, structure, M, 4, seed=4)
    rng = np.random.default_rng(11)
    ans_off, ans_ids, negatives = _inputs(rng, M, 300, n_neg)
    ranks, metrics = gm.eval(gm.host_batch(b), ans_off, ans_ids, negatives)
    ref_ranks, ref_metrics, margin = oracle.oracle_eval(cfg, table, b, ans_off, ans_ids, negatives)
    # the fp32 resolution of the distances of this case
    D = np.concatenate([oracle.oracle_score(cfg, table, {k: (np.asarray(b[k])[i:i + 1] if k != "structure" else b[k])
                                                          for k in ("structure", "anchors", "relations")},
                                            np.concatenate([ans_ids[ans_off[i]:ans_off[i + 1]], negatives[i]]))[0]
                        for i in range(M)])
    tol = 1e-5 * (np.abs(D).max() + 1.0)
    decided = margin > tol
    assert decided.mean() > 0.9
    np.testing.assert_array_equal(ranks[decided], ref_ranks[decided])
    # undecided answers: between the strict and the tie-inclusive count of the oracle
    for i in range(M):
        qb = {"structure": b["structure"], "anchors": np.asarray(b["anchors"])[i:i + 1],
              "relations": np.asarray(b["relations"])[i:i + 1]}
        for k in range(ans_off[i], ans_off[i + 1]):
            if decided[k]:
                continue
            d = oracle.oracle_score(cfg, table, qb, np.concatenate([[ans_ids[k]], negatives[i]]))[0]
            lo = 1 + np.count_nonzero(d[1:] < d[0] - tol)
            hi = 1 + np.count_nonzero(d[1:] <= d[0] + tol)
            assert lo <= ranks[k] <= hi
    # metrics are the App. F formula of the GPU ranks
    for i in range(M):
        np.testing.assert_allclose(metrics[i], oracle.metrics_from_ranks(ranks[ans_off[i]:ans_off[i + 1]]),
                                   rtol=1e-6, atol=1e-7)
    full = np.array([decided[ans_off[i]:ans_off[i + 1]].all() for i in range(M)])
    np.testing.assert_allclose(metrics[full], ref_metrics[full], rtol=1e-6, atol=1e-7)
    gm.close()


def test_eval_edge_cases():
    from paper_2110_14890_b200 import KGError
    cfg = kggen.ModelConfig("q2b", 40, 300, 7)
    gm = _model(cfg, 40)
    b = kggen.make_batch(cfg, "2i", 5, 4, seed=4)
    # no negatives: every answer ranks first
    ranks, metrics = gm.eval(gm.host_batch(b), np.arange(6), np.arange(5), np.zeros((5, 0), np.int64))
    assert ranks.tolist() == [1] * 5 and np.all(metrics == 1.0)
    # the answer itself, three times, as the negatives: the ties count against it
    negs = np.arange(5)[:, None].repeat(3, axis=1)
    ranks, _ = gm.eval(gm.host_batch(b), np.arange(6), np.arange(5), negs)
    assert ranks.tolist() == [4] * 5
    # validation
    with pytest.raises(KGError) as e:
        gm.eval(gm.host_batch(b), np.array([0, 1, 1, 2, 3, 4]), np.arange(4), np.zeros((5, 2), np.int64))
    assert e.value.status == 1                        # a query without missing answers
    with pytest.raises(KGError) as e:
        gm.eval(gm.host_batch(b), np.arange(6), np.array([0, 1, 2, 3, 300]), np.zeros((5, 2), np.int64))
    assert e.value.status == 1                        # answer id out of range
    with pytest.raises(KGError) as e:
        gm.eval(gm.host_batch(kggen.make_batch(cfg, "2in", 5, 4, seed=4)), np.arange(6), np.arange(5),
                np.zeros((5, 2), np.int64))
    assert e.value.status == 2                        # negation needs BetaE
    gm.close()


def test_eval_large_negative_pool_matches_score():
    """1000 negatives per query (App. F): ranks equal those recomputed from kg_score distances."""
    cfg = kggen.ModelConfig("betae", 64, 5000, 11, hidden=64)
    from paper_2110_14890_b200 import KGModel
    gm = KGModel(cfg, 64, 16, 1001)
    gm.init_params(3)
    M = 64
    b = kggen.make_batch(cfg, "ip", M, 4, seed=4)
    rng = np.random.default_rng(2)
    ans_off = np.arange(M + 1)
    ans_ids = rng.integers(0, 5000, size=M)
    negatives = rng.integers(0, 5000, size=(M, 1000))
    negatives[negatives == ans_ids[:, None]] = (ans_ids[:, None].repeat(1000, 1)[negatives == ans_ids[:, None]] + 1) % 5000
    ranks, _ = gm.eval(gm.host_batch(b), ans_off, ans_ids, negatives)
    for i in range(0, M, 8):
        qb = dict(b, anchors=np.asarray(b["anchors"])[i:i + 1], relations=np.asarray(b["relations"])[i:i + 1], M=1)
        d = gm.score(gm.host_batch(qb), np.concatenate([[ans_ids[i]], negatives[i]]))[0]
        # both kernels are fp32 but sum in different orders: allow the near-ties to move
        tol = 1e-5 * np.abs(d).max()
        assert 1 + np.count_nonzero(d[1:] < d[0] - tol) <= ranks[i] <= 1 + np.count_nonzero(d[1:] <= d[0] + tol)
    gm.close()


@pytest.mark.parametrize("kind,structure", [("q2b", "ip"), ("betae", "pin"), ("gqe", "2u")])
def test_eval_on_a_built_eval_set(kind, structure):
    """kg_eval on an App. E evaluation set built by the native sampler on a split synthetic KG
    (queries on G_test, missing answers A(G_test) minus A(G_valid), filtered negatives): ranks
    decided in fp32 equal the oracle's (same decided / undecided rule as test_eval_parity)."""
    from paper_2110_14890_b200 import sampler as N
    kg = kggen.make_kg(300, 7, 3000, seed=9, a=0.6)
    tr, va, te = kggen.split_kg(kg, valid_frac=0.1, test_frac=0.1, seed=2)
    b, ans_off, ans_ids, negatives = N.build_eval_set(N.KGSampler(te, 2), N.KGSampler(va, 2), structure, 24,
                                                      n_neg=120, seed=3)
    cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
    gm = _model(cfg, 24)
    table = oracle.SparseTable(cfg, 5)
    ranks, metrics = gm.eval(gm.host_batch(dict(b, K=0, answers=np.zeros(24, np.int64),
                                                negatives=np.zeros(0, np.int64),
                                                mask=np.zeros((24, 1), np.uint32))),
                             ans_off, ans_ids, negatives)
    ref_ranks, ref_metrics, margin = oracle.oracle_eval(cfg, table, b, ans_off, ans_ids, negatives)
    decided = margin > 1e-3          # far above the fp32 resolution of these distances (<= ~60)
    assert decided.mean() > 0.8
    np.testing.assert_array_equal(ranks[decided], ref_ranks[decided])
    assert np.all((metrics >= 0) & (metrics <= 1))
    gm.close()
