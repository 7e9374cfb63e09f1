"""Pins of the evaluation oracle (oracle/eval.py) against what App. F fixes (-m "not gpu").

PAPER.md App. F: rank each missing answer against (sampled) non-answers,
Metrics(q) = mean over the query's missing answers of f(Rank), f = 1/x (MRR) or
1[x <= k] (Hit@k), then the mean over queries.  Ties are counted against the answer
(reading A26).
"""
import math

import numpy as np
import pytest

import kggen
import oracle


def test_rank_special_cases():
    # strictly closest -> 1; a tie with one negative -> 2 (pessimistic); farthest -> n + 1
    assert oracle.ranks_from_distances([1.0], [2.0, 3.0, 4.0]).tolist() == [1]
    assert oracle.ranks_from_distances([2.0], [2.0, 3.0, 4.0]).tolist() == [2]
    assert oracle.ranks_from_distances([5.0], [2.0, 3.0, 4.0]).tolist() == [4]
    assert oracle.ranks_from_distances([3.0, 0.5], [2.0, 3.0, 4.0]).tolist() == [3, 1]


def test_metric_worked_examples():
    # App. F formula written out by hand
    np.testing.assert_allclose(oracle.metrics_from_ranks([2]), [0.5, 0.0, 1.0, 1.0])
    np.testing.assert_allclose(oracle.metrics_from_ranks([1, 4]), [0.625, 0.5, 0.5, 1.0])
    np.testing.assert_allclose(oracle.metrics_from_ranks([11, 3, 10]),
                               [(1 / 11 + 1 / 3 + 1 / 10) / 3, 0.0, 1 / 3, 2 / 3])


def test_rank_monotone_in_answer_distance():
    rng = np.random.default_rng(0)
    neg = rng.standard_normal(200)
    a = rng.standard_normal(50)
    r0 = oracle.ranks_from_distances(a, neg)
    r1 = oracle.ranks_from_distances(a - np.abs(rng.standard_normal(50)), neg)   # answers move closer
    assert np.all(r1 <= r0)
    r = oracle.ranks_from_distances(a, neg)
    m = oracle.metrics_from_ranks(r)
    assert m[1] <= m[2] <= m[3] and m[1] <= m[0] <= 1.0      # Hit@1 <= Hit@3 <= Hit@10, MRR >= Hit@1


@pytest.mark.parametrize("kind,structure", [("gqe", "2i"), ("q2b", "2u"), ("betae", "ip")])
def test_sampled_ranking_equals_full_enumeration(kind, structure):
    """Negatives = every non-answer of a 60-entity KG: the rank equals the position of v
    in the full sort of {v} + all non-answers (other answers filtered), ties against v."""
    cfg = kggen.ModelConfig(kind, 8, 60, 5, hidden=8)
    table = oracle.SparseTable(cfg, 3)
    b = kggen.make_batch(cfg, structure, 4, 4, seed=2)
    rng = np.random.default_rng(1)
    answers = [np.sort(rng.choice(60, size=3, replace=False)) for _ in range(4)]
    non = [np.setdiff1d(np.arange(60), a) for a in answers]
    ans_off = np.cumsum([0] + [3] * 4)
    negatives = np.stack(non)                                  # 57 non-answers each
    ranks, metrics, _ = oracle.oracle_eval(cfg, table, b, ans_off, np.concatenate(answers), negatives)
    D = oracle.oracle_score(cfg, table, b, np.arange(60))      # every entity
    for i in range(4):
        for t, v in enumerate(answers[i]):
            pool = np.concatenate([[v], non[i]])
            # sort key (distance, answer-last): ties put the answer after the negatives
            order = np.lexsort((np.r_[1, np.zeros(len(non[i]))], D[i, pool]))
            assert ranks[3 * i + t] == int(np.nonzero(order == 0)[0][0]) + 1
        np.testing.assert_allclose(metrics[i], oracle.metrics_from_ranks(ranks[3 * i:3 * i + 3]))


def test_random_model_mrr_matches_uniform_rank_expectation():
    """Answers and negatives drawn i.i.d. from the same law, independent of the query:
    Rank is uniform on {1..n+1} (exchangeability), so E[1/Rank] = H_{n+1} / (n+1)."""
    cfg = kggen.ModelConfig("gqe", 8, 5000, 7)
    table = oracle.SparseTable(cfg, 4)
    M, n = 400, 40
    b = kggen.make_batch(cfg, "1p", M, 4, seed=5)
    rng = np.random.default_rng(9)
    ans = rng.integers(0, 5000, size=M)
    neg = rng.integers(0, 5000, size=(M, n))
    _, metrics, _ = oracle.oracle_eval(cfg, table, b, np.arange(M + 1), ans, neg)
    k = np.arange(1, n + 2)
    mu = np.mean(1.0 / k)
    sd = math.sqrt((np.mean(1.0 / k ** 2) - mu ** 2) / M)
    assert abs(metrics[:, 0].mean() - mu) < 4 * sd
    assert abs(metrics[:, 3].mean() - 10 / (n + 1)) < 4 * math.sqrt((10 / (n + 1)) * (1 - 10 / (n + 1)) / M)
