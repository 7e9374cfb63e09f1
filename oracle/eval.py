"""Filtered ranking metrics of the evaluation path, fp64 (TEST INFRASTRUCTURE ONLY).

PAPER.md App. F P:L700-705 ("Calculation of evaluation metrics"): a missing answer
v of test query q is ranked against the non-answers; "for large-scale graphs ...
we randomly sample 1000 negative answers from V \\ A_q^{G_test} for each query",
and

    Metrics(q) = 1/|A_test \\ A_valid| * sum_v f(Rank(v)),  f(x) = 1/x (MRR),
                                                          f(x) = 1[x <= k] (Hit@k),

averaged over the queries of the set.  Readings (A26): the negatives are
given per query by the caller (already filtered, i.e. disjoint from A_q^{G_test});
Rank(v) = 1 + #{negatives j : Dist(q, v_j) <= Dist(q, v)}, ties counted against v
(pessimistic); Dist is the model's distance with the DNF min over
the disjuncts of a union (A11), lower = closer.
"""
from __future__ import annotations

import numpy as np

import kggen
from .step import SparseTable, oracle_score


def ranks_from_distances(d_ans: np.ndarray, d_neg: np.ndarray) -> np.ndarray:
    """Rank of each answer distance against the negative distances (pessimistic ties)."""
    d_ans = np.asarray(d_ans, np.float64).reshape(-1)
    d_neg = np.asarray(d_neg, np.float64).reshape(-1)
    return np.array([1 + int(np.count_nonzero(d_neg <= a)) for a in d_ans], dtype=np.int64)


def metrics_from_ranks(ranks: np.ndarray) -> np.ndarray:
    """[MRR, Hit@1, Hit@3, Hit@10] of one query from the ranks of its missing answers (App. F)."""
    r = np.asarray(ranks, np.float64)
    return np.array([np.mean(1.0 / r), np.mean(r <= 1), np.mean(r <= 3), np.mean(r <= 10)])


def oracle_eval(cfg: kggen.ModelConfig, table: SparseTable, batch: dict, ans_off, ans_ids, negatives):
    """Ranks of every missing answer, per-query metrics and the per-answer decision margin.

    batch: structure / anchors / relations of M queries; ans_off [M+1], ans_ids (CSR of the
    missing answers); negatives [M][n_neg] (per query).  Returns (ranks [n_ans] int64,
    metrics [M][4], margin [n_ans]: min_j |D_neg_j - D_v|, the distance to the nearest
    tie decision, used by the parity tests to separate ranks fp32 cannot decide).
    """
    ans_off = np.asarray(ans_off, np.int64)
    ans_ids = np.asarray(ans_ids, np.int64)
    negatives = np.asarray(negatives, np.int64)
    M = len(ans_off) - 1
    ranks = np.zeros(len(ans_ids), np.int64)
    margin = np.zeros(len(ans_ids))
    metrics = np.zeros((M, 4))
    for i in range(M):
        qb = {"structure": batch["structure"], "anchors": np.asarray(batch["anchors"])[i:i + 1],
              "relations": np.asarray(batch["relations"])[i:i + 1]}
        a = ans_ids[ans_off[i]:ans_off[i + 1]]
        D = oracle_score(cfg, table, qb, np.concatenate([a, negatives[i]]))[0]
        d_ans, d_neg = D[:len(a)], D[len(a):]
        r = ranks_from_distances(d_ans, d_neg)
        ranks[ans_off[i]:ans_off[i + 1]] = r
        margin[ans_off[i]:ans_off[i + 1]] = [np.min(np.abs(d_neg - x)) if len(d_neg) else np.inf for x in d_ans]
        metrics[i] = metrics_from_ranks(r)
    return ranks, metrics, margin
