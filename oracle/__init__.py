"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import, call or execute anything under `oracle/`.
The product path (`paper_2110_14890_b200/`, `include/kg.h`, the CUDA kernels)
never imports it, and this package never imports the product path: the two
share no code.  Their only common dependency is `kggen` (seeded input
generators and the input format, no method arithmetic).

What it is: a plain, slow, obviously-correct fp64 re-statement of the training
step of SMORE (arXiv 2110.14890) for GQE / Query2Box / BetaE over the 9 query
structures and the single-hop TransE / RotatE / DistMult / ComplEx models:

  model.py  forward definitions: entity activation, relation projection P,
            intersection I, DNF union, distance Dist      (Table 1 P:L137-143,
            Table 2, App. B, App. A, Def. 1
            P:L96-100; readings A1-A13, A19 in DESIGN.md)
  eval.py   filtered ranks and MRR / Hit@k of the evaluation path (App. F
            P:L700-705, reading A26)
  step.py   Eq. 1 loss, gradients, duplicate-row merge,
            sparse Adam on touched rows, dense Adam on theta_D
            (P:L307, L314), multi-worker semantics (reading A18),
            scoring for kg_score

Arithmetic is PyTorch CPU float64.  Gradients are obtained with torch.autograd
(a library primitive: reverse-mode differentiation of the written-out
definition); they are pinned independently by finite differences and by the
hand-derived worked example of tests/golden/ (see tests/test_oracle_pins.py).
Adam and the dedup are written out explicitly.

Parity status: every function here is pinned by at least one test in
tests/test_oracle_pins.py against a value the paper or mathematics fixes
(closed forms, worked examples, quadrature, special cases, finite
differences).  The operator architectures that the paper leaves unstated
(A4-A9, A14, A23) are conventions of DESIGN.md; they are pinned by FD,
invariants and special cases, not by a printed number ("parity unpinned by the
paper" for their exact architecture).
"""
from .model import (anchor_query, embed_entity, project, intersect, distance, negate,
                    query_disjuncts, dense_views)
from .step import (dedup, adam, SparseTable, oracle_step, oracle_score, oracle_score_each, StepResult,
                   softplus, query_loss_terms)
from .eval import ranks_from_distances, metrics_from_ranks, oracle_eval

__all__ = ["anchor_query", "embed_entity", "project", "intersect", "distance", "negate",
           "query_disjuncts", "dense_views", "dedup", "adam", "SparseTable",
           "oracle_step", "oracle_score", "oracle_score_each", "StepResult", "softplus", "query_loss_terms",
           "ranks_from_distances", "metrics_from_ranks", "oracle_eval"]
