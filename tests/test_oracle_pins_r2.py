"""Pins for the oracle functions round 1 left unpinned (-m "not gpu").

Values come from tests/golden/pins_r2.json, written by tests/golden/derive_pins_r2.py,
which evaluates hand-set worked examples with plain numpy / scipy.special closed forms and
never imports oracle/ (see its docstring for the operator closed forms and citations).

  * DNF union = min over disjuncts; the gradient flows only into the argmin disjunct
    (Def. 1, reading A11)                      test_union_*
  * Q2B intersection: softmax attention over the inputs for the center and
    min(offsets) * sigmoid(DeepSet(offsets)) for the offset (Table 1, A4/A5)
                                                                   test_structure_examples[q2b:*]
  * Q2B projection offset o + ReLU(r_o) (A6)               test_q2b_projection_relu
  * Eq. 1's 1/|N_q| over the query's own negatives (Mask P:L389, A12)
                                                                   test_partial_mask_*
  * the structure DAGs' slot wiring and the negated branch of 2in/3in/inp/pin/pni
    (readings A21, A25): every other wiring changes D+ or D- in these
    examples (the derivation script checks it)                   test_structure_examples
  * BetaE projection clamp(MLP + 1, 0.05, 1e9) (A8, A9)   test_betae_projection_zero_mlp
  * oracle/sampler.py's S-expressions and oracle.model.query_disjuncts agree on slot order
                                                                   test_sampler_dsl_matches_query_disjuncts
"""
import json
import os

import numpy as np
import pytest
import torch

import kggen
import oracle
import oracle.model as om
from oracle.model import dense_views
from oracle import sampler as osmp

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins_r2.json")))
F64 = torch.float64
POS, NEG = 5, 6          # entity ids of the positive and the negative in the examples


def _set(cfg, dense, name, value):
    offs, _ = kggen.dense_offsets(cfg)
    o, shape = offs[name]
    dense[o:o + int(np.prod(shape))] = np.asarray(value, np.float32).reshape(-1)


def _special_weights(cfg, dense):
    """The operator weights under which Table 1's operators reduce to the closed forms of
    derive_pins_r2.py (identity MLPs, zero biases)."""
    d = cfg.dim
    eye = np.eye(d)
    if cfg.kind == "gqe":
        _set(cfg, dense, "ds_W1", eye)
        _set(cfg, dense, "ds_W2", eye)
    elif cfg.kind == "q2b":
        for n in ("att_W1", "att_W2", "off_W1", "off_W2"):
            _set(cfg, dense, n, eye)
    elif cfg.kind == "betae":
        H = cfg.hidden
        assert H == 2 * d
        _set(cfg, dense, "prj_W1", np.eye(H))
        _set(cfg, dense, "prj_W2", np.eye(H))
        _set(cfg, dense, "prj_W0", np.concatenate([2 * eye, eye], axis=1))
        _set(cfg, dense, "att_U1", eye)
        _set(cfg, dense, "att_U2", np.concatenate([np.eye(d // 2), np.zeros((d // 2, d // 2))], axis=1))


def _example_step(kind, structure, ex, apply=False):
    na, nr = kggen.N_ANCHORS[structure], kggen.N_RELS[structure]
    d = {"gqe": 2, "q2b": 2, "betae": 4}[kind]
    cfg = kggen.ModelConfig(kind, d, 10, nr, hidden=2 * d if kind == "betae" else None, gamma=ex["gamma"])
    _, n = kggen.dense_offsets(cfg)
    dense = np.zeros(n, np.float32)
    _special_weights(cfg, dense)
    for key in ex["relations"][0]:
        _set(cfg, dense, key, [r[key] for r in ex["relations"]])
    t = oracle.SparseTable(cfg, 0)
    t.dense = dense
    t.dense_m = np.zeros_like(dense)
    t.dense_v = np.zeros_like(dense)
    ids = list(range(na)) + [POS, NEG]
    rows = np.array(ex["anchors"] + [ex["positive"], ex["negative"]], np.float32)
    t.set(ids, rows, np.zeros_like(rows), np.zeros_like(rows))
    b = dict(structure=structure, anchors=np.arange(na, dtype=np.int64)[None],
             relations=np.arange(nr, dtype=np.int32)[None], answers=np.array([POS], np.int64),
             negatives=np.array([NEG], np.int64), mask=kggen.pack_mask(np.ones((1, 1), bool)), K=1, M=1)
    return cfg, oracle.oracle_step(cfg, t, [b], 0.1, apply=apply)


@pytest.mark.parametrize("key", sorted(GOLD["structures"]))
def test_structure_examples(key):
    kind, structure = key.split(":")
    ex = GOLD["structures"][key]
    _, r = _example_step(kind, structure, ex)
    assert r.d_pos[0][0] == pytest.approx(ex["d_pos"], rel=1e-12)
    assert r.d_neg[0][0, 0] == pytest.approx(ex["d_neg"], rel=1e-12)
    assert r.loss == pytest.approx(ex["loss"], rel=1e-12)


@pytest.mark.parametrize("structure", ["2u", "up"])
def test_union_min_and_argmin_gradient(structure):
    ex = GOLD["union_gradient"][structure]
    cfg = kggen.ModelConfig("gqe", 2, 10, len(ex["relations"]), gamma=ex["gamma"])
    _, n = kggen.dense_offsets(cfg)
    dense = np.zeros(n, np.float32)
    _set(cfg, dense, "rel", ex["relations"])
    t = oracle.SparseTable(cfg, 0)
    t.dense, t.dense_m, t.dense_v = dense, np.zeros_like(dense), np.zeros_like(dense)
    rows = np.array(ex["anchors"] + [ex["positive"], ex["negative"]], np.float32)
    t.set([0, 1, POS, NEG], rows, np.zeros_like(rows), np.zeros_like(rows))
    nr = len(ex["relations"])
    b = dict(structure=structure, anchors=np.array([[0, 1]], np.int64), relations=np.arange(nr, dtype=np.int32)[None],
             answers=np.array([POS], np.int64), negatives=np.array([NEG], np.int64),
             mask=kggen.pack_mask(np.ones((1, 1), bool)), K=1, M=1)
    r = oracle.oracle_step(cfg, t, [b], 0.1, apply=False)
    # D = min over the disjuncts, not max or mean (Def. 1, A11)
    assert r.d_pos[0][0] == pytest.approx(ex["d_pos"], rel=1e-14)
    assert r.d_neg[0][0, 0] == pytest.approx(ex["d_neg"], rel=1e-14)
    assert ex["d_pos_max"] > ex["d_pos"] + 1 and ex["d_neg_max"] > ex["d_neg"] + 1
    assert r.loss == pytest.approx(ex["loss"], rel=1e-14)
    g = dict(zip(r.uniq.tolist(), r.grad_rows))
    for a in range(2):     # each anchor receives only the term whose argmin is its disjunct
        np.testing.assert_allclose(g[a], ex["grad_anchors"][a], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(g[POS], ex["grad_positive"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(g[NEG], ex["grad_negative"], rtol=1e-12, atol=1e-15)
    offs, _ = kggen.dense_offsets(cfg)
    o, _ = offs["rel"]
    np.testing.assert_allclose(r.grad_dense[o:o + 2 * nr].reshape(nr, 2), ex["grad_relations"], rtol=1e-12, atol=1e-15)


def test_union_score_is_dnf_min():
    # kg_score's oracle takes the same min over disjuncts (A11)
    ex = GOLD["union_gradient"]["2u"]
    cfg = kggen.ModelConfig("gqe", 2, 10, 2, gamma=ex["gamma"])
    _, n = kggen.dense_offsets(cfg)
    dense = np.zeros(n, np.float32)
    _set(cfg, dense, "rel", ex["relations"])
    t = oracle.SparseTable(cfg, 0, dense=dense)
    rows = np.array(ex["anchors"] + [ex["positive"], ex["negative"]], np.float32)
    t.set([0, 1, POS, NEG], rows, np.zeros_like(rows), np.zeros_like(rows))
    b = dict(structure="2u", anchors=np.array([[0, 1]], np.int64), relations=np.array([[0, 1]], np.int32))
    D = oracle.oracle_score(cfg, t, b, [POS, NEG])
    np.testing.assert_allclose(D[0], [ex["d_pos"], ex["d_neg"]], rtol=1e-14)


def test_score_each_per_query_candidates():
    # kg_score_each's oracle (per-query candidates, SURVEY §8(b) shared = 0) on the same worked
    # 2u example: each query row scores only its own candidates, with the DNF min (A11);
    # a second query with the candidates swapped gets the swapped distances
    ex = GOLD["union_gradient"]["2u"]
    cfg = kggen.ModelConfig("gqe", 2, 10, 2, gamma=ex["gamma"])
    _, n = kggen.dense_offsets(cfg)
    dense = np.zeros(n, np.float32)
    _set(cfg, dense, "rel", ex["relations"])
    t = oracle.SparseTable(cfg, 0, dense=dense)
    rows = np.array(ex["anchors"] + [ex["positive"], ex["negative"]], np.float32)
    t.set([0, 1, POS, NEG], rows, np.zeros_like(rows), np.zeros_like(rows))
    b = dict(structure="2u", anchors=np.array([[0, 1], [0, 1]], np.int64), relations=np.array([[0, 1], [0, 1]], np.int32))
    D = oracle.oracle_score_each(cfg, t, b, np.array([[POS, NEG], [NEG, POS]]))
    np.testing.assert_allclose(D, [[ex["d_pos"], ex["d_neg"]], [ex["d_neg"], ex["d_pos"]]], rtol=1e-14)


@pytest.mark.parametrize("kind,structure", [("q2b", "pi"), ("betae", "2in"), ("rotate", "1p"), ("gqe", "up")])
def test_score_each_rows_equal_shared_scores(kind, structure):
    # with every query given the same candidate list the per-query scores reduce to the
    # shared-candidate scores (oracle_score, pinned above), row by row
    cfg = kggen.ModelConfig(kind, 8, 50, 5, hidden=16 if kind == "betae" else None)
    t = oracle.SparseTable(cfg, 3)
    b = kggen.make_batch(cfg, structure, 4, 6, seed=5)
    cand = np.array([3, 17, 17, 0, 49])
    shared = oracle.oracle_score(cfg, t, b, cand)
    each = oracle.oracle_score_each(cfg, t, b, np.tile(cand, (4, 1)))
    np.testing.assert_allclose(each, shared, rtol=1e-13, atol=0)
    # and a permutation of one query's candidates permutes only that query's row
    perm = np.tile(cand, (4, 1))
    perm[2] = cand[::-1]
    each2 = oracle.oracle_score_each(cfg, t, b, perm)
    np.testing.assert_allclose(each2[2], shared[2][::-1], rtol=1e-13, atol=0)
    np.testing.assert_allclose(np.delete(each2, 2, 0), np.delete(shared, 2, 0), rtol=1e-13, atol=0)


def _partial_mask_run():
    ex = GOLD["partial_mask"]
    cfg = kggen.ModelConfig("gqe", 2, 20, 1, gamma=ex["gamma"])
    _, n = kggen.dense_offsets(cfg)
    t = oracle.SparseTable(cfg, 0, dense=np.zeros(n, np.float32))
    ids = [0, 1, POS, 10, 11, 12]
    rows = np.array(ex["queries"] + [ex["positive"]] + ex["pool"], np.float32)
    t.set(ids, rows, np.zeros_like(rows), np.zeros_like(rows))
    b = dict(structure="1p", anchors=np.array([[0], [1]], np.int64), relations=np.zeros((2, 1), np.int32),
             answers=np.array([POS, POS], np.int64), negatives=np.array([10, 11, 12], np.int64),
             mask=kggen.pack_mask(np.array(ex["mask"], bool)), K=3, M=2)
    return ex, oracle.oracle_step(cfg, t, [b], 0.1, apply=False)


def test_partial_mask_loss_uses_own_negative_count():
    ex, r = _partial_mask_run()
    assert r.loss == pytest.approx(ex["loss"], rel=1e-13)


def test_partial_mask_pool_gradients():
    ex, r = _partial_mask_run()
    g = dict(zip(r.uniq.tolist(), r.grad_rows))
    for j, e in enumerate((10, 11, 12)):
        np.testing.assert_allclose(g[e], ex["grad_pool"][j], rtol=1e-12, atol=1e-15)


def test_q2b_projection_relu():
    ex = GOLD["q2b_projection_relu"]
    cfg = kggen.ModelConfig("q2b", 2, 10, 1)
    _, n = kggen.dense_offsets(cfg)
    dense = np.zeros(n, np.float32)
    _set(cfg, dense, "rel_center", ex["rel_center"])
    _set(cfg, dense, "rel_offset", ex["rel_offset"])
    t = oracle.SparseTable(cfg, 0, dense=dense)
    rows = np.array([ex["anchor"], ex["v"]], np.float32)
    t.set([0, 1], rows, np.zeros_like(rows), np.zeros_like(rows))
    D = oracle.oracle_score(cfg, t, dict(structure="1p", anchors=np.array([[0]]), relations=np.array([[0]])), [1])
    assert D[0, 0] == pytest.approx(ex["dist"], rel=1e-14)


def test_betae_projection_zero_mlp():
    ex = GOLD["betae_projection_zero_mlp"]
    cfg = kggen.ModelConfig("betae", 4, 10, 1, hidden=8)
    _, n = kggen.dense_offsets(cfg)
    dense = np.zeros(n, np.float64)
    offs, _ = kggen.dense_offsets(cfg)
    o, _ = offs["prj_b0"]
    dense[o:o + 4] = ex["b0"]
    P = dense_views(cfg, torch.tensor(dense, dtype=F64))
    q = torch.tensor([[0.7, 1.3, 2.0, 0.4]], dtype=F64)
    out = oracle.project("betae", q, torch.tensor([0]), P)
    np.testing.assert_allclose(out[0].numpy(), ex["out"], rtol=1e-15)


# -------------------------------------------- sampler DSL vs query_disjuncts (A21, S1)
def _dnf(node):
    """Symbolic DNF disjuncts of an oracle/sampler.py tree (slots as written by its parser)."""
    if node.op == "a":
        return [f"a{node.slot}"]
    if node.op == "p":
        return [f"p({q},r{node.slot})" for q in _dnf(node.children[0])]
    if node.op == "n":
        return [f"n({q})" for q in _dnf(node.children[0])]
    if node.op == "u":
        return [q for c in node.children for q in _dnf(c)]
    if node.op == "i":
        parts = [_dnf(c) for c in node.children]
        assert all(len(p) == 1 for p in parts)
        return ["i(" + ",".join(p[0] for p in parts) + ")"]
    raise ValueError(node.op)


@pytest.mark.parametrize("structure", kggen.ALL_STRUCTURES)
def test_sampler_dsl_matches_query_disjuncts(structure, monkeypatch):
    monkeypatch.setattr(om, "anchor_query", lambda kind, x: x)
    monkeypatch.setattr(om, "project", lambda kind, q, r, P: f"p({q},{r})")
    monkeypatch.setattr(om, "intersect", lambda kind, qs, P: "i(" + ",".join(qs) + ")")
    monkeypatch.setattr(om, "negate", lambda kind, q: f"n({q})")
    na, nr = kggen.N_ANCHORS[structure], kggen.N_RELS[structure]
    got = om.query_disjuncts(structure, "betae", [f"a{k}" for k in range(na)], [f"r{k}" for k in range(nr)], {})
    assert got == _dnf(osmp.parse(osmp.STRUCTURE_DSL[structure]))
