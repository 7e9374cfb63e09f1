"""Pin the CPU oracle to things other than itself (-m "not gpu").

Every pin here is fixed by the paper's formulas worked by hand
(tests/golden/pins.json, each entry cited), by mathematics (closed forms,
quadrature, finite differences, invariants) or by a special case that reduces
to a textbook routine (numpy complex arithmetic, scipy special functions) --
never by re-running the oracle's own expression.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import kggen
import oracle
from oracle.model import beta_kl, dense_views

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))
F64 = torch.float64


def _table(cfg, rows=None, dense=None, seed=0):
    t = oracle.SparseTable(cfg, seed)
    if dense is not None:
        t.dense = np.asarray(dense, np.float32)
        t.dense_m = np.zeros_like(t.dense)
        t.dense_v = np.zeros_like(t.dense)
    if rows:
        ids = list(rows)
        p = np.array([rows[i] for i in ids], np.float32)
        t.set(ids, p, np.zeros_like(p), np.zeros_like(p))
    return t


def _batch(structure, anchors, relations, answers, negatives, mask_bits):
    M = len(answers)
    bits = np.asarray(mask_bits, bool).reshape(M, len(negatives))
    return dict(structure=structure, anchors=np.asarray(anchors, np.int64).reshape(M, -1),
                relations=np.asarray(relations, np.int32).reshape(M, -1),
                answers=np.asarray(answers, np.int64), negatives=np.asarray(negatives, np.int64),
                mask=kggen.pack_mask(bits), K=len(negatives), M=M)


# ------------------------------------------------------------------ P2 loss
@pytest.mark.parametrize("key", ["loss_fixed_point", "loss_margin_example"])
def test_loss_closed_forms(key):
    g = GOLD[key]
    # GQE d=2 with anchor 0 and zero relation so q = 0; points at the wanted distances.
    cfg = kggen.ModelConfig("gqe", 2, 10, 1, gamma=g["gamma"])
    offs, n = kggen.dense_offsets(cfg)
    dense = np.zeros(n, np.float32)
    rows = {0: [0.0, 0.0], 1: [g["d_pos"], 0.0]}
    for j, dn in enumerate(g["d_neg"]):
        rows[2 + j] = [0.0, dn]
    t = _table(cfg, rows, dense)
    b = _batch("1p", [0], [0], [1], list(range(2, 2 + len(g["d_neg"]))), [1] * len(g["d_neg"]))
    r = oracle.oracle_step(cfg, t, [b], lr=0.1, apply=False)
    assert r.loss == pytest.approx(g["loss"], rel=1e-14, abs=1e-15)


def test_empty_mask_row_drops_negative_term():
    cfg = kggen.ModelConfig("gqe", 2, 10, 1, gamma=1.0)
    _, n = kggen.dense_offsets(cfg)
    t = _table(cfg, {0: [0, 0], 1: [1, 0], 2: [0, 3]}, np.zeros(n, np.float32))
    b = _batch("1p", [0], [0], [1], [2], [0])
    r = oracle.oracle_step(cfg, t, [b], lr=0.1, apply=False)
    assert r.loss == pytest.approx(math.log(2.0), rel=1e-14)     # softplus(1 - 1) only


# ------------------------------------------------------- P3 worked example
def test_gqe_worked_example():
    g = GOLD["gqe_worked_example"]
    cfg = kggen.ModelConfig("gqe", g["dim"], 10, 1, gamma=g["gamma"])
    offs, n = kggen.dense_offsets(cfg)
    dense = np.zeros(n, np.float32)
    o, _ = offs["rel"]
    dense[o:o + 2] = g["relation"]
    rows = {0: g["anchor"], 1: g["positive"], 2: g["pool"][0], 3: g["pool"][1]}
    t = _table(cfg, rows, dense)
    b = _batch("1p", [0], [0], [1], [2, 3], g["mask"])
    r = oracle.oracle_step(cfg, t, [b], lr=0.1, apply=False)
    assert r.loss == pytest.approx(g["loss"], rel=1e-12)
    assert r.d_pos[0][0] == pytest.approx(0.0, abs=1e-15)
    np.testing.assert_allclose(r.d_neg[0][0], [1.0, 5.0], rtol=1e-14)
    grad = dict(zip(r.uniq.tolist(), r.grad_rows))
    np.testing.assert_allclose(grad[0], g["grad_anchor"], rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(grad[1], g["grad_positive"], atol=1e-15)
    np.testing.assert_allclose(grad[2], g["grad_pool"][0], rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(grad[3], g["grad_pool"][1], rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(r.grad_dense[o:o + 2], g["grad_relation"], rtol=1e-9)
    # DeepSet weights are not on the 1p path: zero gradient
    assert np.all(r.grad_dense[o + 2:] == 0)


def test_gqe_2p_closed_form_3_4_5():
    # GQE 2p q = x_a + y1 + y2; 3-4-5 triangle gives D+ = 5 exactly
    cfg = kggen.ModelConfig("gqe", 2, 10, 2, gamma=3.0)
    offs, n = kggen.dense_offsets(cfg)
    dense = np.zeros(n, np.float32)
    o, _ = offs["rel"]
    dense[o:o + 4] = [1, 0, 0, 2]
    t = _table(cfg, {0: [0, 0], 1: [4, 6], 2: [1, 2]}, dense)
    b = _batch("2p", [0], [0, 1], [1], [2], [1])
    r = oracle.oracle_step(cfg, t, [b], lr=0.1, apply=False)
    assert r.d_pos[0][0] == pytest.approx(5.0, rel=1e-15)
    assert r.d_neg[0][0, 0] == pytest.approx(0.0, abs=1e-15)


# ------------------------------------------------------------------- P4 Q2B
def test_q2b_box_distance():
    g = GOLD["q2b_box_distance"]
    q = torch.tensor(g["center"] + g["offset"], dtype=F64)
    v = torch.tensor(g["v"], dtype=F64)
    assert float(oracle.distance("q2b", q, v, g["alpha"])) == pytest.approx(g["dist"], rel=1e-15)


def test_q2b_zero_offset_is_l1():
    rng = np.random.default_rng(0)
    c, v = rng.normal(size=(2, 16))
    q = torch.tensor(np.concatenate([c, np.zeros(16)]), dtype=F64)
    D = float(oracle.distance("q2b", q, torch.tensor(v, dtype=F64), 0.02))
    assert D == pytest.approx(np.abs(v - c).sum(), rel=1e-14)     # box of width 0 = point, L1


def test_q2b_inside_box_only_in_distance():
    c = np.array([0.0, 1.0]); o = np.array([2.0, 2.0]); v = np.array([0.5, 0.0])
    D = float(oracle.distance("q2b", torch.tensor(np.r_[c, o]), torch.tensor(v), 0.5))
    assert D == pytest.approx(0.5 * (0.5 + 1.0), rel=1e-15)


# ------------------------------------------------------------------ P5 Beta
def test_beta_kl_closed_forms():
    for case in GOLD["beta_kl"]["cases"]:
        a1, b1 = case["entity"]; a2, b2 = case["query"]
        t = lambda x: torch.tensor([x], dtype=F64)
        val = float(beta_kl(t(a1), t(b1), t(a2), t(b2)))
        assert val == pytest.approx(case["kl"], rel=1e-13, abs=1e-14)


def test_beta_kl_quadrature():
    from scipy import integrate, stats
    rng = np.random.default_rng(1)
    for _ in range(5):
        a1, b1, a2, b2 = rng.uniform(0.6, 4.0, size=4)
        p, q = stats.beta(a1, b1), stats.beta(a2, b2)
        ref, _ = integrate.quad(lambda x: p.pdf(x) * (p.logpdf(x) - q.logpdf(x)), 0, 1, limit=200)
        t = lambda x: torch.tensor([x], dtype=F64)
        assert float(beta_kl(t(a1), t(b1), t(a2), t(b2))) == pytest.approx(ref, rel=1e-7)


def test_betae_distance_uses_entity_first_and_activation():
    # Em(v) = clamp(x + 1, 0.05, 1e9) (A8): raw row x = (alpha - 1, beta - 1)
    q = torch.tensor([3.0, 3.0], dtype=F64)           # query Beta(3, 3)
    v = torch.tensor([1.0, 4.0], dtype=F64)           # entity Beta(2, 5)
    assert float(oracle.distance("betae", q, v)) == pytest.approx(43 / 60, rel=1e-13)


# ------------------------------------------------------ single-hop closed forms
def test_single_hop_against_numpy_complex():
    rng = np.random.default_rng(2)
    m = 6
    h = rng.normal(size=m) + 1j * rng.normal(size=m)
    t = rng.normal(size=m) + 1j * rng.normal(size=m)
    th = rng.uniform(-np.pi, np.pi, size=m)
    r = rng.normal(size=m) + 1j * rng.normal(size=m)
    cat = lambda z: torch.tensor(np.r_[z.real, z.imag], dtype=F64)
    # RotatE: ||h o e^{i theta} - t|| as a sum of complex moduli (A3), numpy complex as reference
    P = {"rel_phase": torch.tensor(th[None], dtype=F64)}
    q = oracle.project("rotate", cat(h)[None], torch.tensor([0]), P)
    assert float(oracle.distance("rotate", q[0], cat(t))) == pytest.approx(
        np.abs(h * np.exp(1j * th) - t).sum(), rel=1e-13)
    # ComplEx: -Re(<h o r, conj(t)>) (Table 2)
    P = {"rel": cat(r)[None]}
    q = oracle.project("complex", cat(h)[None], torch.tensor([0]), P)
    assert float(oracle.distance("complex", q[0], cat(t))) == pytest.approx(
        -(h * r * np.conj(t)).real.sum(), rel=1e-13)
    # DistMult: -<h o r, t> with zero imaginary parts == ComplEx
    hr, rr, tr = h.real, r.real, t.real
    z = np.zeros(m)
    qc = oracle.project("complex", torch.tensor(np.r_[hr, z])[None], torch.tensor([0]),
                        {"rel": torch.tensor(np.r_[rr, z])[None]})
    qd = oracle.project("distmult", torch.tensor(hr)[None], torch.tensor([0]), {"rel": torch.tensor(rr)[None]})
    dc = float(oracle.distance("complex", qc[0], torch.tensor(np.r_[tr, z])))
    dd = float(oracle.distance("distmult", qd[0], torch.tensor(tr)))
    assert dc == pytest.approx(dd, rel=1e-14) and dd == pytest.approx(-(hr * rr * tr).sum(), rel=1e-13)
    # TransE ||h + r - t||_2 (Table 2, A2)
    P = {"rel": torch.tensor(rr)[None]}
    q = oracle.project("transe", torch.tensor(hr)[None], torch.tensor([0]), P)
    assert float(oracle.distance("transe", q[0], torch.tensor(tr))) == pytest.approx(
        np.linalg.norm(hr + rr - tr), rel=1e-14)


def test_rotate_quarter_turn():
    # h = 1 + 0i rotated by pi/2 is i: distance to t = i is 0, to t = 0 is 1
    P = {"rel_phase": torch.tensor([[math.pi / 2]], dtype=F64)}
    q = oracle.project("rotate", torch.tensor([[1.0, 0.0]], dtype=F64), torch.tensor([0]), P)[0]
    assert float(oracle.distance("rotate", q, torch.tensor([0.0, 1.0], dtype=F64))) == pytest.approx(0, abs=1e-15)
    assert float(oracle.distance("rotate", q, torch.tensor([0.0, 0.0], dtype=F64))) == pytest.approx(1, rel=1e-15)


# --------------------------------------------------------------- operators
def _rand_cfg(kind, d=8, R=4, hidden=16):
    return kggen.ModelConfig(kind, d, 50, R, hidden=hidden)


@pytest.mark.parametrize("kind", ["q2b", "betae"])
def test_attention_intersection_of_identical_inputs(kind):
    cfg = _rand_cfg(kind)
    P = dense_views(cfg, torch.tensor(kggen.init_dense(cfg, 3), dtype=F64))
    rng = np.random.default_rng(3)
    q = torch.tensor(np.abs(rng.normal(size=(2, 2 * cfg.dim if kind == "q2b" else cfg.dim))) + 0.1, dtype=F64)
    out = oracle.intersect(kind, [q, q, q], P)
    if kind == "betae":
        torch.testing.assert_close(out, q, rtol=1e-14, atol=0)     # equal softmax weights 1/3
    else:
        d = cfg.dim
        torch.testing.assert_close(out[:, :d], q[:, :d], rtol=1e-14, atol=0)
        assert torch.all(out[:, d:] <= q[:, d:])                   # o * sigmoid(.) <= min o


def test_gqe_deepset_identical_inputs_numpy():
    cfg = _rand_cfg("gqe")
    dense = kggen.init_dense(cfg, 4).astype(np.float64)
    offs, _ = kggen.dense_offsets(cfg)
    g = lambda n: dense[offs[n][0]:offs[n][0] + int(np.prod(offs[n][1]))].reshape(offs[n][1])
    x = np.random.default_rng(4).normal(size=cfg.dim)
    ref = g("ds_W2") @ np.maximum(g("ds_W1") @ x + g("ds_b1"), 0) + g("ds_b2")
    P = dense_views(cfg, torch.tensor(dense))
    out = oracle.intersect("gqe", [torch.tensor(x)[None]] * 2, P)[0].numpy()
    np.testing.assert_allclose(out, ref, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("kind", ["gqe", "q2b", "betae"])
def test_intersection_permutation_invariance(kind):
    cfg = _rand_cfg(kind)
    P = dense_views(cfg, torch.tensor(kggen.init_dense(cfg, 5), dtype=F64))
    rng = np.random.default_rng(5)
    w = 2 * cfg.dim if kind == "q2b" else cfg.dim
    xs = [torch.tensor(np.abs(rng.normal(size=(3, w))) + 0.1, dtype=F64) for _ in range(3)]
    a = oracle.intersect(kind, xs, P)
    b = oracle.intersect(kind, [xs[2], xs[0], xs[1]], P)
    torch.testing.assert_close(a, b, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("kind", ["gqe", "q2b", "betae", "transe", "rotate"])
def test_distances_nonnegative(kind):
    cfg = _rand_cfg(kind)
    rng = np.random.default_rng(6)
    w = 2 * cfg.dim if kind == "q2b" else cfg.dim
    q = torch.tensor(rng.normal(size=(20, w)), dtype=F64)
    if kind == "q2b":
        q[:, cfg.dim:] = q[:, cfg.dim:].abs()
    if kind == "betae":
        q = q.abs() + 0.05
    v = torch.tensor(rng.normal(size=(20, cfg.dim)) * 0.3, dtype=F64)
    assert torch.all(oracle.distance(kind, q, v) >= -1e-12)


# ---------------------------------------------------------------- P6 Adam
def test_adam_t1():
    g = GOLD["adam_t1"]
    p, m, v = oracle.adam(np.array(g["p0"]), np.zeros(3), np.zeros(3), np.array(g["g"]),
                          g["lr"], 1, g["beta1"], g["beta2"], g["eps"])
    np.testing.assert_allclose(p, g["p1"], rtol=1e-14, atol=1e-18)


def test_adam_constant_gradient_closed_form():
    # with constant g, m_hat = g and v_hat = g^2 at every t => each step moves -lr g/(|g|+eps)
    g = np.array([0.3, -2.0, 1e-3])
    p, m, v = np.zeros(3), np.zeros(3), np.zeros(3)
    for t in range(1, 6):
        p, m, v = oracle.adam(p, m, v, g, 0.01, t, 0.9, 0.999, 1e-8)
    np.testing.assert_allclose(p, -5 * 0.01 * g / (np.abs(g) + 1e-8), rtol=1e-12)


# --------------------------------------------------------------- P1 dedup
def test_dedup_brute_force():
    ids = np.random.default_rng(7).integers(0, 50, size=300)
    uniq, inv = oracle.dedup(ids)
    assert np.all(np.diff(uniq) > 0) and set(uniq.tolist()) == set(ids.tolist())
    assert np.array_equal(uniq[inv], ids)


# ------------------------------------------------- P7 structural special cases
def _rand_batch(cfg, structure, M=3, K=5, seed=0):
    return kggen.make_batch(cfg, structure, M, K, seed=seed, mask_p=0.8)


@pytest.mark.parametrize("kind", ["gqe", "q2b", "betae"])
def test_2u_identical_branches_equals_1p(kind):
    cfg = _rand_cfg(kind)
    b = _rand_batch(cfg, "2u")
    b["anchors"][:, 1] = b["anchors"][:, 0]
    b["relations"][:, 1] = b["relations"][:, 0]
    b1 = dict(b, structure="1p", anchors=b["anchors"][:, :1].copy(), relations=b["relations"][:, :1].copy())
    r2 = oracle.oracle_step(cfg, oracle.SparseTable(cfg, 1), [b], 0.1, apply=False)
    r1 = oracle.oracle_step(cfg, oracle.SparseTable(cfg, 1), [b1], 0.1, apply=False)
    assert r2.loss == pytest.approx(r1.loss, rel=1e-14)


def test_transe_is_gqe_1p():
    # P:L55 KG completion is the single-relation special case; Table 2 TransE == GQE 1p (A2)
    cg = _rand_cfg("gqe"); ct = _rand_cfg("transe")
    b = _rand_batch(cg, "1p")
    tg = oracle.SparseTable(cg, 2); tt = oracle.SparseTable(ct, 2)
    R, d = cg.n_relations, cg.dim
    tt.dense = tg.dense[:R * d].copy()         # both start with the relation table
    rg = oracle.oracle_step(cg, tg, [b], 0.1, apply=False)
    rt = oracle.oracle_step(ct, tt, [b], 0.1, apply=False)
    assert rg.loss == pytest.approx(rt.loss, rel=1e-14)
    np.testing.assert_allclose(rg.grad_rows, rt.grad_rows, rtol=1e-13, atol=1e-16)


def test_multi_worker_equals_concatenated_batch():
    # 2 workers on halves (same pool) == 1 worker on the concatenation (A18)
    cfg = _rand_cfg("q2b")
    b = _rand_batch(cfg, "2i", M=6, K=7)
    bits = kggen.unpack_mask(b["mask"], 7)
    halves = [dict(b, anchors=b["anchors"][s], relations=b["relations"][s], answers=b["answers"][s],
                   mask=kggen.pack_mask(bits[s]), M=3) for s in (slice(0, 3), slice(3, 6))]
    r1 = oracle.oracle_step(cfg, oracle.SparseTable(cfg, 3), [b], 0.05)
    r2 = oracle.oracle_step(cfg, oracle.SparseTable(cfg, 3), halves, 0.05)
    assert r1.loss == pytest.approx(r2.loss, rel=1e-13)
    np.testing.assert_array_equal(r1.uniq, r2.uniq)
    np.testing.assert_allclose(r1.grad_rows, r2.grad_rows, rtol=1e-12, atol=1e-16)
    np.testing.assert_allclose(r1.grad_dense, r2.grad_dense, rtol=1e-12, atol=1e-16)


def test_untouched_rows_unchanged_and_zero_grad_rows_decay():
    cfg = _rand_cfg("gqe")
    t = oracle.SparseTable(cfg, 4)
    b = _rand_batch(cfg, "1p")
    b["mask"][:] = 0                          # pool rows get zero gradient but are touched (A16)
    r = oracle.oracle_step(cfg, t, [b], 0.1)
    pool_only = sorted(set(b["negatives"].tolist()) - set(b["anchors"].ravel().tolist())
                       - set(b["answers"].tolist()))
    k = [r.uniq.tolist().index(i) for i in pool_only]
    assert np.all(r.grad_rows[k] == 0) and np.all(r.m_new[k] == 0)
    untouched = [i for i in range(cfg.n_entities) if i not in set(r.uniq.tolist())][:5]
    p, m, v = t.get(untouched)
    np.testing.assert_array_equal(p, kggen.init_entity_rows(cfg, 4, untouched))


# ---------------------------------------- -m multi-hop variants (App. B, f4)
def test_m_variants_against_numpy_complex():
    """RotatE-m: h o e^{i theta} (no normalisation); DistMult-m: (h o r) / ||h o r||;
    ComplEx-m: h o r with Re and Im parts each normalised; distances of the base models."""
    rng = np.random.default_rng(3)
    m = 5
    h = rng.normal(size=m) + 1j * rng.normal(size=m)
    t = rng.normal(size=m) + 1j * rng.normal(size=m)
    r1, r2 = (rng.normal(size=m) + 1j * rng.normal(size=m) for _ in range(2))
    th1, th2 = (rng.uniform(-np.pi, np.pi, size=m) for _ in range(2))
    cat = lambda z: np.r_[z.real, z.imag]
    T = lambda x: torch.tensor(np.asarray(x)[None], dtype=F64)
    unit_parts = lambda z: z.real / np.linalg.norm(z.real) + 1j * z.imag / np.linalg.norm(z.imag)
    # 2p of each variant, written with numpy complex arithmetic
    P = {"rel_phase": torch.tensor(np.stack([th1, th2]), dtype=F64)}
    q = oracle.query_disjuncts("2p", "rotate-m", [T(cat(h))], [torch.tensor([0]), torch.tensor([1])], P)[0]
    assert float(oracle.distance("rotate-m", q[0], torch.tensor(cat(t)))) == pytest.approx(
        np.abs(h * np.exp(1j * th1) * np.exp(1j * th2) - t).sum(), rel=1e-12)
    P = {"rel": torch.tensor(np.stack([cat(r1), cat(r2)]), dtype=F64)}
    q = oracle.query_disjuncts("2p", "complex-m", [T(cat(h))], [torch.tensor([0]), torch.tensor([1])], P)[0]
    z = unit_parts(unit_parts(h * r1) * r2)
    assert float(oracle.distance("complex-m", q[0], torch.tensor(cat(t)))) == pytest.approx(
        -(z * np.conj(t)).real.sum(), rel=1e-12)
    hr, a, b, tr = h.real, r1.real, r2.real, t.real
    P = {"rel": torch.tensor(np.stack([a, b]), dtype=F64)}
    q = oracle.query_disjuncts("2p", "distmult-m", [T(hr)], [torch.tensor([0]), torch.tensor([1])], P)[0]
    y = hr * a / np.linalg.norm(hr * a)
    y = y * b / np.linalg.norm(y * b)
    assert float(oracle.distance("distmult-m", q[0], torch.tensor(tr))) == pytest.approx(-(y * tr).sum(), rel=1e-12)


@pytest.mark.parametrize("kind", ["distmult-m", "complex-m", "rotate-m"])
def test_m_variants_unit_norm_and_deepset(kind):
    """Every projection / intersection output of DistMult-m is a unit vector, of ComplEx-m
    has unit Re and Im parts; the intersection is GQE's DeepSet followed
    by that normalisation, checked against numpy."""
    cfg = kggen.ModelConfig(kind, 8, 40, 5)
    tab = oracle.SparseTable(cfg, 2)
    P = dense_views(cfg, torch.tensor(tab.dense, dtype=F64))
    rng = np.random.default_rng(4)
    X = [torch.tensor(rng.normal(size=(3, 8))) for _ in range(2)]
    out = oracle.intersect(kind, X, P).numpy()
    W1, b1, W2, b2 = (P[k].numpy() for k in ("ds_W1", "ds_b1", "ds_W2", "ds_b2"))
    ref = np.mean([np.maximum(x.numpy() @ W1.T + b1, 0) for x in X], axis=0) @ W2.T + b2
    if kind == "distmult-m":
        ref = ref / np.linalg.norm(ref, axis=1, keepdims=True)
    elif kind == "complex-m":
        ref = np.concatenate([ref[:, :4] / np.linalg.norm(ref[:, :4], axis=1, keepdims=True),
                              ref[:, 4:] / np.linalg.norm(ref[:, 4:], axis=1, keepdims=True)], axis=1)
    np.testing.assert_allclose(out, ref, rtol=1e-12)
    q = oracle.project(kind, X[0], torch.tensor([0, 1, 2]), P).numpy()
    if kind == "distmult-m":
        np.testing.assert_allclose(np.linalg.norm(q, axis=1), 1.0, rtol=1e-12)
    elif kind == "complex-m":
        np.testing.assert_allclose(np.linalg.norm(q[:, :4], axis=1), 1.0, rtol=1e-12)
        np.testing.assert_allclose(np.linalg.norm(q[:, 4:], axis=1), 1.0, rtol=1e-12)


# ------------------------------------------------------- P9 finite differences
CASES = [(k, s) for k in ("gqe", "q2b", "betae") for s in kggen.STRUCTURES] + \
        [(k, "1p") for k in ("transe", "rotate", "distmult", "complex")] + \
        [(k, s) for k in ("rotate-m", "distmult-m", "complex-m") for s in kggen.STRUCTURES]


@pytest.mark.parametrize("kind,structure", CASES)
def test_finite_differences(kind, structure):
    cfg = kggen.ModelConfig(kind, 4, 12, 3, hidden=8, gamma=3.0)
    b = kggen.make_batch(cfg, structure, 2, 3, seed=11, mask_p=0.9)
    tab = oracle.SparseTable(cfg, 9)
    r = oracle.oracle_step(cfg, tab, [b], 0.1, apply=False)

    def loss_at(rows, dense):
        t2 = oracle.SparseTable(cfg, 9, dense=dense)
        t2.set(r.uniq, rows, np.zeros_like(rows), np.zeros_like(rows))
        # evaluate in fp64 without the fp32 storage round-trip
        X = torch.tensor(rows, dtype=F64)
        th = torch.tensor(dense, dtype=F64)
        P = dense_views(cfg, th)
        inv = oracle.dedup(np.concatenate([b["anchors"].ravel(), b["answers"], b["negatives"]]))[1]
        M, na = b["anchors"].shape
        slot = {"anchors": inv[:M * na].reshape(M, na), "answers": inv[M * na:M * na + M],
                "negatives": inv[M * na + M:]}
        with torch.no_grad():
            l, _, _ = oracle.query_loss_terms(cfg, structure, P, X, slot, b["relations"],
                                              kggen.unpack_mask(b["mask"], b["K"]), 0, M, M, 1)
        return float(l)

    rows0 = tab.get(r.uniq)[0].astype(np.float64)
    dense0 = tab.dense.astype(np.float64)
    rng = np.random.default_rng(0)
    h = 1e-6
    checked = 0
    for _ in range(24):
        if rng.random() < 0.5:
            i, j = rng.integers(0, rows0.shape[0]), rng.integers(0, rows0.shape[1])
            rp, rm = rows0.copy(), rows0.copy(); rp[i, j] += h; rm[i, j] -= h
            fd = (loss_at(rp, dense0) - loss_at(rm, dense0)) / (2 * h)
            an = r.grad_rows[i, j]
        else:
            k = rng.integers(0, dense0.size)
            dp, dm = dense0.copy(), dense0.copy(); dp[k] += h; dm[k] -= h
            fd = (loss_at(rows0, dp) - loss_at(rows0, dm)) / (2 * h)
            an = r.grad_dense[k]
        scale = max(np.abs(r.grad_rows).max(), np.abs(r.grad_dense).max())
        assert abs(fd - an) <= 1e-6 * abs(an) + 1e-7 * scale, (fd, an)
        checked += 1
    assert checked == 24


# ------------------------------------------------- negation
def test_negation_closed_forms():
    # Table 1 P:L143 N(q) = 1/Em(q): (alpha, beta) = (2, 4) -> (0.5, 0.25); N(N(q)) = q
    q = torch.tensor([[2.0, 4.0]], dtype=F64)
    torch.testing.assert_close(oracle.negate("betae", q), torch.tensor([[0.5, 0.25]], dtype=F64))
    r = torch.tensor(np.random.default_rng(8).uniform(0.05, 5, size=(3, 6)), dtype=F64)
    torch.testing.assert_close(oracle.negate("betae", oracle.negate("betae", r)), r, rtol=1e-15, atol=0)
    for kind in ("gqe", "q2b"):
        with pytest.raises(ValueError):
            oracle.negate(kind, q)


def test_negated_beta_kl_closed_form():
    # KL(B(2,5) || N(B(1/3, 1/3))) = KL(B(2,5) || B(3,3)) = 43/60
    q = oracle.negate("betae", torch.tensor([1 / 3, 1 / 3], dtype=F64))
    v = torch.tensor([1.0, 4.0], dtype=F64)        # raw row of Beta(2, 5) (A8)
    assert float(oracle.distance("betae", q, v)) == pytest.approx(43 / 60, rel=1e-13)


def test_2in_with_identical_inputs_negates_one_branch():
    # with identical attention logits the 2in output is the mean of q and 1/q (A5)
    cfg = kggen.ModelConfig("betae", 4, 12, 3, hidden=8)
    dense = kggen.init_dense(cfg, 1).astype(np.float64)
    offs, _ = kggen.dense_offsets(cfg)
    o, shape = offs["att_U2"]
    dense[o:o + int(np.prod(shape))] = 0.0           # U2 = 0 -> equal logits whatever the input
    o, shape = offs["att_c2"]
    dense[o:o + int(np.prod(shape))] = 0.0
    P = dense_views(cfg, torch.tensor(dense))
    q = torch.tensor([[0.5, 2.0, 1.5, 0.25]], dtype=F64)
    out = oracle.intersect("betae", [q, oracle.negate("betae", q)], P)
    torch.testing.assert_close(out, (q + 1.0 / q) / 2, rtol=1e-14, atol=0)


@pytest.mark.parametrize("structure", kggen.NEG_STRUCTURES)
def test_finite_differences_negation(structure):
    test_finite_differences("betae", structure)
