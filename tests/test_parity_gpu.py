"""GPU parity: the CUDA path through the C-ABI vs the fp64 oracle (-m gpu).

Tolerance (BASELINE.json north_star): indices and touched-row sets bit-exact;
losses, gradients and updated rows within rtol = 1e-5 (fp32), measured per
tensor as |x - ref| <= rtol*|ref| + rtol*max|ref|.  Parity is checked in the
three stages of SURVEY §8(c): (i) gradients vs oracle gradients, (ii) Adam as
a pure function of the GPU's own gradient (1e-6), (iii) end-to-end rows, where
elements with |g_ref| < 1e-4 max|g_ref| are excluded (Adam's first step is
~ -lr*sign(g), reading H9) and counted.

Sizes span several CUDA tiles with ragged tails: M = 70 (tiles of 64/32
rows), K = 100 (tiles of 64/32), d = 40 (chunks of 16/32 units, m = 20).
"""
import numpy as np
import pytest

import kggen
import oracle

pytestmark = pytest.mark.gpu
RTOL = 1e-5


def assert_close(x, ref, rtol=RTOL, what="", mask=None):
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    assert x.shape == ref.shape, (what, x.shape, ref.shape)
    if ref.size == 0:
        return 0
    err = np.abs(x - ref)
    tol = rtol * np.abs(ref) + rtol * np.abs(ref).max()
    bad = err > tol
    if mask is not None:
        bad &= mask
    if bad.any():
        k = np.unravel_index(np.argmax(np.where(bad, err / np.maximum(tol, 1e-300), 0)), err.shape)
        raise AssertionError(f"{what}: {bad.sum()}/{bad.size} out of tolerance; worst at {k}: "
                             f"got {x[k]!r} ref {ref[k]!r} (max|ref| {np.abs(ref).max():.3g})")
    return int((~mask).sum()) if mask is not None else 0


def _model(cfg, max_M, max_K, max_cand=0, seed=5):
    from paper_2110_14890_b200 import KGModel
    m = KGModel(cfg, max_M, max_K, max_cand)
    m.init_params(seed)
    m.set_apply(True, keep_grads=True)
    return m


def _check_step(gm, table, cfg, batch, lr, step_no=1):
    M, K = batch["M"], batch["K"]
    ref = oracle.oracle_step(cfg, table, [batch], lr, apply=False)
    # the GPU's own state before the step, for the pure-function Adam check (ii)
    p0, m0, v0 = (gm.read_rows(ref.uniq, w) for w in range(3))
    d0, dm0, dv0 = (gm.read_dense(w) for w in range(3))
    info = gm.step(gm.host_batch(batch), lr)
    assert info.step == step_no
    g = gm.last_grads(cap=4 * M + M + K + 8, M=M, K=K)
    # (i) forward values, touched set, gradients
    assert abs(info.loss - ref.loss) <= RTOL * abs(ref.loss) + 1e-12, (info.loss, ref.loss)
    assert_close(g["d_pos"], ref.d_pos[0], what="D+")
    if K:
        assert_close(g["d_neg"], ref.d_neg[0], what="D")
    np.testing.assert_array_equal(g["uniq"], ref.uniq)
    assert info.n_touched == len(ref.uniq)
    assert_close(g["grad_rows"], ref.grad_rows, what="dL/dtheta_E rows")
    assert_close(g["grad_dense"], ref.grad_dense, what="dL/dtheta_D")
    # (ii) Adam as a pure function of the GPU's gradient
    t = step_no
    rows_gpu = gm.read_rows(ref.uniq)
    pa, ma, va = oracle.adam(p0, m0, v0, g["grad_rows"].astype(np.float64), lr, t, cfg.beta1, cfg.beta2, cfg.eps)
    assert_close(rows_gpu, pa, rtol=1e-6, what="sparse Adam(p | g_gpu)")
    assert_close(gm.read_rows(ref.uniq, 1), ma, rtol=1e-6, what="sparse Adam(m | g_gpu)")
    assert_close(gm.read_rows(ref.uniq, 2), va, rtol=1e-6, what="sparse Adam(v | g_gpu)")
    dense_gpu = gm.read_dense(0)
    pd, md, vd = oracle.adam(d0, dm0, dv0, g["grad_dense"].astype(np.float64), lr, t, cfg.beta1, cfg.beta2, cfg.eps)
    assert_close(dense_gpu, pd, rtol=1e-6, what="dense Adam(p | g_gpu)")
    # (iii) end-to-end updated rows against the oracle's own update
    ref2 = oracle.oracle_step(cfg, table, [batch], lr, apply=True)
    # the update direction m_hat/sqrt(v_hat) is ill-conditioned where the first moment is
    # ~0 relative to its tensor (at t = 1: ~ -lr*sign(g), H9): those elements are excluded
    keep = np.abs(ref2.m_new) >= 1e-4 * np.abs(ref2.m_new).max()
    assert_close(rows_gpu, ref2.rows_new, what="theta_E rows after step", mask=keep)
    keepd = np.abs(ref2.dense_m_new) >= 1e-4 * np.abs(ref2.dense_m_new).max()
    assert_close(dense_gpu, ref2.dense_new, what="theta_D after step", mask=keepd)
    return info


# multi-hop models x 9 structures, single-hop 1p, BetaE negation (f1), the -m variants (f4)
CASES = [(k, s) for k in ("gqe", "q2b", "betae") for s in kggen.STRUCTURES] + \
        [(k, "1p") for k in ("transe", "rotate", "distmult", "complex")] + \
        [("betae", s) for s in kggen.NEG_STRUCTURES] + \
        [(k, s) for k in ("rotate-m", "distmult-m", "complex-m") for s in kggen.STRUCTURES]


@pytest.mark.parametrize("kind,structure", CASES)
def test_step_parity(kind, structure):
    cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
    gm = _model(cfg, 70, 100)
    table = oracle.SparseTable(cfg, 5)
    b = kggen.make_batch(cfg, structure, 70, 100, seed=1, step=0, mask_p=0.9)
    # step 1 with a tiny lr: elements whose first update is sign-amplified (H9) then differ by
    # at most 2*lr from the oracle, so step 2 starts from parameters equal within tolerance
    _check_step(gm, table, cfg, b, lr=1e-6, step_no=1)
    # a second step on another batch (t = 2, non-zero moments)
    b2 = kggen.make_batch(cfg, structure, 70, 100, seed=1, step=1, mask_p=0.9)
    _check_step(gm, table, cfg, b2, lr=0.01, step_no=2)
    gm.close()


def test_init_matches_generator_bit_exact():
    for kind in ("q2b", "betae", "rotate", "complex-m"):
        cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
        gm = _model(cfg, 8, 8, seed=11)
        ids = np.array([0, 1, 17, 299])
        np.testing.assert_array_equal(gm.read_rows(ids), kggen.init_entity_rows(cfg, 11, ids))
        np.testing.assert_array_equal(gm.read_dense(), kggen.init_dense(cfg, 11))
        assert not gm.read_rows(ids, 1).any() and not gm.read_dense(2).any()
        gm.close()


@pytest.mark.parametrize("kind,structure", [("gqe", "ip"), ("q2b", "up"), ("betae", "pi"), ("rotate", "1p"),
                                            ("complex", "1p"), ("q2b", "3i"), ("betae", "pni"),
                                            ("betae", "3in"), ("rotate-m", "ip"), ("distmult-m", "up"),
                                            ("complex-m", "pi")])
def test_score_parity(kind, structure):
    cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
    gm = _model(cfg, 70, 100, max_cand=90)
    table = oracle.SparseTable(cfg, 5)
    b = kggen.make_batch(cfg, structure, 70, 100, seed=3)
    cand = np.random.default_rng(0).integers(0, 300, size=90)
    assert_close(gm.score(gm.host_batch(b), cand), oracle.oracle_score(cfg, table, b, cand), what="kg_score")
    gm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("kind,structure", [("gqe", "2i"), ("q2b", "up"), ("q2b", "pi"), ("betae", "ip"),
                                            ("betae", "pin"), ("rotate", "1p"), ("distmult", "1p"),
                                            ("complex", "1p"), ("transe", "1p"), ("complex-m", "2u")])
def test_score_each_parity(kind, structure):
    """kg_score_each (per-query candidates, SURVEY §8(b) shared = 0) against the oracle, with
    duplicate ids inside a row and n_cand not a multiple of the warp count."""
    cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
    gm = _model(cfg, 70, 100, max_cand=90)
    table = oracle.SparseTable(cfg, 5)
    b = kggen.make_batch(cfg, structure, 70, 100, seed=3)
    cand = np.random.default_rng(1).integers(0, 300, size=(70, 37))
    cand[:, 5] = cand[:, 4]
    assert_close(gm.score_each(gm.host_batch(b), cand), oracle.oracle_score_each(cfg, table, b, cand),
                 what="kg_score_each")
    with pytest.raises(Exception):
        bad = cand.copy()
        bad[3, 3] = 300
        gm.score_each(gm.host_batch(b), bad)
    gm.close()


def test_determinism_bitwise():
    cfg = kggen.ModelConfig("q2b", 40, 300, 7)
    outs = []
    for _ in range(2):
        gm = _model(cfg, 70, 100)
        for s, st in enumerate(["2i", "up", "3p"]):
            gm.step(gm.host_batch(kggen.make_batch(cfg, st, 70, 100, seed=2, step=s)), 0.01)
        outs.append((gm.read_rows(np.arange(300)), gm.read_dense()))
        gm.close()
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


def test_device_inputs_equal_host_inputs():
    cfg = kggen.ModelConfig("betae", 40, 300, 7, hidden=24)
    res = []
    for on_dev in (False, True):
        gm = _model(cfg, 70, 100)
        b = kggen.make_batch(cfg, "ip", 70, 100, seed=4)
        info = gm.step(gm.device_batch(b) if on_dev else gm.host_batch(b), 0.01, on_device=on_dev)
        res.append((info.loss, gm.read_rows(np.arange(300)), gm.read_dense()))
        gm.close()
    assert res[0][0] == res[1][0]
    np.testing.assert_array_equal(res[0][1], res[1][1])
    np.testing.assert_array_equal(res[0][2], res[1][2])


def test_async_step_then_sync():
    cfg = kggen.ModelConfig("gqe", 40, 300, 7)
    gm = _model(cfg, 70, 100)
    table = oracle.SparseTable(cfg, 5)
    b = kggen.make_batch(cfg, "2i", 70, 100, seed=6)
    assert gm.step(gm.host_batch(b), 0.01, sync=False) is None
    info = gm.sync()
    ref = oracle.oracle_step(cfg, table, [b], 0.01, apply=False)
    assert abs(info.loss - ref.loss) <= RTOL * abs(ref.loss)
    gm.close()


def test_untouched_rows_bit_identical():
    cfg = kggen.ModelConfig("q2b", 40, 300, 7)
    gm = _model(cfg, 70, 100)
    before = gm.read_rows(np.arange(300))
    b = kggen.make_batch(cfg, "2p", 70, 100, seed=7)
    gm.step(gm.host_batch(b), 0.01)
    after = gm.read_rows(np.arange(300))
    touched = set(np.concatenate([b["anchors"].ravel(), b["answers"], b["negatives"]]).tolist())
    untouched = np.array(sorted(set(range(300)) - touched))
    assert len(untouched) > 0
    np.testing.assert_array_equal(after[untouched], before[untouched])
    assert not np.array_equal(after[sorted(touched)], before[sorted(touched)])
    gm.close()


def test_validation_errors_leave_tables_untouched():
    from paper_2110_14890_b200 import KGError
    cfg = kggen.ModelConfig("rotate", 40, 300, 7)
    gm = _model(cfg, 70, 100)
    before = gm.read_dense()
    b = kggen.make_batch(cfg, "2p", 8, 16, seed=8)
    with pytest.raises(KGError) as e:
        gm.step(gm.host_batch(b), 0.01)                     # single-hop model, multi-hop structure
    assert e.value.status == 2
    b = kggen.make_batch(cfg, "1p", 8, 16, seed=8)
    b["negatives"][3] = 300
    with pytest.raises(KGError) as e:
        gm.step(gm.host_batch(b), 0.01)
    assert e.value.status == 1
    b["negatives"][3] = 0
    b["relations"][0, 0] = 7
    with pytest.raises(KGError) as e:
        gm.step(gm.host_batch(b), 0.01)
    assert e.value.status == 1
    with pytest.raises(KGError):
        gm.step(gm.host_batch(kggen.make_batch(cfg, "1p", 71, 16, seed=8)), 0.01)   # M > max_M
    np.testing.assert_array_equal(gm.read_dense(), before)
    gm.close()


@pytest.mark.parametrize("kind", ["gqe", "q2b"])
def test_negation_structures_need_betae(kind):
    """Table 1 'Negation' column: only BetaE has N(q); other kinds get KG_EUNSUPPORTED."""
    from paper_2110_14890_b200 import KGError
    cfg = kggen.ModelConfig(kind, 40, 300, 7)
    gm = _model(cfg, 70, 100, max_cand=10)
    before = gm.read_dense()
    b = kggen.make_batch(cfg, "2in", 8, 16, seed=8)
    with pytest.raises(KGError) as e:
        gm.step(gm.host_batch(b), 0.01)
    assert e.value.status == 2
    with pytest.raises(KGError) as e:
        gm.score(gm.host_batch(b), np.arange(10))
    assert e.value.status == 2
    np.testing.assert_array_equal(gm.read_dense(), before)
    gm.close()


def test_device_side_validation_of_device_inputs():
    from paper_2110_14890_b200 import KGError
    cfg = kggen.ModelConfig("gqe", 40, 300, 7)
    gm = _model(cfg, 70, 100)
    before = (gm.read_rows(np.arange(300)), gm.read_dense())
    b = kggen.make_batch(cfg, "2i", 20, 30, seed=9)
    b["anchors"][2, 1] = 10_000
    with pytest.raises(KGError) as e:
        gm.step(gm.device_batch(b), 0.01, on_device=True)
    assert e.value.status == 1
    np.testing.assert_array_equal(gm.read_rows(np.arange(300)), before[0])
    np.testing.assert_array_equal(gm.read_dense(), before[1])
    gm.close()


def test_nonfinite_loss_is_transactional():
    from paper_2110_14890_b200 import KGError
    cfg = kggen.ModelConfig("gqe", 40, 300, 7)
    gm = _model(cfg, 70, 100)
    b = kggen.make_batch(cfg, "1p", 10, 20, seed=10)
    bad = gm.read_rows([b["anchors"][0, 0]])
    bad[0, 3] = np.nan
    gm.write_rows([b["anchors"][0, 0]], bad)
    before = (gm.read_rows(np.arange(300)), gm.read_dense())
    with pytest.raises(KGError) as e:
        gm.step(gm.host_batch(b), 0.01)
    assert e.value.status == 6
    np.testing.assert_array_equal(gm.read_rows(np.arange(300)), before[0])
    np.testing.assert_array_equal(gm.read_dense(), before[1])
    gm.close()


@pytest.mark.parametrize("kind", ["q2b", "betae"])
def test_empty_pool_and_empty_mask_rows(kind):
    cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
    gm = _model(cfg, 70, 100)
    table = oracle.SparseTable(cfg, 5)
    b = kggen.make_batch(cfg, "2u", 33, 0, seed=12)          # K = 0: positive term only
    _check_step(gm, table, cfg, b, 0.01, step_no=1)
    b = kggen.make_batch(cfg, "2i", 33, 40, seed=13)
    b["mask"][::2] = 0                                      # half the queries with n_i = 0 (A12)
    _check_step(gm, table, cfg, b, 0.01, step_no=2)
    gm.close()


def test_all_ids_identical():
    cfg = kggen.ModelConfig("betae", 40, 300, 7, hidden=24)
    gm = _model(cfg, 70, 100)
    table = oracle.SparseTable(cfg, 5)
    b = kggen.make_batch(cfg, "3i", 64, 64, seed=14)
    b["anchors"][:] = 5
    b["negatives"][:] = 5
    b["answers"][:] = 6
    b["mask"][:] = 0xFFFFFFFF
    _check_step(gm, table, cfg, b, 0.01, step_no=1)
    gm.close()


def test_graph_replay_equals_direct_launches(monkeypatch):
    """The CUDA-graph replay of kg_step is bitwise identical to launching the kernels directly."""
    cfg = kggen.ModelConfig("q2b", 40, 300, 7)
    res = []
    for no_graph in ("0", "1"):
        monkeypatch.setenv("KG_NO_GRAPH", no_graph)
        gm = _model(cfg, 70, 100)
        for s, st in enumerate(["3i", "up", "2p", "3i"]):       # 3i twice: graph reuse
            gm.step(gm.host_batch(kggen.make_batch(cfg, st, 70, 100, seed=15, step=s)), 0.01)
        res.append((gm.read_rows(np.arange(300)), gm.read_dense(), gm.read_dense(1)))
        gm.close()
    for a, b in zip(*res):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("host_tables", [("ent_v",), ("ent", "ent_m", "ent_v")])
def test_host_tier_equals_device_tables_bitwise(host_tables):
    """theta_E tables in pinned host memory (kg_bind host tier): the same
    kernels run zero-copy over the host link, so every result is bit-identical."""
    from paper_2110_14890_b200 import KGModel
    cfg = kggen.ModelConfig("q2b", 40, 300, 7)
    dev = KGModel(cfg, 70, 100)
    host = KGModel(cfg, 70, 100, host_tables=host_tables)
    assert not host.ent_v.is_cuda and dev.ent_v.is_cuda
    losses = []
    for m in (dev, host):
        m.init_params(5)
        m.set_apply(True)
        out = []
        for s in range(3):
            b = kggen.make_batch(cfg, kggen.STRUCTURES[s * 3], 70, 100, seed=1, step=s)
            out.append(m.step(m.host_batch(b), 0.01).loss)
        losses.append(out)
    assert losses[0] == losses[1]
    ids = np.arange(300)
    for which in (0, 1, 2):
        np.testing.assert_array_equal(dev.read_rows(ids, which), host.read_rows(ids, which))
    np.testing.assert_array_equal(dev.read_dense(), host.read_dense())
    dev.close()
    host.close()


def test_bind_rejects_pageable_host_memory():
    import ctypes as C
    import torch
    from paper_2110_14890_b200 import KGModel, kg
    cfg = kggen.ModelConfig("gqe", 16, 100, 5)
    m = KGModel(cfg, 8, 8)
    pageable = torch.empty((m.rows, 16), dtype=torch.float32)        # not pinned
    t = kg.kg_tables(pageable.data_ptr(), m.ent_m.data_ptr(), m.ent_v.data_ptr(), m.dense.data_ptr(),
                     m.dense_m.data_ptr(), m.dense_v.data_ptr())
    assert kg.kg_bind(m.h, C.byref(t), C.c_void_p(m.stream.cuda_stream)) == kg.KG_EINVAL
    m.close()


def test_stage_timing_with_and_without_graphs(monkeypatch):
    """kg_set_apply bit 2 (stage events) works in graph replay and in eager launches (world > 1
    and KG_NO_GRAPH run eagerly): every stage time is finite and they add up to the step."""
    cfg = kggen.ModelConfig("q2b", 40, 300, 7)
    for no_graph in ("0", "1"):
        monkeypatch.setenv("KG_NO_GRAPH", no_graph)
        gm = _model(cfg, 70, 100)
        gm.set_apply(True, stage_timing=True)
        for s in range(3):
            info = gm.step(gm.host_batch(kggen.make_batch(cfg, "2i", 70, 100, seed=16, step=s)), 0.01)
        st = np.array(info.stage_ms[:10])
        assert np.all(np.isfinite(st)) and np.all(st >= 0) and st[7] > 0, st
        assert abs(st[:7].sum() - st[7]) <= 0.05 * st[7] + 1e-3, st
        gm.close()


def test_checkpoint_resume_is_bitwise(tmp_path):
    """Checkpoint / resume: the tables (caller-owned) and the Adam step counter saved after two
    steps and loaded into a fresh handle continue bit-identically to the uninterrupted run."""
    cfg = kggen.ModelConfig("q2b", 40, 300, 7)
    batches = [kggen.make_batch(cfg, st, 70, 100, seed=17, step=s) for s, st in enumerate(["2i", "up", "3p", "ip"])]
    a = _model(cfg, 70, 100)
    for b in batches[:2]:
        a.step(a.host_batch(b), 0.01)
    a.save(tmp_path / "ck.pt")
    assert a.get_step() == 2
    b_ = _model(cfg, 70, 100, seed=99)          # different init, overwritten by the checkpoint
    b_.load(tmp_path / "ck.pt")
    for b in batches[2:]:
        ia = a.step(a.host_batch(b), 0.01)
        ib = b_.step(b_.host_batch(b), 0.01)
        assert ia.loss == ib.loss and ia.step == ib.step
    np.testing.assert_array_equal(a.read_rows(np.arange(300)), b_.read_rows(np.arange(300)))
    np.testing.assert_array_equal(a.read_dense(2), b_.read_dense(2))
    a.close()
    b_.close()


def test_pipelined_results_in_order():
    """kg_result returns unread step results oldest first (two in flight); the losses equal those
    of synchronous steps, and a third unread step drops the oldest."""
    from paper_2110_14890_b200 import KGError
    cfg = kggen.ModelConfig("gqe", 40, 300, 7)
    bs = [kggen.make_batch(cfg, "2i", 70, 100, seed=18, step=s) for s in range(4)]
    a, b_ = _model(cfg, 70, 100), _model(cfg, 70, 100)
    ref = [a.step(a.host_batch(b), 0.01) for b in bs]
    b_.step(b_.host_batch(bs[0]), 0.01, sync=False)
    b_.step(b_.host_batch(bs[1]), 0.01, sync=False)
    r0 = b_.result()
    b_.step(b_.host_batch(bs[2]), 0.01, sync=False)
    b_.step(b_.host_batch(bs[3]), 0.01, sync=False)     # three unread (1, 2, 3): step 1 dropped
    r2, r3 = b_.result(), b_.result()
    assert (r0.step, r2.step, r3.step) == (1, 3, 4)
    assert (r0.loss, r2.loss, r3.loss) == (ref[0].loss, ref[2].loss, ref[3].loss)
    with pytest.raises(KGError):
        b_.result()
    a.close()
    b_.close()


@pytest.mark.parametrize("kind,structure,dim", [("distmult", "1p", 40), ("complex", "1p", 40),
                                                ("complex", "1p", 200), ("distmult-m", "ip", 400),
                                                ("complex-m", "pi", 200)])
def test_bf16_score_mode(kind, structure, dim):
    """score_precision = bf16 (SURVEY §8(a) a8 opt-in, tolerance 2e-2 of §8(c)): the three
    scoring contractions take bf16-rounded operands; distances, loss and gradients stay within
    2e-2 of the fp64 oracle, and the mode is really active (the distances differ from the fp32
    path's).  No union structures here: the DNF min over disjuncts (A11) is a discrete decision
    that bf16 distances may take differently from the fp64 oracle on near ties (reading A28)."""
    from paper_2110_14890_b200 import KGModel
    cfg = kggen.ModelConfig(kind, dim, 300, 7, hidden=24)
    M, K = 130, 200
    table = oracle.SparseTable(cfg, 5)
    b = kggen.make_batch(cfg, structure, M, K, seed=1, step=0, mask_p=0.9)
    ref = oracle.oracle_step(cfg, table, [b], 1e-3, apply=False)
    out = {}
    for prec in ("bf16", "fp32"):
        gm = KGModel(cfg, M, K, score_precision=prec)
        gm.init_params(5)
        gm.set_apply(True, keep_grads=True)
        info = gm.step(gm.host_batch(b), 1e-3)
        out[prec] = (info, gm.last_grads(cap=4 * M + M + K + 8, M=M, K=K))
        gm.close()
    info, g = out["bf16"]
    assert abs(info.loss - ref.loss) <= 2e-2 * abs(ref.loss), (info.loss, ref.loss)
    assert_close(g["d_neg"], ref.d_neg[0], rtol=2e-2, what="D (bf16)")
    assert_close(g["d_pos"], ref.d_pos[0], what="D+ (fp32 in both modes)")
    np.testing.assert_array_equal(g["uniq"], ref.uniq)
    assert_close(g["grad_rows"], ref.grad_rows, rtol=2e-2, what="dL/dtheta_E rows (bf16)")
    assert_close(g["grad_dense"], ref.grad_dense, rtol=2e-2, what="dL/dtheta_D (bf16)")
    err_bf16 = np.abs(g["d_neg"] - ref.d_neg[0]).max()
    err_fp32 = np.abs(out["fp32"][1]["d_neg"] - ref.d_neg[0]).max()
    assert err_bf16 > 10 * err_fp32, (err_bf16, err_fp32)


def _offsets(cfg):
    off, out = 0, {}
    for name, shape, _, _ in kggen.dense_layout(cfg):
        n = int(np.prod(shape))
        out[name] = (off, shape)
        off += n
    return out


@pytest.mark.parametrize("structure", ["1p", "2i", "2u"])
def test_q2b_exact_kinks_follow_A19(structure):
    """Hand-built exact ties (reading A19; generated data never hits them): query centers equal
    to candidate rows (t = v - c = 0, d|t|/dt = 0), candidates exactly on the box boundary
    (|t| = o: ReLU'(0) = 0, min(|t|, o) -> o), relation offsets exactly 0 and negative
    (ReLU'(0) = 0 in the projection), identical intersection inputs (min ties -> lowest
    index) and identical union branches (DNF min ties -> lowest disjunct).  The GPU's
    gradients equal the oracle's (which applies A19 by construction) within 1e-5."""
    cfg = kggen.ModelConfig("q2b", 16, 50, 3)
    M, K = 6, 8
    b = kggen.make_batch(cfg, structure, M, K, seed=21)
    na = np.asarray(b["anchors"]).reshape(M, -1).shape[1]
    b["anchors"] = np.tile(np.arange(na, dtype=np.int64), (M, 1)) + 1          # anchors 1 .. na, every query
    b["relations"] = np.zeros_like(np.asarray(b["relations"]))                   # relation 0 everywhere
    b["answers"] = np.full(M, 10, np.int64)
    b["negatives"] = np.array([1, 11, 12, 13, 1, 11, 14, 15], np.int64)          # duplicates on purpose
    b["mask"] = np.full_like(np.asarray(b["mask"]), 0xFF)
    d = cfg.dim
    lay = _offsets(cfg)
    dense = kggen.init_dense(cfg, 5)
    oc, _ = lay["rel_center"]
    oo, _ = lay["rel_offset"]
    dense[oc:oc + d] = 0.0                                                       # center shift 0: c = anchor
    roff = np.full(d, 0.25, np.float32)
    roff[:4] = 0.0                                                               # ReLU'(0) = 0
    roff[4:6] = -0.5                                                             # ReLU'(<0) = 0
    dense[oo:oo + d] = roff
    base = np.full(d, 0.5, np.float32)
    rows = {i: base.copy() for i in range(1, na + 1)}                            # identical anchors
    o_box = np.maximum(roff, 0.0)                                                # the 1p offset
    rows[10] = base + o_box                                                      # answer on the boundary
    rows[11] = base.copy()                                                       # t = 0 everywhere
    rows[12] = base - o_box                                                      # other boundary
    rows[13] = base + 2 * o_box + 0.125                                          # outside / ties where o = 0
    rows[14] = base + 0.5 * o_box                                                # inside
    rows[15] = base - 3.0
    ids = np.array(sorted(rows), np.int64)
    R = np.stack([rows[i] for i in ids]).astype(np.float32)
    table = oracle.SparseTable(cfg, 5, dense=dense)
    table.set(ids, R, np.zeros_like(R), np.zeros_like(R))
    gm = _model(cfg, M, K)
    gm.write_dense(dense)
    gm.write_rows(ids, R)
    ref = oracle.oracle_step(cfg, table, [b], 1e-3, apply=False)
    info = gm.step(gm.host_batch(b), 1e-3)
    g = gm.last_grads(cap=4 * M + M + K + 8, M=M, K=K)
    assert abs(info.loss - ref.loss) <= RTOL * abs(ref.loss) + 1e-12, (info.loss, ref.loss)
    np.testing.assert_array_equal(g["uniq"], ref.uniq)
    assert_close(g["d_neg"], ref.d_neg[0], what="D (ties)")
    assert_close(g["grad_rows"], ref.grad_rows, what="dL/dtheta_E rows (ties)")
    assert_close(g["grad_dense"], ref.grad_dense, what="dL/dtheta_D (ties)")
    gm.close()


@pytest.mark.parametrize("kind,structure", [("q2b", "up"), ("betae", "pin"), ("complex", "1p"), ("gqe", "3i")])
def test_minimal_sizes(kind, structure):
    """The degenerate batch sizes: one query against a one-entry pool (every tile a ragged
    tail, split counts of 1)."""
    cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
    gm = _model(cfg, 1, 1)
    table = oracle.SparseTable(cfg, 5)
    b = kggen.make_batch(cfg, structure, 1, 1, seed=2, step=0, mask_p=1.0)
    _check_step(gm, table, cfg, b, lr=1e-6, step_no=1)
    gm.close()
