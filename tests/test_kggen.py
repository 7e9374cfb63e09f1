"""Input generators: determinism, ranges, mask format (-m "not gpu")."""
import numpy as np
import pytest

import kggen


def test_counter_uniform_pure_function_and_range():
    a = kggen.counter_uniform(7, 3, np.arange(10000), -0.5, 0.25)
    b = kggen.counter_uniform(7, 3, np.arange(10000), -0.5, 0.25)
    assert a.dtype == np.float32 and np.array_equal(a, b)
    assert a.min() >= -0.5 and a.max() < 0.25
    assert abs(a.mean() - (-0.125)) < 0.01
    c = kggen.counter_uniform(8, 3, np.arange(10000), -0.5, 0.25)
    assert not np.array_equal(a, c)
    # any subset of indices gives the same values (counter-based)
    idx = np.array([5, 9999, 17])
    assert np.array_equal(kggen.counter_uniform(7, 3, idx, -0.5, 0.25), a[idx])


def test_entity_rows_are_pure_function_of_id():
    cfg = kggen.ModelConfig("q2b", 16, 100, 5)
    r = kggen.init_entity_rows(cfg, 1, [3, 50, 3])
    assert np.array_equal(r[0], r[2])
    assert np.all(np.abs(r) <= cfg.rho)


@pytest.mark.parametrize("kind", kggen.MODELS)
def test_dense_layout_sizes(kind):
    cfg = kggen.ModelConfig(kind, 16, 100, 7, hidden=24)
    offs, total = kggen.dense_offsets(cfg)
    assert total == kggen.init_dense(cfg, 0).size
    for name, (o, shape) in offs.items():
        assert o % 4 == 0


def test_mask_roundtrip():
    rng = np.random.default_rng(0)
    for K in (1, 31, 32, 33, 100):
        bits = rng.random((5, K)) < 0.5
        words = kggen.pack_mask(bits)
        assert words.shape == (5, (K + 31) // 32)
        assert np.array_equal(kggen.unpack_mask(words, K), bits)


@pytest.mark.parametrize("structure", kggen.ALL_STRUCTURES)
def test_make_batch_shapes(structure):
    cfg = kggen.ModelConfig("betae", 8, 1000, 10)
    b = kggen.make_batch(cfg, structure, 40, 70, seed=3, step=2)
    assert b["anchors"].shape == (40, kggen.N_ANCHORS[structure])
    assert b["relations"].shape == (40, kggen.N_RELS[structure])
    assert b["anchors"].min() >= 0 and b["anchors"].max() < 1000
    assert b["relations"].max() < 10
    bits = kggen.unpack_mask(b["mask"], 70)
    # the positive is never marked as a negative (A20)
    assert not np.any(bits & (b["negatives"][None, :] == b["answers"][:, None]))
    b2 = kggen.make_batch(cfg, structure, 40, 70, seed=3, step=2)
    assert all(np.array_equal(b[k], b2[k]) for k in ("anchors", "relations", "answers", "negatives", "mask"))
