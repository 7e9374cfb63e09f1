"""The evaluation-set construction of App. E on the native sampler: answer sets by
forward traversal (kgs_answers) bit-exact against the oracle's exhaustive traversal, and the
built set's invariants (missing answers = A(G_test) minus A(G_valid), negatives outside
A(G_test)).  Host code only."""
import numpy as np
import pytest

import kggen
from oracle import sampler as S
from paper_2110_14890_b200 import sampler as N


@pytest.mark.parametrize("structure", kggen.ALL_STRUCTURES)
def test_answers_match_exhaustive_traversal(structure):
    kg = kggen.make_kg(48, 3, 260, seed=2, a=0.5)
    smp, okg = N.KGSampler(kg, 2), S.OracleKG(kg)
    root = S.parse(S.STRUCTURE_DSL[structure])
    rng = np.random.default_rng(3)
    a = rng.integers(0, 48, (25, kggen.N_ANCHORS[structure]))
    r = rng.integers(0, 3, (25, kggen.N_RELS[structure])).astype(np.int32)
    off, ids = smp.answers(structure, a, r)
    for i in range(25):
        assert ids[off[i]:off[i + 1]].tolist() == sorted(S.exhaustive_answers(okg, root, a[i], r[i]))


def test_split_partitions_edges():
    kg = kggen.make_kg(500, 5, 4000, seed=1)
    tr, va, te = kggen.split_kg(kg, seed=3)
    key = lambda g: set(zip(g["h"].tolist(), g["r"].tolist(), g["t"].tolist()))
    assert key(tr) < key(va) < key(te) and key(te) == key(kg)
    assert 0.8 < len(tr["h"]) / len(kg["h"]) < 0.93


@pytest.mark.parametrize("structure", ["1p", "2p", "ip", "2u", "pin"])
def test_eval_set_invariants(structure):
    kg = kggen.make_kg(300, 4, 3000, seed=5, a=0.6)
    tr, va, te = kggen.split_kg(kg, valid_frac=0.1, test_frac=0.1, seed=1)
    smp_v, smp_t = N.KGSampler(va, 2), N.KGSampler(te, 2)
    ov, ot = S.OracleKG(va), S.OracleKG(te)
    root = S.parse(S.STRUCTURE_DSL[structure])
    b, off, ids, neg = N.build_eval_set(smp_t, smp_v, structure, 12, n_neg=40, seed=7)
    assert neg.shape == (12, 40) and off[-1] == len(ids)
    for i in range(12):
        At = S.exhaustive_answers(ot, root, b["anchors"][i], b["relations"][i])
        Av = S.exhaustive_answers(ov, root, b["anchors"][i], b["relations"][i])
        assert ids[off[i]:off[i + 1]].tolist() == sorted(At - Av) and off[i + 1] > off[i]
        assert not (set(neg[i].tolist()) & At)
