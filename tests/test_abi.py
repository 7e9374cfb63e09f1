"""C-ABI contract checks that need no GPU (-m "not gpu").

* libkg.so loads and exports every function include/kg.h declares;
* the ctypes mirrors of the structs have the C layout (checked against a
  gcc-compiled probe of include/kg.h);
* kg_create rejects invalid configurations before touching the device.
"""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kg.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(kg_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    import paper_2110_14890_b200 as kgb
    lib = C.CDLL(kgb.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(kgb.EXPORTED) == declared


def test_struct_layouts_match_c():
    import paper_2110_14890_b200 as kgb
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "kg.h"
#define O(T, f) printf(#T "." #f " %zu\n", offsetof(T, f))
int main(void) {
  printf("kg_config %zu\nkg_tables %zu\nkg_batch %zu\nkg_step_info %zu\n", sizeof(kg_config),
         sizeof(kg_tables), sizeof(kg_batch), sizeof(kg_step_info));
  O(kg_config, n_entities); O(kg_config, gamma); O(kg_config, max_M); O(kg_config, nccl_id);
  O(kg_config, score_precision);
  O(kg_batch, anchors); O(kg_batch, mask); O(kg_batch, on_device); O(kg_step_info, step);
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "p")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split("\n")
    got = dict(l.split() for l in out if l.strip())
    assert int(got["kg_config"]) == C.sizeof(kgb.kg_config)
    assert int(got["kg_tables"]) == C.sizeof(kgb.kg_tables)
    assert int(got["kg_batch"]) == C.sizeof(kgb.kg_batch)
    assert int(got["kg_step_info"]) == C.sizeof(kgb.kg_step_info)
    for key, v in got.items():
        if "." in key:
            t, f = key.split(".")
            assert getattr(getattr(kgb, t), f).offset == int(v), key


@pytest.mark.parametrize("field,value", [("dim", 12), ("dim", 0), ("n_entities", 0), ("n_relations", 0),
                                         ("max_M", 0), ("world", 0), ("kind", 10), ("kind", -1), ("beta1", 1.0),
                                         ("eps", 0.0), ("score_precision", 2), ("score_precision", -1)])
def test_create_rejects_bad_config(field, value):
    import kggen
    import paper_2110_14890_b200 as kgb
    cfg = kggen.ModelConfig("q2b", 16, 100, 5)
    conf = kgb.make_config(cfg, 8, 8, 8)
    setattr(conf, field, value)
    h = C.c_void_p()
    assert kgb.kg_create(C.byref(conf), C.byref(h)) == kgb.kg.KG_EINVAL
    assert not h.value


def test_create_rejects_odd_hidden_for_betae():
    import kggen
    import paper_2110_14890_b200 as kgb
    cfg = kggen.ModelConfig("betae", 16, 100, 5, hidden=12)
    h = C.c_void_p()
    assert kgb.kg_create(C.byref(kgb.make_config(cfg, 8, 8)), C.byref(h)) == kgb.kg.KG_EINVAL


@pytest.mark.parametrize("kind,status", [("q2b", "KG_EUNSUPPORTED"), ("betae", "KG_EUNSUPPORTED"),
                                         ("rotate", "KG_EUNSUPPORTED"), ("gqe", "KG_EUNSUPPORTED")])
def test_bf16_scoring_only_for_dot_product_scorers(kind, status):
    """the bf16 score mode on a non-dot-product scorer is EUNSUPPORTED (checked
    before the device is touched)."""
    import kggen
    import paper_2110_14890_b200 as kgb
    cfg = kggen.ModelConfig(kind, 16, 100, 5, hidden=16)
    h = C.c_void_p()
    conf = kgb.make_config(cfg, 8, 8, score_precision="bf16")
    assert kgb.kg_create(C.byref(conf), C.byref(h)) == getattr(kgb.kg, status)
    assert not h.value


def test_sampler_library_exports_every_declared_symbol():
    from paper_2110_14890_b200 import sampler as kgs
    txt = open(os.path.join(ROOT, "include", "kg_sample.h")).read()
    declared = sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(kgs_\w+)\s*\(", txt, re.M)))
    assert len(declared) >= 10
    lib = C.CDLL(kgs.SAMPLER_LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(kgs.SAMPLER_EXPORTED) == declared
