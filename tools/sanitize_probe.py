"""Small steps of every model kind through kg_step / kg_score / kg_score_each, for compute-sanitizer
(memcheck / racecheck / synccheck):  compute-sanitizer --tool memcheck python tools/sanitize_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ.setdefault("KG_NO_GRAPH", "1")    # launches the kernels directly (the sanitizer sees each)
import kggen  # noqa: E402
from paper_2110_14890_b200 import KGModel  # noqa: E402

cases = [("gqe", "ip"), ("q2b", "up"), ("q2b", "2u"), ("q2b", "3i"), ("betae", "pni"), ("betae", "2i"),
         ("transe", "1p"), ("rotate", "1p"), ("rotate-m", "up"), ("distmult", "1p"), ("complex", "1p"),
         ("complex", "1p", "bf16"), ("distmult-m", "pi")]
for kind, st, *prec in cases:
    cfg = kggen.ModelConfig(kind, 40, 300, 7, hidden=24)
    gm = KGModel(cfg, 70, 100, max_cand=50, score_precision=prec[0] if prec else "fp32")
    gm.init_params(1)
    for s in range(2):
        b = kggen.make_batch(cfg, st, 70, 100, seed=2, step=s)
        gm.step(gm.host_batch(b), 1e-3)
    gm.score(gm.host_batch(b), np.arange(50))
    gm.score_each(gm.host_batch(b), np.random.default_rng(0).integers(0, 300, size=(70, 13)))   # per-query candidates
    gm.close()
    print("ok", kind, st, *prec, flush=True)
