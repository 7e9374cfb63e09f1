"""End-to-end demo: the native sampler feeds kg_step on a split FB15k-237-shaped synthetic KG
(G_train), and kg_eval scores App. E evaluation sets built on G_test / G_valid.

python tools/train_eval.py [model] [steps]   (one GPU; prints loss and filtered MRR / Hits@10)
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import kggen  # noqa: E402
from paper_2110_14890_b200 import KGModel  # noqa: E402
from paper_2110_14890_b200 import sampler as N  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "q2b"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
V, R, E = kggen.KG_SHAPES["FB15k-237"]
kg = kggen.make_kg(V, R, E, seed=0)
tr, va, te = kggen.split_kg(kg, seed=0)
s_tr, s_va, s_te = N.KGSampler(tr), N.KGSampler(va), N.KGSampler(te)
cfg = kggen.ModelConfig(kind, 400, V, R, hidden=800)
structs = ["1p", "2p", "3p", "2i", "3i", "ip", "pi", "2u", "up"] if kind in ("gqe", "q2b", "betae") else ["1p"]
evals = {s: N.build_eval_set(s_te, s_va, s, 256, n_neg=1000, seed=1) for s in (["1p", "2p", "2i"] if len(structs) > 1 else ["1p"])}
M, K = 512, 128
gm = KGModel(cfg, M, K, max_cand=1000)
gm.init_params(0)


def evaluate():
    out = {}
    for s, (b, off, ids, neg) in evals.items():
        hb = dict(b, K=0, answers=np.zeros(b["M"], np.int64), negatives=np.zeros(0, np.int64),
                  mask=np.zeros((b["M"], 1), np.uint32))
        _, met = gm.eval(gm.host_batch(hb), off, ids, neg)
        out[s] = (round(float(met[:, 0].mean()), 4), round(float(met[:, 3].mean()), 4))
    return out


print("eval before training (MRR, Hits@10):", evaluate(), flush=True)
pipe = s_tr.pipeline(structs, M, K, seed=0, n_workers=8)
t0 = time.time()
for step in range(1, steps + 1):
    info = gm.step(pipe.next(), 1e-3, sync=(step % 500 == 0))
    if step % 500 == 0:
        print(f"step {step}: loss {info.loss:.4f}  ({(time.time() - t0):.1f} s)", evaluate(), flush=True)
pipe.close()
