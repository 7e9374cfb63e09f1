"""Run a few training steps of one workload / structure (for ncu launch lists).

usage: python tools/step_probe.py WORKLOAD STRUCTURE [STEPS]
"""
import sys

import torch

sys.path.insert(0, ".")
import kggen  # noqa: E402
from paper_2110_14890_b200 import KGModel  # noqa: E402

wl, structure = sys.argv[1], sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = kggen.WORKLOADS[wl]
cfg = w.model_config()
if wl.startswith("C5"):
    cfg.n_entities = kggen.shard_rows(w.n_entities, 8)
gm = KGModel(cfg, w.M, w.K)
gm.init_params(0)
gm.set_apply(True)
bs = [gm.device_batch(kggen.make_batch(cfg, structure, w.M, w.K, seed=0, step=s)) for s in range(steps)]
for b in bs:
    gm.step(b, 1e-3, sync=False, on_device=True)
gm.sync()
torch.cuda.synchronize()
print("ok", structure)
