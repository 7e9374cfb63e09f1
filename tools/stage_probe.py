"""Per-structure step time (graph replay, CUDA events) and stage breakdown (stage events in the
captured graph) of one workload: python tools/stage_probe.py WORKLOAD [STRUCTURE ...]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import kggen  # noqa: E402
from paper_2110_14890_b200 import KGModel  # noqa: E402

wl = sys.argv[1]
w = kggen.WORKLOADS[wl]
structs = sys.argv[2:] or w.structures
cfg = w.model_config()
if wl.startswith("C5"):
    cfg.n_entities = kggen.shard_rows(w.n_entities, 8)
gm = KGModel(cfg, w.M, w.K)
gm.init_params(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
names = ["ingest+dedup", "dag_forward", "scoring_forward", "scoring_backward", "dag_backward", "sparse_adam",
         "dense_adam", "total", "dense_late", "dense_early"]
out = {}
for st in structs:
    bs = [gm.device_batch(kggen.make_batch(cfg, st, w.M, w.K, seed=0, step=s)) for s in range(4)]
    gm.set_apply(True)
    for b in bs:
        gm.step(b, 1e-4, sync=False, on_device=True)
    gm.sync()
    ts = []
    for r in range(40):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gm.step(bs[r % 4], 1e-4, sync=False, on_device=True)
        e1.record()
        ts.append((e0, e1))
    gm.sync()
    torch.cuda.synchronize()
    step_ms = float(np.median([a.elapsed_time(b) for a, b in ts]))
    gm.set_apply(True, stage_timing=True)
    acc = np.zeros(10)
    for r in range(12):
        flush.zero_()
        inf = gm.step(bs[r % 4], 1e-4, sync=True, on_device=True)
        if r >= 2:
            acc += np.array(inf.stage_ms[:10])
    acc /= 10
    out[st] = {"step_ms": round(step_ms, 4), "kernels": inf.kernels,
               **{n: round(float(v), 4) for n, v in zip(names, acc)}}
    print(st, json.dumps(out[st]), flush=True)
gm.close()
