"""Where do the full-size GPU vs oracle differences sit?  python tools/fullsize_diag.py C4 2i"""
import sys
import numpy as np
sys.path.insert(0, ".")
import kggen, oracle
from paper_2110_14890_b200 import KGModel
wl, st = sys.argv[1], sys.argv[2]
w = kggen.WORKLOADS[wl]; cfg = w.model_config()
if wl.startswith("C5"): cfg.n_entities = kggen.shard_rows(w.n_entities, 8)
M, K = w.M, w.K
gm = KGModel(cfg, M, K); gm.init_params(5); gm.set_apply(True, keep_grads=True)
table = oracle.SparseTable(cfg, 5)
b = kggen.make_batch(cfg, st, M, K, seed=3, step=0)
ref = oracle.oracle_step(cfg, table, [b], 1e-3, apply=True)
info = gm.step(gm.host_batch(b), 1e-3)
g = gm.last_grads(cap=4 * M + M + K + 8, M=M, K=K)
na = kggen.N_ANCHORS[st]
role = {}
for x in b["negatives"]: role[int(x)] = "pool"
for x in b["answers"]: role[int(x)] = role.get(int(x), "") + "+ans"
for x in b["anchors"].reshape(-1): role[int(x)] = role.get(int(x), "") + "+anc"
for name, x, r in (("rows", g["grad_rows"], ref.grad_rows), ("dense", g["grad_dense"], ref.grad_dense),
                   ("dneg", g["d_neg"], ref.d_neg[0]), ("dpos", g["d_pos"], ref.d_pos[0])):
    x = np.asarray(x, np.float64); r = np.asarray(r, np.float64)
    err = np.abs(x - r); mx = np.abs(r).max()
    tol = 1e-5 * (np.abs(r) + mx)
    print(name, "max|ref|", mx, "max err", err.max(), "max err/tol", (err / tol).max(), "n bad", int((err > tol).sum()))
    if name == "rows":
        bad = np.argwhere(err > tol)
        rows = np.unique(bad[:, 0])
        from collections import Counter
        print("  bad rows", len(rows), Counter(role.get(int(ref.uniq[i]), "?") for i in rows).most_common(6))
        rel = err.max(axis=1) / np.abs(r).max(axis=1)
        print("  per-row max err / row max|ref|: worst", rel.max(), "median", np.median(rel))
        for i in rows[:5]:
            print("   row", int(ref.uniq[i]), role.get(int(ref.uniq[i])), "row max|ref|", np.abs(r[i]).max(), "row max err", err[i].max())
    if name == "dense":
        offs, _ = kggen.dense_offsets(cfg)
        for seg, (o, shape) in offs.items():
            n = int(np.prod(shape)); e = err[o:o + n]; rr = np.abs(r[o:o + n])
            print(f"  {seg:10s} max|ref| {rr.max():.3e} max err {e.max():.3e} n bad {int((e > tol[o:o+n]).sum())}")
