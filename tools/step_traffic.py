"""DRAM traffic per bench stage, per step, for profiles/ncu_traffic.json (bench.py's
roofline.traffic).

Run under ncu on the GPU box (one GPU, cold caches = ncu's default cache control):

    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --csv --log-file gpurun_out/traffic_<W>.csv python tools/step_traffic.py --workload <W>

The script builds the bench's model and batches for the workload, runs one warm-up step per
structure (graph capture), then profiles exactly one step per structure between
cudaProfilerStart / Stop.  `python tools/step_traffic.py --parse <csv>... ` then sums the
launches' DRAM bytes per stage (kernel-name classes below) and divides by the step count.
"""
import argparse
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

DOT = ("distmult", "complex", "distmult-m", "complex-m")
# kernel-name substrings -> bench stage (first match wins); GEMMs go to "scoring" for the
# single-hop dot-product kinds (their only contractions), else to "dag"
CLASSES = [
    ("ingest+dedup", ("ids_concat", "rel_occ", "dedup_kernel")),
    ("sparse_adam", ("seg_piece", "sparse_adam")),
    ("dense_adam", ("dense_adam", "rel_reduce", "rel_stamp", "scatter_rel")),
    ("scoring", ("pos_kernel", "pair_fwd", "pair_epi", "pair_bwd", "bwd_q_combine", "bwd_v_combine",
                 "loss_finalize", "loss_check", "beta_query", "beta_entity", "gather_rows")),
    ("dag", ("proj_", "gemm_", "transpose", "mean_stack", "q2b_", "colsum", "relu_mask", "gqe_inter",
             "betae_", "beta_att", "neg_", "qnorm_", "bias_act")),
]


def classify(name, kind, single_hop):
    for stage, keys in CLASSES:
        if any(k in name for k in keys):
            if stage == "dag" and "gemm" in name and kind in DOT and single_hop:
                return "scoring"
            return stage
    return None


def run(workload, only=None):
    import torch
    import kggen
    from paper_2110_14890_b200 import KGModel
    w = kggen.WORKLOADS[workload]
    cfg = w.model_config()
    if workload.startswith("C5"):
        cfg.n_entities = min(w.n_entities, kggen.shard_rows(w.n_entities, 8))
    gm = KGModel(cfg, w.M, w.K)
    gm.init_params(0)
    gm.set_apply(True)
    batches = [gm.device_batch(kggen.make_batch(cfg, s, w.M, w.K, seed=0, step=i))
               for i, s in enumerate(w.structures) if not only or s in only]
    for b in batches:                                  # warm-up: one graph per structure
        gm.step(b, 1e-4, sync=False, on_device=True)
    gm.sync()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for b in batches:
        gm.step(b, 1e-4, sync=False, on_device=True)
    gm.sync()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(json.dumps({"workload": workload, "steps": len(batches)}))


def parse(paths, out):
    import kggen
    res = json.load(open(out)) if os.path.exists(out) else {}
    for path in paths:
        workload = os.path.basename(path).split("traffic_")[1].rsplit(".", 1)[0]
        w = kggen.WORKLOADS[workload]
        kind = w.model_config().kind
        single_hop = all(s == "1p" for s in w.structures)
        rows = list(csv.reader(open(path)))
        hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        per = collections.defaultdict(lambda: collections.defaultdict(float))
        names = {}
        for r in rows[hdr + 1:]:
            d = dict(zip(rows[hdr], r))
            if not d.get("Metric Name"):
                continue
            try:
                v = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                continue
            unit = d.get("Metric Unit", "")
            if d["Metric Name"].startswith("dram__bytes"):
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            per[d["ID"]][d["Metric Name"]] += v
            names[d["ID"]] = d["Kernel Name"]
        stage = collections.defaultdict(float)
        unclassified = collections.defaultdict(float)
        for i, m in per.items():
            b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
            s = classify(names[i], kind, single_hop)
            if s is None:
                unclassified[names[i].split("(")[0]] += b
            else:
                stage[s] += b
        n = len(w.structures)
        res[workload] = {s: round(v / n) for s, v in sorted(stage.items())}
        res[workload]["_launches_per_step"] = round(len(per) / n, 2)
        if unclassified:
            res[workload]["_unclassified_bytes_per_step"] = {k: round(v / n) for k, v in unclassified.items()}
    res["_about"] = ("DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per step of each bench stage: "
                     "one step per structure of the workload profiled by ncu (cold caches, serialised; "
                     "tools/step_traffic.py), summed over the stage's kernels and divided by the step count. "
                     "bench.py copies the dominant stage's figure into roofline.traffic.")
    json.dump(res, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(res, indent=1, sort_keys=True))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload")
    ap.add_argument("--structures", default="", help="comma list: profile only these structures")
    ap.add_argument("--parse", nargs="*")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_traffic.json"))
    a = ap.parse_args()
    if a.parse:
        parse(a.parse, a.out)
    else:
        run(a.workload, [x for x in a.structures.split(",") if x])
