"""Time the fused sparse-Adam kernel alone on the bench's id streams (tools/sparse_probe.cu).

    python tools/sparse_probe.py [--workload C5-q2b] [--reps 50]

For every structure of the workload: dedup of the step's ids (anchors, answers, pool), a
random occurrence-gradient buffer, then `reps` launches of the kernel, each after a 256 MB
L2 flush (the bench's write flush; --clean-flush adds a read pass so the kernel pays no write-back
of dirty flush lines), timed with CUDA events on the launching stream.  Reports us per launch and the
algorithmic GB/s (24 d bytes per touched row for p, m, v read + write, plus 4 d bytes per
occurrence gradient row read) against MEASURED_PEAKS.json.
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import kggen  # noqa: E402

CSRC = os.path.join(ROOT, "paper_2110_14890_b200", "csrc")
SO = os.path.join(ROOT, "tools", "libsparse_probe.so")


def build(extra=(), so=None):
    so = so or SO
    srcs = [os.path.join(ROOT, "tools", "sparse_probe.cu"), os.path.join(CSRC, "k_adam.cu"),
            os.path.join(CSRC, "k_dedup.cu")]
    if os.path.exists(so) and all(os.path.getmtime(so) >= os.path.getmtime(s) for s in srcs):
        return
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"), *extra,
           *srcs, "-o", so]
    subprocess.run(cmd, check=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5-q2b")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--build-only", action="store_true")
    ap.add_argument("--variant", default="", help="extra nvcc define for a probe variant (e.g. KG_SA_PROBE=1)")
    ap.add_argument("--clean-flush", action="store_true",
                    help="after the 256 MB write flush, read another 256 MB buffer (L2 clean: the kernel pays no "
                         "write-back of the flush)")
    ap.add_argument("--trace", action="store_true", help="with --variant KG_SA_PROBE=3: per-warp globaltimer trace")
    args = ap.parse_args()
    so = SO if not args.variant else SO.replace(".so", "_" + args.variant + ".so")
    build(["-D" + args.variant] if args.variant else (), so)
    if args.build_only:
        return
    import torch
    lib = ctypes.CDLL(so)
    w = kggen.WORKLOADS[args.workload]
    cfg = w.model_config()
    if args.workload.startswith("C5"):
        cfg.n_entities = kggen.shard_rows(w.n_entities, 8)
    d, dev = cfg.dim, torch.device("cuda", 0)
    n = cfg.n_entities
    ent = torch.rand(n, d, device=dev)
    mm = torch.zeros(n, d, device=dev)
    vv = torch.zeros(n, d, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush2 = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
    lr = torch.tensor([1e-4], device=dev)
    bc = torch.tensor([1.0 / (1 - 0.9), 1.0 / (1 - 0.999)], device=dev)
    flags = torch.zeros(2, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = {"workload": args.workload, "d": d, "rows": n, "peak_gbs": peak, "structures": {}}
    tot_bytes = tot_us = 0.0
    for si, s in enumerate(w.structures):
        b = kggen.make_batch(cfg, s, w.M, w.K, seed=0, step=si)
        ids = np.concatenate([b["anchors"].ravel(), b["answers"].ravel(), b["negatives"].ravel()]).astype(np.int64)
        L = len(ids)
        idd = torch.from_numpy(ids).to(dev)
        uniq = torch.empty(L, dtype=torch.int64, device=dev)
        inv, perm, sinv, hrow = (torch.empty(L, dtype=torch.int32, device=dev) for _ in range(4))
        seg = torch.empty(L + 1, dtype=torch.int32, device=dev)
        U = torch.empty(1, dtype=torch.int32, device=dev)
        assert lib.probe_dedup(P(idd), L, int(n).bit_length(), P(uniq), P(inv), P(perm), P(seg), P(U), P(sinv), P(hrow), sp) == 0
        OG = torch.randn(L, d, device=dev) * 1e-3
        PS = torch.empty(L, d, device=dev)
        cnt = torch.zeros(L * 16, dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        Uh = int(U.item())
        res = {}
        for early in (0, 1):
            ts = []
            for r in range(args.reps + 3):
                flush.zero_()
                if args.clean_flush:       # leave L2 holding clean lines: no write-back inside the timing
                    flush2.sum()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                assert lib.probe_sparse(P(uniq), P(seg), P(perm), P(sinv), P(hrow), P(U), L, P(OG), P(PS), P(cnt), d, P(ent),
                                        P(mm), P(vv), P(lr), P(bc), P(flags), early, sp) == 0
                e1.record(st)
                if r >= 3:
                    ts.append((e0, e1))
            torch.cuda.synchronize()
            us = float(np.median([a.elapsed_time(b_) * 1e3 for a, b_ in ts]))
            res["early" if early else "plain"] = us
        assert int(cnt.abs().sum().item()) == 0, "arrival counters not reset"
        if args.trace:
            tr = np.zeros((1 << 16, 4), dtype=np.uint64)
            lib.probe_trace_clear()
            flush.zero_()
            torch.cuda.synchronize()
            lib.probe_sparse(P(uniq), P(seg), P(perm), P(sinv), P(hrow), P(U), L, P(OG), P(PS), P(cnt), d, P(ent),
                             P(mm), P(vv), P(lr), P(bc), P(flags), 0, sp)
            torch.cuda.synchronize()
            lib.probe_trace(ctypes.c_void_p(tr.ctypes.data))
            ns_ = (d // 4 + 31) // 32
            nchunk = (L + 15) // 16 * ns_
            t = tr.astype(np.int64)
            used = t[:, 0] > 0
            t0 = t[used, 0].min()
            for name, sel in (("chunk", np.arange(1 << 16) < nchunk), ("head", np.arange(1 << 16) >= nchunk)):
                m_ = used & sel
                for k in range(4):
                    v_ = t[m_ & (t[:, k] > 0), k] - t0
                    if len(v_):
                        print(f"  {name} t{k}: n={len(v_)} p10={np.percentile(v_, 10):.0f} p50={np.median(v_):.0f} "
                              f"p90={np.percentile(v_, 90):.0f} max={v_.max()} ns")
        nbytes = 24.0 * Uh * d + 4.0 * L * d
        res.update(U=Uh, L=L, mbytes=round(nbytes / 1e6, 2), gbs=round(nbytes / (res["plain"] * 1e-6) / 1e9, 1))
        out["structures"][s] = res
        tot_bytes += nbytes
        tot_us += res["plain"]
        print(s, json.dumps(res), flush=True)
    out["mean_us"] = round(tot_us / len(w.structures), 2)
    out["gbs"] = round(tot_bytes / (tot_us * 1e-6) / 1e9, 1)
    out["frac"] = round(out["gbs"] / peak, 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
