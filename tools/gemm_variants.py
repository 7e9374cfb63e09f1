"""Tile / split-K variants of the tcgen05 GEMM on the DAG's shapes, for an ncu launch list
(GPU time per kernel; the GEMM and its split-K combine are separate launches):
    ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum,launch__grid_size --csv \\
        --log-file out.csv python tools/gemm_variants.py
    python tools/gemm_variants.py --parse out.csv
Each (shape, variant) runs 3 times; the parse keeps the last run of each."""
import ctypes as C
import sys

H, D = 1600, 400
SHAPES = []
for gm in (512, 1024, 1536):
    SHAPES += [(gm, H, 2 * D, 0, 0), (gm, H, H, 0, 0), (gm, D, H, 0, 0),        # BetaE MLP forward
               (gm, H, D, 0, 0), (gm, 2 * D, H, 0, 0),                       # dX (K-major W^T)
               (D, H, gm, 1, 1), (H, H, gm, 1, 1), (H, 2 * D, gm, 1, 1)]     # dW = dY^T X
for nr in (512, 1024, 1536):
    SHAPES += [(nr, D, D, 0, 0), (D, D, nr, 1, 1)]                            # d x d intersection MLPs
DW = [(D, H, nr, 1, 0) for nr in (512, 1024, 1536)] + [(H, H, nr, 1, 0) for nr in (512, 1024, 1536)] + \
     [(H, 2 * D, nr, 1, 0) for nr in (512, 1024, 1536)]                     # BetaE dW = dY^T X, X^T stored
if "--dw" in sys.argv:
    SHAPES = DW
if "--kmajor" in sys.argv:   # the K-major-B shapes of the BetaE step (forward, dX, dW on X^T)
    SHAPES = [sh for sh in SHAPES if sh[4] == 0 and sh[3] == 0] + DW
VARIANTS = [(None, "auto"), (1 | (1 << 1), "bn64-nosplit"), (1 | (2 << 1), "bn128-nosplit"),
            (1 | (3 << 1), "bn160-nosplit"), (1 << 1, "bn64-split"), (2 << 1, "bn128-split"), (3 << 1, "bn160-split"),
            (8, "bn64-occ2-split"), (8 | 1, "bn64-occ2-nosplit"), (16, "bn96-split"), (16 | 1, "bn96-nosplit")]
if "--small" in sys.argv:   # the d x d shapes only
    SHAPES = [sh for sh in SHAPES if sh[0] <= 1536 and sh[1] <= 400 and sh[2] <= 1536 and min(sh[:3]) == 400]


def run():
    import torch
    sys.path.insert(0, ".")
    import paper_2110_14890_b200 as kgb
    st = torch.cuda.current_stream()
    for M, N, K, ta, tb in SHAPES:
        A = torch.randn((K, M) if ta else (M, K), device="cuda")
        B = torch.randn((K, N) if tb else (N, K), device="cuda")
        Cm = torch.empty((M, N), device="cuda")
        for force, name in VARIANTS:
            fl = 2 if force is None else 2 | (force << 2)
            for _ in range(3):
                assert kgb.kg_test_gemm(ta, tb, M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1],
                                        Cm.data_ptr(), N, None, fl, 0.0, C.c_void_p(st.cuda_stream)) == 0
            r2 = (A.t() if ta else A).double() @ (B if tb else B.t()).double()
            err = float((Cm.double() - r2).abs().max() / r2.abs().max())
            print(f"{M}x{N}x{K} ta{ta} tb{tb} {name} relerr {err:.1e}", flush=True)


def parse(path):
    import csv
    from collections import OrderedDict
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID')
    d = OrderedDict()
    for r in rows[1:]:
        d.setdefault(int(r[ii]), {'name': r[ki]})[r[mi]] = r[vi]
    launches = [(v['name'], float(v['gpu__time_duration.sum']) / 1000) for _, v in sorted(d.items())]
    # group launches into calls: a GEMM kernel starts a call, a combine / mask kernel joins it
    calls = []
    for name, t in launches:
        if 'gemm_tf32x3' in name:
            calls.append([t, 1])
        elif calls and ('gemm_reduce' in name or 'relu_mask' in name):   # the call's combine / mask pass
            calls[-1][0] += t
            calls[-1][1] += 1
    i = 0
    for M, N, K, ta, tb in SHAPES:
        line = []
        for _, vname in VARIANTS:
            t, n = calls[i + 2]            # the last of 3 runs
            i += 3
            line.append(f"{vname} {t:6.2f}/{n}")
        print(f"{M:5d}x{N:5d}x{K:5d} ta{ta}tb{tb}: " + "  ".join(line))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--parse":
        if "--small" in sys.argv:
            pass
        parse(sys.argv[2])
    else:
        run()
