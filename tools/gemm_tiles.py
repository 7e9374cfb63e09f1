"""Tile / split-K choices of the tcgen05 GEMM on the DAG's shapes (run under ncu for kernel times):
    ncu --metrics gpu__time_duration.sum --csv python tools/gemm_tiles.py"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_14890_b200 as kgb

# (M, N, K, ta, tb): the Q2B intersection MLPs (d = 400, 2M / M rows), their backward, BetaE shapes
shapes = [(1024, 400, 400, 0, 0), (512, 400, 400, 0, 0), (1024, 400, 400, 0, 1), (400, 400, 1024, 1, 1),
          (1536, 400, 400, 0, 0), (1536, 1600, 800, 0, 0), (1536, 1600, 1600, 0, 0), (1536, 400, 1600, 0, 0),
          (1600, 800, 1536, 1, 1), (512, 1600, 800, 0, 0)]
variants = [(0, "auto drain"), (-1, "auto nodrain"), (1 | (2 << 1), "bn128 nosplit drain"),
            (-(1 | (2 << 1)) - 2, "bn128 nosplit nodrain")]
if len(sys.argv) > 1 and sys.argv[1] == "all":
    variants += [(1 | (1 << 1), "bn64 nosplit"), (2 << 1, "bn128 split"), (1 << 1, "bn64 split")]
st = torch.cuda.current_stream()


def flags(force):
    """relu-argument bits of kg_test_gemm: bit 1 drained accumulation, bits 2.. the tile force;
    a negative force = the same tile choice undrained (-1: the heuristic, undrained)."""
    if force == -1:
        return 0
    if force < 0:
        return (-(force + 2)) << 2
    return 2 | (force << 2)
for M, N, K, ta, tb in shapes:
    A = torch.randn((K, M) if ta else (M, K), device="cuda")
    B = torch.randn((K, N) if tb else (N, K), device="cuda")
    Cm = torch.empty((M, N), device="cuda")
    r2 = (A.t() if ta else A).double() @ (B if tb else B.t()).double()
    for force, name in variants:
        for _ in range(3):
            assert kgb.kg_test_gemm(ta, tb, M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], Cm.data_ptr(),
                                    N, None, flags(force), 0.0, C.c_void_p(st.cuda_stream)) == 0
        err = float((Cm.double() - r2).abs().max() / r2.abs().max())
        print(f"M={M} N={N} K={K} ta={ta} tb={tb} {name}: relerr {err:.2e}", flush=True)
