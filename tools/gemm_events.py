"""CUDA-event timing of the tcgen05 GEMM's tile / split-K variants on the DAG's shapes
(one launch chain per call through kg_test_gemm, 200 back-to-back calls, mean per call):
    python tools/gemm_events.py"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_14890_b200 as kgb

# (M, N, K, ta, tb): Q2B / GQE intersection MLP forward (2M, 3M rows), its dX / dW, the offset DeepSet's M rows
shapes = [(1024, 400, 400, 0, 0), (1536, 400, 400, 0, 0), (512, 400, 400, 0, 0), (1024, 400, 400, 0, 1),
          (400, 400, 1024, 1, 1), (400, 400, 1536, 1, 1), (400, 400, 512, 1, 1)]
variants = [(None, "auto"), (1 | (1 << 1), "bn64 nosplit"), (1 | (2 << 1), "bn128 nosplit"), (1 << 1, "bn64 split"),
            (2 << 1, "bn128 split")]
st = torch.cuda.current_stream()
for M, N, K, ta, tb in shapes:
    A = torch.randn((K, M) if ta else (M, K), device="cuda")
    B = torch.randn((K, N) if tb else (N, K), device="cuda")
    Cm = torch.empty((M, N), device="cuda")
    r2 = (A.t() if ta else A).double() @ (B if tb else B.t()).double()
    for force, name in variants:
        fl = 2 if force is None else 2 | (force << 2)

        def call(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert kgb.kg_test_gemm(ta, tb, M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1],
                                    Cm.data_ptr(), N, None, fl | (reps << 8), 0.0, C.c_void_p(st.cuda_stream)) == 0
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1)
        call(1)
        t = min(call(401) - call(1) for _ in range(3)) / 400   # the malloc / sync of one call cancels
        err = float((Cm.double() - r2).abs().max() / r2.abs().max())
        print(f"M={M} N={N} K={K} ta={ta} tb={tb} {name:14s}: {t * 1000:7.2f} us  relerr {err:.1e}", flush=True)
