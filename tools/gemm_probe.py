"""Time the tensor-core GEMM (kg_test_gemm includes malloc/sync: use ncu for kernel times)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_14890_b200 as kgb

shapes = [(2048, 1600, 1600, 0, 0), (2048, 1600, 800, 0, 0), (512, 1600, 1600, 0, 0), (512, 400, 1600, 0, 0),
          (1600, 1600, 2048, 1, 1), (1024, 400, 400, 0, 0)]
st = torch.cuda.current_stream()
torch.backends.cuda.matmul.allow_tf32 = False
for M, N, K, ta, tb in shapes:
    A = torch.randn((K, M) if ta else (M, K), device="cuda")
    B = torch.randn((K, N) if tb else (N, K), device="cuda")
    Cm = torch.empty((M, N), device="cuda")
    args = (ta, tb, M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], Cm.data_ptr(), N, None, 0, 0.0,
            C.c_void_p(st.cuda_stream))
    for _ in range(2):
        kgb.kg_test_gemm(*args)
        r2 = (A.t() if ta else A) @ (B if tb else B.t())
    torch.cuda.synchronize()
    err = float((Cm - r2).abs().max() / r2.abs().max())
    print(f"M={M} N={N} K={K} ta={ta} tb={tb} relerr vs cublas-fp32 {err:.2e}")
