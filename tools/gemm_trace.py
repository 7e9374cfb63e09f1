"""Per-k-block pipeline timeline of the tcgen05 GEMM (CTA 0): k_gemm.cu built with -DKG_GEMM_TRACE.
    python tools/gemm_trace.py M N K ta tb [force]"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "tools", "libgemm_trace.so")
SRC = os.path.join(ROOT, "paper_2110_14890_b200", "csrc", "k_gemm.cu")
SRC2 = os.path.join(ROOT, "paper_2110_14890_b200", "csrc", "k_dag.cu")   # launch_relu_mask
WRAP = os.path.join(ROOT, "tools", "gemm_trace.cu")
if not os.path.exists(SO) or os.path.getmtime(SO) < max(os.path.getmtime(SRC), os.path.getmtime(WRAP)):
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-DKG_GEMM_TRACE", "-Xcompiler", "-fPIC", "-shared", "-lcuda", "-I", os.path.join(ROOT, "include"),
                    WRAP, SRC, SRC2, "-o", SO], check=True)
lib = C.CDLL(SO)
M, N, K, ta, tb = (int(x) for x in sys.argv[1:6])
force = int(sys.argv[6]) if len(sys.argv) > 6 else 0
A = torch.randn((K, M) if ta else (M, K), device="cuda")
B = torch.randn((K, N) if tb else (N, K), device="cuda")
Cm = torch.empty((M, N), device="cuda")
P = torch.empty(8 * M * N, device="cuda")
st = torch.cuda.current_stream()
for _ in range(3):
    assert lib.trace_gemm(ta, tb, M, N, K, C.c_void_p(A.data_ptr()), A.shape[1], C.c_void_p(B.data_ptr()), B.shape[1],
                          C.c_void_p(Cm.data_ptr()), N, C.c_void_p(P.data_ptr()), P.numel(), force,
                          C.c_void_p(st.cuda_stream)) == 1
torch.cuda.synchronize()
tr = np.zeros((8, 512), dtype=np.uint64)
lib.gemm_trace_get(C.c_void_p(tr.ctypes.data))
t = tr.astype(np.int64)
t0 = t[0, 0]
n = int((t[0] > 0).sum())
print("k-block  produce  split_saw_full  split_done  mma_saw_conv  mma_issued  lastwarp_done | chunk: drain_begin drain_end"
      "   (SM cycles from the first load issue)")
for kb in range(n):
    extra = f" | {t[6, kb] - t0:8d} {t[7, kb] - t0:8d}" if t[6, kb] > 0 else " |"
    extra += f" || group {kb}: mma start {t[7, 256 + kb] - t0:8d} committed {t[6, 256 + kb] - t0:8d}" if t[7, 256 + kb] > 0 else ""
    print(f"{kb:4d} " + " ".join(f"{(t[r, kb] - t0):10d}" for r in (0, 1, 2, 3, 4, 5)) + extra)
