"""Precision of the tcgen05 3xTF32 GEMM vs cuBLAS SGEMM: error / (|A| |B|) per element (condition-free)."""
import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2110_14890_b200 as kgb
dev = torch.device("cuda")
torch.backends.cuda.matmul.allow_tf32 = False
def run(ta, tb, M, N, K, kind, drain=0):
    rng = np.random.default_rng(1)
    if kind == "normal":
        A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
        B = rng.standard_normal((K, N) if tb else (N, K)).astype(np.float32)
    else:   # relu activations x mixed-sign small gradients, magnitudes spread over 3 decades
        A = np.maximum(rng.standard_normal((K, M) if ta else (M, K)), 0).astype(np.float32)
        B = (rng.standard_normal((K, N) if tb else (N, K)) * 10 ** rng.uniform(-3, 0, (K, N) if tb else (N, K))).astype(np.float32)
    tA, tB = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
    tC = torch.zeros((M, N), device=dev)
    st = torch.cuda.current_stream()
    s = kgb.kg_test_gemm(int(ta), int(tb), M, N, K, tA.data_ptr(), A.shape[1], tB.data_ptr(), B.shape[1],
                         tC.data_ptr(), N, None, 2 * drain, 0.0, C.c_void_p(st.cuda_stream))
    assert s == 0
    opA = A.T if ta else A
    opB = B if tb else B.T
    ref = opA.astype(np.float64) @ opB.astype(np.float64)
    absr = np.abs(opA).astype(np.float64) @ np.abs(opB).astype(np.float64)
    cub = (torch.from_numpy(np.ascontiguousarray(opA)).to(dev) @ torch.from_numpy(np.ascontiguousarray(opB)).to(dev)).cpu().numpy()
    got = tC.cpu().numpy()
    e_tc = np.abs(got - ref) / np.maximum(absr, 1e-30)
    e_cb = np.abs(cub - ref) / np.maximum(absr, 1e-30)
    print(f"{kind:7s} drain={drain} ta={ta} tb={tb} {M}x{N}x{K}: tc max {e_tc.max():.2e} mean {e_tc.mean():.2e} | cublas max {e_cb.max():.2e} mean {e_cb.mean():.2e}")
for kind in ("normal", "relu"):
    for ta, tb, M, N, K in ((0, 0, 1024, 1600, 800), (0, 0, 1024, 1600, 1600), (0, 1, 1024, 800, 1600), (1, 1, 1600, 800, 1024), (1, 0, 1600, 1600, 1024), (0, 0, 512, 400, 1600)):
        run(ta, tb, M, N, K, kind)
        run(ta, tb, M, N, K, kind, drain=1)
