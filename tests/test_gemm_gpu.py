"""The tcgen05 3xTF32 GEMM of the query-DAG contractions vs fp64 numpy (-m gpu).

The contractions are plain linear algebra (Y = X W^T, dX = dY W, dW = dY^T X),
so the reference is numpy's float64 matmul; the bar is the fp32 parity bar of
the step (1e-5 relative to the tensor, BASELINE north_star).
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(ta, tb, M, N, K, bias=False, relu=False, beta=0.0, seed=0, drain=False, force=0):
    import torch
    import paper_2110_14890_b200 as kgb
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((K, N) if tb else (N, K)).astype(np.float32)
    C0 = rng.standard_normal((M, N)).astype(np.float32)
    b = rng.standard_normal(N).astype(np.float32)
    dev = torch.device("cuda")

    def padded(x):   # leading dimension rounded up to 4 floats; the padding is NaN and must be ignored
        ld = (x.shape[1] + 3) // 4 * 4
        y = np.full((x.shape[0], ld), np.nan, dtype=np.float32)
        y[:, :x.shape[1]] = x
        return y

    Ap, Bp = padded(A), padded(B)
    tA, tB, tC, tb_ = (torch.from_numpy(x).to(dev) for x in (Ap, Bp, C0, b))
    st = torch.cuda.current_stream()
    s = kgb.kg_test_gemm(int(ta), int(tb), M, N, K, tA.data_ptr(), Ap.shape[1], tB.data_ptr(), Bp.shape[1],
                         tC.data_ptr(), N, tb_.data_ptr() if bias else None, int(relu) | (2 if drain else 0) | (force << 2), beta,
                         C.c_void_p(st.cuda_stream))
    assert s == 0
    opA = A.T.astype(np.float64) if ta else A.astype(np.float64)
    opB = B.astype(np.float64) if tb else B.T.astype(np.float64)
    ref = opA @ opB
    if bias:
        ref = ref + b.astype(np.float64)
    if relu:
        ref = np.maximum(ref, 0)
    if beta:
        ref = ref + beta * C0.astype(np.float64)
    got = tC.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref)
    tol = 1e-5 * (np.abs(ref) + np.abs(ref).max())
    assert np.all(err <= tol), (float(err.max()), float(np.abs(ref).max()), np.unravel_index(np.argmax(err / tol), err.shape))
    return float((err / (np.abs(ref).max())).max())


@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("M,N,K", [(70, 40, 40), (128, 128, 32), (200, 136, 100), (512, 400, 800),
                                   (33, 257, 17), (1, 1, 1), (300, 600, 1500)])
def test_gemm_layouts_and_ragged_shapes(ta, tb, M, N, K):
    _run(ta, tb, M, N, K)


def test_gemm_betae_shapes_and_epilogues():
    _run(False, False, 1024, 1600, 800, bias=True, relu=True)     # H1 = ReLU(X W1^T + b1)
    _run(False, True, 1024, 800, 1600)                            # dX = dH1 W1
    _run(True, True, 1600, 800, 1024)                             # dW1 = dH1^T X
    _run(False, False, 300, 400, 400, beta=1.0)                   # dstack += dH U1


def test_gemm_rejects_unaligned_leading_dimension():
    import torch
    import paper_2110_14890_b200 as kgb
    A = torch.zeros((8, 10), device="cuda")
    st = torch.cuda.current_stream()
    s = kgb.kg_test_gemm(0, 0, 8, 8, 10, A.data_ptr(), 10, A.data_ptr(), 10, A.data_ptr(), 8, None, 0, 0.0,
                         C.c_void_p(st.cuda_stream))
    assert s == 1   # lda % 4 != 0 -> KG_EINVAL


@pytest.mark.parametrize("ta,tb,M,N,K", [(False, True, 1536, 1600, 800),    # H1 = X W1^T: 128 x 160 tiles
                                         (True, True, 1600, 1600, 1536),    # dW2 = dH2^T H1 (MN-major both)
                                         (False, False, 1536, 800, 1600),   # dX = dH1 W1
                                         (False, True, 200, 72, 40), (True, False, 70, 130, 33),
                                         (False, True, 1024, 1024, 200),    # S = Q E^T (ComplEx C3): 128 x 64
                                         (True, True, 300, 200, 120),
                                         # 32-deep k-blocks (K-major B): the unsplit 128 x 64 short-K form,
                                         # 128 x 128 with split K, and MN-major A (dW = dY^T X with X^T stored)
                                         (False, False, 1024, 400, 400), (False, False, 512, 1600, 400),
                                         (False, False, 1024, 1600, 1600), (True, False, 400, 1600, 1024),
                                         (True, False, 1600, 800, 512), (True, False, 100, 60, 70)])
def test_gemm_drained_accumulation(ta, tb, M, N, K):
    """The drained form (fp32-accurate, the default; 128 x 128, 128 x 160 or, for few tiles and a
    short K, 128 x 64 tiles)."""
    _run(ta, tb, M, N, K, bias=not ta, relu=not ta, drain=True)


@pytest.mark.gpu
@pytest.mark.parametrize("ta,M,N,K", [(False, 512, 1600, 1600), (False, 200, 100, 70), (True, 400, 1600, 1024),
                                      (False, 130, 96, 33)])
def test_gemm_96_wide_tiles(ta, M, N, K):
    """The 128 x 96 tile form (32-deep k-blocks, K-major B; chosen for fuller SM coverage), forced."""
    _run(ta, False, M, N, K, bias=not ta, relu=not ta, drain=True, force=16)

