"""tcgen05 3xTF32 GEMM (the MLP gradient's tensor-core path) against an fp64
reference of the same contraction (-m gpu)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_1710_06952_b200 import build
    build.build()
    import paper_1710_06952_b200 as P
    return P


@pytest.mark.parametrize("M,N,K,splits", [(128, 128, 32, 1), (128, 128, 256, 1), (256, 384, 512, 2),
                                          (128, 512, 3072, 12), (128, 512, 3072, 16), (128, 512, 3072, 8),
                                          (256, 128, 1024, 4), (512, 3072, 128, 1)])
def test_gemm_tf32x3_matches_fp64(P, M, N, K, splits):
    """splits a power of two <= 16: split-K reduced in DSMEM over a cluster; 12: partial planes"""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g)
    C = torch.empty(M, N, device="cuda")
    P.gemm_tf32x3(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, splits)
    ref = (A.double() @ B.double().T)
    err = (C.double() - ref).abs() / (A.double().abs() @ B.double().abs().T)
    # 3xTF32 ~ fp32: error relative to sum |a||b| well below 1e-5 (1xTF32 would be ~1e-3)
    assert err.max().item() < 2e-6, err.max().item()
