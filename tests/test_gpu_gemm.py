"""tcgen05 GEMM engine vs a float64 reference of the same (bf16-rounded) operands."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def bf16(a):
    return torch.tensor(a, dtype=torch.float32).bfloat16().double().numpy()


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (200, 384, 512), (1, 256, 1024), (300, 1024, 192)])
def test_gemm_bf16(M, N, K):
    from paper_1605_04809_b200 import nmt
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    bias = rng.standard_normal(N).astype(np.float32)
    C = nmt.test_gemm(A, B, bias, split=False)
    ref = bf16(A) @ bf16(B) + bias
    assert np.max(np.abs(C - ref)) < 1e-4 * np.sqrt(K) * 4


@pytest.mark.parametrize("M,N,K", [(130, 256, 512), (77, 128, 2048)])
def test_gemm_split_bf16x3(M, N, K):
    from paper_1605_04809_b200 import nmt
    rng = np.random.default_rng(M * 7 + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    C = nmt.test_gemm(A, B, None, split=True)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    # bf16x3 drops lo*lo (~2^-16 relative per product) plus fp32 accumulation
    assert np.max(np.abs(C - ref)) < 2e-5 * np.sqrt(K) * 4
