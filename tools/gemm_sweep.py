"""Time the tcgen05 GEMM engine on the decoder/encoder shapes next to cuBLAS (torch.matmul bf16)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1605_04809_b200 import nmt

SHAPES = [("h1", 1024, 3072, 1024), ("q", 1024, 2048, 1024), ("g2(full K)", 1024, 4096, 3072),
          ("ro", 1024, 1024, 3072), ("big", 4096, 4096, 4096), ("vocab", 1024, 100096, 512)]


def cublas_ms(M, N, K, iters=20):
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(a, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for name, M, N, K in SHAPES:
    epi = 1 if name == "vocab" else 0
    ours = nmt.bench_gemm(M, N, K, epi=epi)
    ours256 = nmt.bench_gemm(M, N, K, epi=2) if epi == 0 else float("nan")
    cb = cublas_ms(M, N, K)
    tf = 2 * M * N * K / 1e9
    print(f"{name:12s} M={M:5d} N={N:6d} K={K:5d}  ours {ours*1000:8.1f} us ({tf/ours:7.1f} TF/s)  "
          f"BN256 {ours256*1000:8.1f} us ({tf/ours256:7.1f})  cuBLAS {cb*1000:8.1f} us ({tf/cb:7.1f} TF/s)")
