import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1605_04809_b200 import nmt
for M, N, K in [(1024, 1024, 3072), (1, 128, 384), (128, 128, 384), (200, 256, 384)]:
    print(M, N, K, flush=True)
    print("  ms", nmt.bench_gemm(M, N, K, epi=5, ksplit=1, iters=2), flush=True)
