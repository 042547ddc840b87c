"""MMA-issuer wait accounting and phase stamps for GEMM shapes in isolation (diagnostic library):
  NMT_LIB_PATH=paper_1605_04809_b200/libnmt_diag.so NMT_GEMM_TRACE=1 python tools/gemm_phase2.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1605_04809_b200 import nmt  # noqa: E402

for name, M, N, K, epi in [("vocab LSE pair", 1024, 100096, 512, 4), ("vocab shape, store pair", 1024, 100096, 512, 3),
                           ("K=512 square store pair", 4096, 8192, 512, 3), ("big store pair", 4096, 4096, 4096, 3)]:
    print(f"== {name} M={M} N={N} K={K}", file=sys.stderr, flush=True)
    ms = nmt.bench_gemm(M, N, K, epi=epi, ksplit=1, iters=2)
    print(f"{name}: {ms*1000:.1f} us  {2*M*N*K/ms/1e9:.0f} TFLOP/s", file=sys.stderr, flush=True)
