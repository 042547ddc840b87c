"""Phase stamps of single GEMM launches in isolation (diagnostic library, NMT_GEMM_TRACE=1): operands
device-resident (L2-warm after the first launch), no preceding kernel of the step.
  NMT_LIB_PATH=paper_1605_04809_b200/libnmt_diag.so NMT_GEMM_TRACE=1 python tools/gemm_phase.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1605_04809_b200 import nmt  # noqa: E402

for name, M, N, K, epi, ks in [("q pair ks2", 1024, 2048, 1024, 3, 2), ("q pair ks1", 1024, 2048, 1024, 3, 1),
                               ("ro pair ks4", 1024, 1024, 3072, 3, 4), ("h1 pair", 1024, 4096, 1024, 3, 1),
                               ("big pair", 4096, 4096, 4096, 3, 1), ("vocab pair", 1024, 100096, 512, 4, 1)]:
    print(f"== {name} M={M} N={N} K={K} ks={ks}", file=sys.stderr, flush=True)
    ms = nmt.bench_gemm(M, N, K, epi=epi, ksplit=ks, iters=2)
    print(f"{name}: {ms*1000:.1f} us", file=sys.stderr, flush=True)
