"""First-stage latency of a decoder-shaped GEMM with warm operands (diagnostic build, NMT_GEMM_TRACE):
  NMT_LIB_PATH=paper_1605_04809_b200/libnmt_diag.so NMT_GEMM_TRACE=1 python tools/gemm_fill.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1605_04809_b200 import nmt  # noqa: E402

for _ in range(3):
    nmt.bench_gemm(1024, 2048, 1024, epi=2, ksplit=1, iters=3)   # 128 x 256 tiles, 1 CTA (q-like)
    nmt.bench_gemm(1024, 4096, 1088, epi=0, ksplit=1, iters=3)   # 128 x 128 tiles
