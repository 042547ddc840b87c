import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1605_04809_b200 import nmt  # noqa: E402
nmt.bench_gemm(1024, 100096, 512, epi=4, ksplit=1, iters=2)
