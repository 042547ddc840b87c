import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1605_04809_b200 import nmt
for R in (256, 1024, 4096):
    one = nmt.bench_gemm(R, 100096, 512, epi=1, iters=30)
    pair = nmt.bench_gemm(R, 100096, 512, epi=4, iters=30)
    tf = 2 * R * 100096 * 512 / 1e9
    print(f"R={R}: 1-CTA {one*1000:.1f} us ({tf/one:.0f} TF/s)   CTA pair {pair*1000:.1f} us ({tf/pair:.0f} TF/s)", flush=True)
