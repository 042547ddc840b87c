"""Diagnostic driver for ncu: one nmt_encode_batch of n sentences (L ~ U[10,50]) at the En->Ru shape."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1605_04809_b200 import nmt  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
d = synth.Dims(500, 1024, 50000, 100000, "maxout")
M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016)), precision="bf16")
rng = np.random.default_rng(3000)
srcs = [synth.make_source(d.vocab_src, int(rng.integers(10, 51)), seed=7000 + i) for i in range(n)]
cs = M.encode_batch(srcs)
cs[0].check()
print("encoded", len(cs))
