"""Time the encoder recurrence kernel at several source lengths (per-step vs fixed cost)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from paper_1605_04809_b200 import nmt

d = synth.Dims(500, 1024, 50000, 100000, "maxout")
M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016)), precision="bf16")
ri = nmt.STAGES.index("enc_recurrence")
for Tx in [1, 2, 5, 10, 25, 50, 64]:
    src = synth.make_source(d.vocab_src, Tx - 1, seed=Tx)
    for _ in range(3):
        M.encode(src).close()
    M.profile(2)
    M.profile_read()
    for _ in range(20):
        M.encode(src).close()
    ms, cnt = M.profile_read()
    M.profile(0)
    print(f"Tx={Tx:3d}  recurrence {1000 * ms[ri] / cnt[ri]:8.1f} us")
