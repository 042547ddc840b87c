import sys, os
sys.path.insert(0, "/root/repo")
import torch, numpy as np, synth
from paper_1605_04809_b200 import nmt
d = synth.TINY
blob = synth.params_bytes(d, synth.make_model(d, 7))
for alloc in ("torch", None):
    print("alloc", alloc, nmt.live_objects(), nmt.device_allocations(), flush=True)
    M = nmt.Model(blob, precision="fp32class", allocator=alloc)
    print(" loaded", nmt.live_objects(), nmt.device_allocations(), flush=True)
    c = M.encode(synth.make_source(d.vocab_src, 4, seed=1))
    print(" encoded", nmt.live_objects(), nmt.device_allocations(), flush=True)
    lp, _, _ = c.score_batch([0], [0, 3], [5, 9, 2])
    c.close()
    print(" ctx closed", nmt.live_objects(), nmt.device_allocations(), flush=True)
    M.close()
    print(" model closed", nmt.live_objects(), nmt.device_allocations(), flush=True)
