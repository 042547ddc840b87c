"""Diagnostic: per-stage device time of one fused multi-context call (nmt_score_batch_multi) for
G contexts x B fresh parents (1 word each), with the model's CUDA-event stage profile."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def main():
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(500, 1024, 50000, 100000, "maxout")
    M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016)), precision="bf16")
    for G, B in [(32, 1024), (130, 256), (256, 128), (512, 64)]:
        srcs = [synth.make_source(d.vocab_src, 30, seed=i) for i in range(G)]
        cs = M.encode_batch(srcs)
        s, y = synth.make_states(B, d.dim_hid, d.vocab_tgt, seed=1)
        for c in cs:
            c.reserve(20 * B, 20 * B)
        hnd = np.repeat(np.array([c.handle for c in cs], np.int64), B)
        off = np.arange(G * B + 1, dtype=np.int32)
        words = synth.zipf_ids(np.random.default_rng(0), G * B, d.vocab_tgt)
        res = []
        for it in range(6):
            par = np.concatenate([c.inject_states(s, y) for c in cs])
            if it == 3:
                M.profile(2)
                M.profile_read()
            t0 = time.perf_counter()
            nmt.score_batch_multi(hnd, par, off, words, with_argmax=False)
            res.append(time.perf_counter() - t0)
        ms, cnt = M.profile_read()
        M.profile(0)
        print(json.dumps({"G": G, "B": B, "rows": G * B, "wall_ms": [round(1000 * x, 2) for x in res],
                          "stages_ms_3calls": {k: round(float(v), 3) for k, v in zip(nmt.STAGES, ms) if v > 0}}),
              flush=True)
        for c in cs:
            c.close()


if __name__ == "__main__":
    main()
