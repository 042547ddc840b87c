"""Diagnostic: where the time of one C5 sentence goes (host generation, forest call, device stages)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def main():
    import torch
    from paper_1605_04809_b200 import nmt
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    d = synth.Dims(500, 1024, 50000, 100000, "tanh")
    M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016)), precision="bf16")
    for rep in range(3):
        L = 30
        src = synth.make_source(d.vocab_src, L, seed=rep)
        g = np.random.default_rng(rep)
        t0 = time.perf_counter()
        ctx = M.encode_batch([src])[0]
        s, y = synth.make_states(B, d.dim_hid, d.vocab_tgt, seed=rep)
        t1 = time.perf_counter()
        hyps = ctx.inject_states(s, y)
        t2 = time.perf_counter()
        tg = tf = 0.0
        M.profile(2)
        M.profile_read()
        for stk in range(L + 1):
            a = time.perf_counter()
            Ls = g.choice(4, size=B, p=[.4, .3, .2, .1]).astype(np.int32) + 1
            off = np.zeros(B + 1, np.int32)
            off[1:] = np.cumsum(Ls)
            words = synth.zipf_ids(g, int(off[-1]), d.vocab_tgt)
            b = time.perf_counter()
            lp, fin, st = ctx.score_forest(hyps, off, words)
            c = time.perf_counter()
            hyps = fin
            tg += b - a
            tf += c - b
        ms, cnt = M.profile_read()
        M.profile(0)
        ctx.close()
        print(json.dumps({"B": B, "rep": rep, "encode+states_ms": 1000 * (t1 - t0), "inject_ms": 1000 * (t2 - t1),
                          "gen_ms_per_stack": 1000 * tg / (L + 1), "forest_ms_per_stack": 1000 * tf / (L + 1),
                          "device_ms_per_stack": {k: round(float(v) / (L + 1), 4) for k, v in zip(nmt.STAGES, ms) if v > 0},
                          "device_total_ms_per_stack": float(ms.sum()) / (L + 1)}), flush=True)


if __name__ == "__main__":
    main()
