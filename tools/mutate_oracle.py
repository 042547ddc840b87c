#!/usr/bin/env python
"""Mutation check of the oracle's pins (VERDICT r01 "What's weak" #2): apply one plausible mistake at a
time to a COPY of oracle/nmt_oracle.py and run tests/test_oracle.py against it.  Every mutation must
make at least one test fail; the script exits 1 if any mutation survives.

  python tools/mutate_oracle.py [-k NAME]

Mutations (each names the line it corrupts):
  query_from_s      attention query q = s W_comb_att instead of s1 (reading A4, cGRU)
  gru2_state_s      GRU2 state s instead of s1
  pctx_transposed   pctx = ctx Wc_att^T instead of ctx Wc_att
  mode0_unweighted  ensemble mode 0 as the plain mean instead of sum_m lambda_m log p_m
  maxout_pairing    maxout over (k, k+E) instead of adjacent (2k, 2k+1) units (reading A7)
  readout_ctx_s1    readout takes s1 instead of s2
  gru_u_new_state   u weights the NEW state (h' = (1-u) h + u h~) (reading A2)
  bxnl_outside_r2   GRU2 bx_nl outside the reset product (reading A3)
  mean_ctx_sum      s0 from the SUM of ctx instead of the mean
  bos_embedding     BOS uses Wemb_dec[0] instead of the zero embedding (reading A9)
  no_b_att          pctx without b_att
  logz_no_max       logZ = log sum exp(z) - max (dropped the max term)
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = {
    "query_from_s": ('q = s1 @ p["decoder_W_comb_att"]', 'q = s @ p["decoder_W_comb_att"]'),
    "gru2_state_s": ("s2 = gru_nl(s1, ctx_r,", "s2 = gru_nl(s, ctx_r,"),
    "pctx_transposed": ('pctx = ctx @ p["decoder_Wc_att"]', 'pctx = ctx @ p["decoder_Wc_att"].T'),
    "mode0_unweighted": ("return (w * L).sum(axis=0)", "return L.mean(axis=0)"),
    "maxout_pairing": ("t = np.maximum(pre[:, 0::2], pre[:, 1::2])",
                       "t = np.maximum(pre[:, :pre.shape[1] // 2], pre[:, pre.shape[1] // 2:])"),
    "readout_ctx_s1": ('pre = (s2 @ p["ff_logit_lstm_W"]', 'pre = (s1 @ p["ff_logit_lstm_W"]'),
    "gru_u_new_state": ("return u * h + (1.0 - u) * htilde", "return (1.0 - u) * h + u * htilde"),
    "bxnl_outside_r2": ("htilde = np.tanh(r2 * (h1 @ Ux_nl + bx_nl) + c @ Wcx)",
                        "htilde = np.tanh(r2 * (h1 @ Ux_nl) + bx_nl + c @ Wcx)"),
    "mean_ctx_sum": ('s0 = np.tanh(ctx.mean(axis=0) @ p["ff_state_W"]', 's0 = np.tanh(ctx.sum(axis=0) @ p["ff_state_W"]'),
    "bos_embedding": ('e = np.where((y >= 0)[:, None], p["Wemb_dec"][np.maximum(y, 0)], 0.0)',
                      'e = p["Wemb_dec"][np.maximum(y, 0)]'),
    "no_b_att": ('pctx = ctx @ p["decoder_Wc_att"] + p["decoder_b_att"]', 'pctx = ctx @ p["decoder_Wc_att"]'),
    "logz_no_max": ("return (m + np.log(np.sum(np.exp(z - m), axis=axis, keepdims=True))).squeeze(axis)",
                    "return (np.log(np.sum(np.exp(z - m), axis=axis, keepdims=True))).squeeze(axis)"),
}


def run_one(name: str, old: str, new: str, verbose: bool) -> bool:
    """True if the mutation is KILLED (some test fails)."""
    src = open(os.path.join(ROOT, "oracle", "nmt_oracle.py")).read()
    if src.count(old) != 1:
        raise SystemExit(f"{name}: pattern not found exactly once in the oracle: {old!r}")
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("oracle", "synth", "tests"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("__pycache__"))
        with open(os.path.join(tmp, "oracle", "nmt_oracle.py"), "w") as f:
            f.write(src.replace(old, new))
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                            "tests/test_oracle.py"], cwd=tmp, capture_output=True, text=True)
        tail = [ln for ln in r.stdout.splitlines() if ln.strip()][-2:]
        if verbose:
            print("   ", " | ".join(tail))
        return r.returncode != 0


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default=None)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    survivors = []
    for name, (old, new) in MUTATIONS.items():
        if a.k and a.k not in name:
            continue
        killed = run_one(name, old, new, a.v)
        print(f"{name:18s} {'killed' if killed else 'SURVIVED'}", flush=True)
        if not killed:
            survivors.append(name)
    if survivors:
        print("surviving mutations:", ", ".join(survivors))
        return 1
    print("every mutation is killed by tests/test_oracle.py")
    return 0


if __name__ == "__main__":
    sys.exit(main())
