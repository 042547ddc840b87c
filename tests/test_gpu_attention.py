"""Attention (D3-D5) through both of its arithmetic paths, against the float64 oracle.

The kernel evaluates tanh(p + q) as 1 - 2 / (1 + e^2p e^2q) with e^2p precomputed per context and e^2q per
row (reading A30); when an exponent had to be clamped (|2 pctx| or |2 q| > 21, kAttnExpClamp) the context or
the CTA's rows take the direct tanh path.  These tests force each path with saturating weights
(PAPER.md:13, :30 - the DL4MT cGRU attention) and check alpha, c and the scores against the oracle."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

TOL = {"fp32class": 1e-3, "bf16": 2e-2}


def nmt():
    from paper_1605_04809_b200 import nmt as m
    return m


def _model(scale_batt: float, scale_wq: float, prec: str, seed: int = 7):
    d = synth.Dims(8, 16, 50, 50, "tanh")
    p = synth.make_model(d, seed)
    p["decoder_b_att"] = (p["decoder_b_att"] * scale_batt).astype(np.float32)
    p["decoder_W_comb_att"] = (p["decoder_W_comb_att"] * scale_wq).astype(np.float32)
    return d, p, nmt().Model(synth.params_bytes(d, p), precision=prec), O.Model(d, p)


# (b_att scale, W_comb_att scale): exp path; keys beyond the clamp (whole context on the tanh path);
# queries beyond the clamp on some rows (per-CTA fallback next to exp-path CTAs)
CASES = [(1.0, 1.0), (400.0, 1.0), (1.0, 60.0)]


@pytest.mark.parametrize("prec", ["fp32class", "bf16"])
@pytest.mark.parametrize("sb,sq", CASES, ids=["exp", "big-keys", "big-queries"])
def test_attention_paths_vs_oracle(sb, sq, prec):
    d, p, M, om = _model(sb, sq, prec)
    src = synth.make_source(d.vocab_src, 6, seed=4)
    c = M.encode(src)
    sess = O.Session(om, src)
    if sb > 1:  # the keys really exceed the clamp
        assert np.max(np.abs(2 * O.encode(om, src).pctx)) > 21
    g = c.debug_intermediates(c.root)
    r = sess.intermediates(0)
    tol = {"fp32class": 2e-4, "bf16": 2e-2}[prec]
    for k in ("alpha", "c", "s2"):
        assert np.max(np.abs(g[k] - r[k])) < tol, k
    # a batch of parents (root children) so that several attention CTAs run, each with its rows
    lp1, ch1, _ = c.score_batch([0], [0, 12], list(range(2, 14)))
    rl1, rc1, _ = sess.score_batch([0], [0, 12], list(range(2, 14)))
    assert list(ch1) == list(rc1)
    parents = [int(x) for x in ch1]
    words = [int(w) for w in np.random.default_rng(1).integers(0, d.vocab_tgt, size=3 * len(parents))]
    off = list(range(0, 3 * len(parents) + 1, 3))
    lp, ch, _ = c.score_batch(parents, off, words)
    rl, rc, _ = sess.score_batch(parents, off, words)
    assert list(ch) == list(rc)
    assert max(np.max(np.abs(lp1 - rl1)), np.max(np.abs(lp - rl))) < TOL[prec]


def test_attention_rows_balanced_large_batch():
    """R = 1000 injected parents (not a multiple of the 296 CTAs): every row's alpha-weighted context
    enters its scores; sampled rows against the oracle."""
    d = synth.Dims(8, 16, 50, 50, "maxout")
    p = synth.make_model(d, 11)
    M = nmt().Model(synth.params_bytes(d, p), precision="fp32class")
    om = O.Model(d, p)
    src = synth.make_source(d.vocab_src, 9, seed=5)
    c = M.encode(src)
    R = 1000
    rng = np.random.default_rng(3)
    s = np.tanh(rng.standard_normal((R, d.dim_hid))).astype(np.float32)
    y = rng.integers(-1, d.vocab_tgt, size=R).astype(np.int32)
    ids = c.inject_states(s, y)
    words = rng.integers(0, d.vocab_tgt, size=R).astype(np.int32)
    lp, _, _ = c.score_batch(ids, np.arange(R + 1, dtype=np.int32), words)
    sess = O.Session(om, src)
    for i in list(range(0, R, 97)) + [R - 1]:
        sid = sess.inject_state(s[i].astype(np.float64), int(y[i]))
        ref, _, _ = sess.score_batch([sid], [0, 1], [int(words[i])])
        assert abs(float(lp[i]) - float(ref[0])) < 1e-3, i
