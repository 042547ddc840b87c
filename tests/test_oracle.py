"""Pins of the float64 oracle against things other than itself (SURVEY §8(c) "What pins
each part"): torch float64 library routines after a weight re-pack, scipy, closed forms, saturation
cases, brute-force enumeration, invariants, and the paper's Fig. 1 worked example."""
import itertools
import math
import os

import numpy as np
import pytest
import scipy.special
import torch

import oracle as O
import synth

TINY = synth.TINY
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def tiny_model(seed=7, readout="tanh", **over):
    d = synth.Dims(TINY.dim_emb, TINY.dim_hid, TINY.vocab_src, TINY.vocab_tgt, readout)
    p = synth.make_model(d, seed)
    p.update({k: np.asarray(v, np.float32) for k, v in over.items()})
    return d, p, O.Model(d, p)


def t64(a):
    return torch.tensor(np.asarray(a, np.float64), dtype=torch.float64)


# ------------------------------------------------------------------ GRU forms vs torch.nn.GRUCell
def test_gru1_matches_torch_grucell():
    d, p, m = tiny_model()
    H = d.dim_hid
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, d.dim_emb))
    h = np.tanh(rng.standard_normal((5, H)))
    cell = torch.nn.GRUCell(d.dim_emb, H).double()
    with torch.no_grad():
        cell.weight_ih.copy_(t64(np.concatenate([m.p["decoder_W"], m.p["decoder_Wx"]], 1).T))
        cell.bias_ih.copy_(t64(np.concatenate([m.p["decoder_b"], m.p["decoder_bx"]])))
        cell.weight_hh.copy_(t64(np.concatenate([m.p["decoder_U"], m.p["decoder_Ux"]], 1).T))
        cell.bias_hh.zero_()
        ref = cell(t64(x), t64(h)).numpy()
    got = O.gru(x, h, m.p["decoder_W"], m.p["decoder_b"], m.p["decoder_U"],
                m.p["decoder_Wx"], m.p["decoder_bx"], m.p["decoder_Ux"])
    assert np.max(np.abs(got - ref)) < 1e-14


def test_gru2_matches_torch_grucell_bias_inside_reset():
    d, p, m = tiny_model()
    H, C = d.dim_hid, d.ctx_dim
    rng = np.random.default_rng(1)
    c = rng.standard_normal((4, C))
    h1 = np.tanh(rng.standard_normal((4, H)))
    cell = torch.nn.GRUCell(C, H).double()
    with torch.no_grad():
        cell.weight_ih.copy_(t64(np.concatenate([m.p["decoder_Wc"], m.p["decoder_Wcx"]], 1).T))
        cell.bias_ih.zero_()
        cell.weight_hh.copy_(t64(np.concatenate([m.p["decoder_U_nl"], m.p["decoder_Ux_nl"]], 1).T))
        cell.bias_hh.copy_(t64(np.concatenate([m.p["decoder_b_nl"], m.p["decoder_bx_nl"]])))
        ref = cell(t64(c), t64(h1)).numpy()
    got = O.gru_nl(h1, c, m.p["decoder_U_nl"], m.p["decoder_b_nl"], m.p["decoder_Ux_nl"],
                   m.p["decoder_bx_nl"], m.p["decoder_Wc"], m.p["decoder_Wcx"])
    assert np.max(np.abs(got - ref)) < 1e-14


def test_encoder_matches_torch_bidirectional_gru_and_mean_init():
    d, p, m = tiny_model()
    H = d.dim_hid
    src = synth.make_source(d.vocab_src, 6, seed=3)
    gru = torch.nn.GRU(d.dim_emb, H, bidirectional=True).double()
    with torch.no_grad():
        for suf, pre in (("", "encoder"), ("_reverse", "encoder_r")):
            getattr(gru, "weight_ih_l0" + suf).copy_(t64(np.concatenate([m.p[pre + "_W"], m.p[pre + "_Wx"]], 1).T))
            getattr(gru, "bias_ih_l0" + suf).copy_(t64(np.concatenate([m.p[pre + "_b"], m.p[pre + "_bx"]])))
            getattr(gru, "weight_hh_l0" + suf).copy_(t64(np.concatenate([m.p[pre + "_U"], m.p[pre + "_Ux"]], 1).T))
            getattr(gru, "bias_hh_l0" + suf).zero_()
        out, _ = gru(t64(m.p["Wemb"][src])[:, None, :])
    ref_ctx = out[:, 0, :].numpy()
    c = O.encode(m, src)
    assert c.ctx.shape == (len(src), 2 * H)
    assert np.max(np.abs(c.ctx - ref_ctx)) < 1e-14
    # s0 with ff_state_W = [I; 0] is tanh(mean_j fwd_j + b): pins the mean over positions
    W = np.zeros((2 * H, H), np.float32)
    W[:H] = np.eye(H)
    _, _, m2 = tiny_model(ff_state_W=W)
    c2 = O.encode(m2, src)
    ref_s0 = torch.tanh(out[:, 0, :H].mean(0) + t64(m2.p["ff_state_b"])).numpy()
    assert np.max(np.abs(c2.s0 - ref_s0)) < 1e-14
    # pctx with Wc_att = I, b_att = 0 is ctx itself
    _, _, m3 = tiny_model(decoder_Wc_att=np.eye(2 * H, dtype=np.float32),
                          decoder_b_att=np.zeros((1, 2 * H), np.float32))
    c3 = O.encode(m3, src)
    assert np.array_equal(c3.pctx, c3.ctx)


def test_encoder_reversal_invariant():
    d, p, _ = tiny_model()
    q = dict(p)
    for s in ("W", "b", "U", "Wx", "bx", "Ux"):
        q["encoder_r_" + s] = p["encoder_" + s]
    m = O.Model(d, q)
    src = synth.make_source(d.vocab_src, 7, seed=5)
    c = O.encode(m, src)
    cr = O.encode(m, src[::-1].copy())
    H = d.dim_hid
    assert np.max(np.abs(c.ctx[:, H:] - cr.ctx[::-1, :H])) < 1e-15


def test_gru_closed_form_zero_matrices():
    H = 16
    rng = np.random.default_rng(2)
    b = rng.standard_normal(2 * H)
    bx = rng.standard_normal(H)
    Z = lambda *s: np.zeros(s)
    h = np.zeros(H)
    x = rng.standard_normal(8)
    for t in range(1, 6):
        h = O.gru(x, h, Z(8, 2 * H), b, Z(H, 2 * H), Z(8, H), bx, Z(H, H))
        u = 1 / (1 + math.e ** (-b[H:]))
        assert np.max(np.abs(h - (1 - u ** t) * np.tanh(bx))) < 1e-15
    # GRU2 with zero matrices: h2 = u2*h1 + (1-u2)*tanh(sigm(b_r)*bx_nl)
    h1 = np.tanh(rng.standard_normal(H))
    h2 = O.gru_nl(h1, rng.standard_normal(2 * H), Z(H, 2 * H), b, Z(H, H), bx, Z(2 * H, 2 * H), Z(2 * H, H))
    r2, u2 = 1 / (1 + np.exp(-b[:H])), 1 / (1 + np.exp(-b[H:]))
    assert np.max(np.abs(h2 - (u2 * h1 + (1 - u2) * np.tanh(r2 * bx)))) < 1e-15


# ------------------------------------------------------------------ cGRU composition (closed forms)
# The conditional GRU of DL4MT (reading A4) is defined by WHERE s1 goes: the
# attention query and the GRU2 state both come from s1, the output of GRU1, not from the input
# state s.  With GRU1's matrices zero, s1 is known in closed form (u weights the old state, A2):
#   s1 = u1*s + (1-u1)*tanh(bx),  u1 = sigm(b_u)
# and it can be made to have the opposite sign of s on a chosen coordinate.  These tests fail if the
# query or the GRU2 state is taken from s (tools/mutate_oracle.py checks exactly that).
def _cgru_probe_model(H=16, E=8, V=50):
    d = synth.Dims(E, H, 50, V, "tanh")
    p = synth.make_model(d, 31)
    for k in ("decoder_W", "decoder_U", "decoder_Wx", "decoder_Ux"):
        p[k] = np.zeros_like(p[k])
    return d, p


def _s1_closed_form(p, s, H):
    b = p["decoder_b"].astype(np.float64).reshape(-1)
    bx = p["decoder_bx"].astype(np.float64).reshape(-1)
    u1 = 1.0 / (1.0 + np.exp(-b[H:]))
    return u1 * s + (1.0 - u1) * np.tanh(bx)


def test_attention_query_comes_from_gru1_output():
    d, p = _cgru_probe_model()
    H, C, k, col, Tx, jstar = d.dim_hid, d.ctx_dim, 3, 5, 6, 2
    p["decoder_b"] = p["decoder_b"].copy()
    p["decoder_b"][0, H + k] = -30.0            # u1[k] ~ 0: s1[k] = tanh(bx[k])
    p["decoder_bx"] = p["decoder_bx"].copy()
    p["decoder_bx"][0, k] = 2.0                  # s1[k] = tanh(2) > 0
    W = np.zeros((H, C), np.float32)
    W[k, col] = 40.0                             # q[col] = 40 s1[k]: one-hot route of coordinate k
    p["decoder_W_comb_att"] = W
    ua = np.zeros((C, 1), np.float32)
    ua[col, 0] = 8.0
    p["decoder_U_att"] = ua
    m = O.Model(d, p)
    rng = np.random.default_rng(12)
    ctx = rng.standard_normal((Tx, C))
    pctx = np.full((Tx, C), -40.0)
    pctx[jstar, :] = 0.0                         # position j* lights up only for a POSITIVE query
    c = O.Context(ctx=ctx, pctx=pctx, s0=np.zeros(H))
    s = np.zeros((1, H))
    s[0, k] = -0.9                               # the input state has the opposite sign
    out = O.step(m, c, s, [O.BOS])
    s1 = _s1_closed_form(m.p, s[0], H)
    assert s1[k] > 0.9 and s[0, k] < 0
    # by hand: a_j = 8 tanh(pctx[j, col] + 40 s1[k]) + c_tt, alpha = softmax_j(a)
    a = 8.0 * np.tanh(pctx[:, col] + 40.0 * s1[k])
    alpha = np.exp(a - a.max())
    alpha /= alpha.sum()
    assert np.max(np.abs(out["s1"][0] - s1)) < 1e-15
    assert np.max(np.abs(out["alpha"][0] - alpha)) < 1e-12
    assert out["alpha"][0, jstar] > 0.99         # (a query from s would give uniform attention)
    assert np.max(np.abs(out["c"][0] - alpha @ ctx)) < 1e-12


def test_gru2_state_is_gru1_output():
    d, p = _cgru_probe_model()
    H = d.dim_hid
    for k in ("decoder_U_nl", "decoder_Wc", "decoder_Ux_nl", "decoder_Wcx"):
        p[k] = np.zeros_like(p[k])
    p["decoder_b"] = p["decoder_b"].copy()
    p["decoder_b"][0, H:] = -30.0                # u1 ~ 0: s1 = tanh(bx), independent of s
    p["decoder_bx"] = np.full((1, H), 1.5, np.float32)
    p["decoder_b_nl"] = np.zeros((1, 2 * H), np.float32)   # r2 = u2 = 1/2
    m = O.Model(d, p)
    c = O.encode(m, synth.make_source(d.vocab_src, 5, seed=3))
    s = -np.tanh(np.abs(np.random.default_rng(4).standard_normal((2, H))))   # s < 0 everywhere
    out = O.step(m, c, s, [7, O.BOS])
    s1 = np.stack([_s1_closed_form(m.p, s[r], H) for r in range(2)])
    bx_nl = m.p["decoder_bx_nl"]
    s2 = 0.5 * s1 + 0.5 * np.tanh(0.5 * bx_nl)   # GRU2 with zero matrices: state s1, bx_nl inside r2
    assert np.max(np.abs(out["s2"] - s2)) < 1e-15
    assert np.min(s1) > 0.9                      # (a GRU2 state s < 0 would differ by >= 0.45)


def test_encoder_closed_form_and_pctx_orientation():
    """Zero encoder matrices: fwd_j = (1 - u_f^(j+1)) tanh(bx_f), bwd_j = (1 - u_b^(Tx-j)) tanh(bx_b)
    (GRU closed form, h_{-1} = h_{Tx} = 0).  pctx = ctx Wc_att + b_att with a NON-symmetric
    permutation Wc_att (pctx[:, pi(i)] = ctx[:, i]) pins the orientation of the product."""
    d = synth.Dims(8, 16, 50, 50, "tanh")
    p = synth.make_model(d, 41)
    H, C = d.dim_hid, d.ctx_dim
    for pre in ("encoder", "encoder_r"):
        for s in ("W", "U", "Wx", "Ux"):
            p[f"{pre}_{s}"] = np.zeros_like(p[f"{pre}_{s}"])
    pi = np.random.default_rng(5).permutation(C)
    P = np.zeros((C, C), np.float32)
    P[np.arange(C), pi] = 1.0
    assert not np.array_equal(P, P.T)
    p["decoder_Wc_att"] = P
    p["decoder_b_att"] = np.zeros((1, C), np.float32)
    m = O.Model(d, p)
    src = synth.make_source(d.vocab_src, 6, seed=9)
    Tx = len(src)
    c = O.encode(m, src)
    sg = lambda x: 1.0 / (1.0 + np.exp(-x))
    bf, bb = m.p["encoder_b"], m.p["encoder_r_b"]
    for j in range(Tx):
        fwd = (1 - sg(bf[H:]) ** (j + 1)) * np.tanh(m.p["encoder_bx"])
        bwd = (1 - sg(bb[H:]) ** (Tx - j)) * np.tanh(m.p["encoder_r_bx"])
        assert np.max(np.abs(c.ctx[j, :H] - fwd)) < 1e-14
        assert np.max(np.abs(c.ctx[j, H:] - bwd)) < 1e-14
    assert np.array_equal(c.pctx[:, pi], c.ctx)


def test_ensemble_weighted_combine_hand_values():
    """PAPER.md:92 (models as separately WEIGHTED features), reading A16, with unequal weights."""
    L1 = np.log([0.5, 0.25, 0.25])
    L2 = np.log([0.25, 0.25, 0.5])
    ln2 = math.log(2.0)
    got0 = O.ensemble_combine([L1, L2], [0.75, 0.25], 0)
    assert np.max(np.abs(got0 - np.array([-1.25 * ln2, -2 * ln2, -1.75 * ln2]))) < 1e-15
    got1 = O.ensemble_combine([L1, L2], [0.75, 0.25], 1)
    assert np.max(np.abs(got1 - np.log([0.4375, 0.25, 0.3125]))) < 1e-15


# ------------------------------------------------------------------ whole model / attention closed forms
def test_zero_model_uniform():
    d = TINY
    m = O.Model(d, synth.zero_model(d))
    sess = O.Session(m, synth.make_source(d.vocab_src, 4, seed=1))
    lp, ch, am = sess.score_batch([0], [0, 3], [5, 9, 2])
    assert np.max(np.abs(lp + math.log(d.vocab_tgt))) < 1e-15
    inter = sess.intermediates(0)
    assert np.max(np.abs(inter["alpha"] - 1.0 / 5)) < 1e-16
    assert am[0] == 0  # all logits equal -> lowest id


def _ctx_by_hand(Tx, C, rng):
    ctx = rng.standard_normal((Tx, C))
    return ctx


def test_attention_saturated_one_hot_selects_context():
    d, p, m = tiny_model()
    C = d.ctx_dim
    rng = np.random.default_rng(4)
    Tx, jstar, k = 6, 4, 3
    ctx = rng.standard_normal((Tx, C))
    pctx = np.zeros((Tx, C))
    pctx[:, k] = -50.0
    pctx[jstar, k] = 50.0
    m.p["decoder_U_att"] = np.zeros(C)
    m.p["decoder_U_att"][k] = 10.0
    m.p["decoder_W_comb_att"] = m.p["decoder_W_comb_att"] * 0.01
    c = O.Context(ctx=ctx, pctx=pctx, s0=np.zeros(d.dim_hid))
    out = O.step(m, c, np.tanh(rng.standard_normal((3, d.dim_hid))), [5, O.BOS, 7])
    assert np.all(np.abs(out["alpha"][:, jstar] - 1) < 1e-7)
    assert np.max(np.abs(out["c"] - ctx[jstar])) < 1e-6
    assert np.allclose(out["alpha"].sum(1), 1, atol=1e-15)


def test_attention_saturated_bias_and_query_give_uniform():
    d, p, m = tiny_model()
    src = synth.make_source(d.vocab_src, 5, seed=2)
    s = np.tanh(np.random.default_rng(6).standard_normal((2, d.dim_hid)))
    # b_att huge: every tanh saturates to 1 -> uniform attention (pins that b_att enters)
    _, _, mb = tiny_model(decoder_b_att=np.full((1, d.ctx_dim), 1e3, np.float32))
    out = O.step(mb, O.encode(mb, src), s, [3, 4])
    assert np.max(np.abs(out["alpha"] - 1 / 6)) < 1e-15
    assert np.max(np.abs(out["c"] - O.encode(mb, src).ctx.mean(0))) < 1e-14
    # W_comb_att huge: tanh saturates to sign(q) for every source position -> uniform
    _, _, mq = tiny_model(decoder_W_comb_att=p["decoder_W_comb_att"] * 1e5)
    out = O.step(mq, O.encode(mq, src), s, [3, 4])
    assert np.max(np.abs(out["alpha"] - 1 / 6)) < 1e-12
    # Tx = 1 -> alpha = [1]
    out = O.step(m, O.encode(m, [0]), s, [3, 4])
    assert np.array_equal(out["alpha"], np.ones((2, 1)))


def test_c_tt_and_b_o_shift_invariance():
    d, p, m = tiny_model()
    src = synth.make_source(d.vocab_src, 5, seed=2)
    base = O.Session(m, src).logprobs_full(0)
    _, _, m1 = tiny_model(decoder_c_tt=p["decoder_c_tt"] + 5)
    _, _, m2 = tiny_model(ff_logit_b=p["ff_logit_b"] + 3)
    assert np.max(np.abs(O.Session(m1, src).logprobs_full(0) - base)) < 1e-13
    assert np.max(np.abs(O.Session(m2, src).logprobs_full(0) - base)) < 1e-13


# ------------------------------------------------------------------ readout terms vs torch Linear
@pytest.mark.parametrize("readout", ["tanh", "maxout"])
@pytest.mark.parametrize("term", ["lstm", "prev", "ctx", "bias"])
def test_readout_single_term_matches_torch(readout, term):
    d, p, _ = tiny_model(readout=readout)
    q = dict(p)
    for t in ("lstm", "prev", "ctx"):
        if t != term:
            q[f"ff_logit_{t}_W"] = np.zeros_like(p[f"ff_logit_{t}_W"])
        q[f"ff_logit_{t}_b"] = np.zeros_like(p[f"ff_logit_{t}_b"]) if term != "bias" else p[f"ff_logit_{t}_b"]
    if term == "bias":
        for t in ("lstm", "prev", "ctx"):
            q[f"ff_logit_{t}_W"] = np.zeros_like(p[f"ff_logit_{t}_W"])
    m = O.Model(d, q)
    src = synth.make_source(d.vocab_src, 5, seed=8)
    c = O.encode(m, src)
    rng = np.random.default_rng(9)
    y = [6, 11, 3]
    out = O.step(m, c, np.tanh(rng.standard_normal((3, d.dim_hid))), y)
    with torch.no_grad():
        if term == "lstm":
            pre = torch.nn.functional.linear(t64(out["s2"]), t64(m.p["ff_logit_lstm_W"]).T)
        elif term == "prev":
            emb = torch.nn.functional.embedding(torch.tensor(y), t64(m.p["Wemb_dec"]))
            pre = torch.nn.functional.linear(emb, t64(m.p["ff_logit_prev_W"]).T)
        elif term == "ctx":
            pre = torch.nn.functional.linear(t64(out["c"]), t64(m.p["ff_logit_ctx_W"]).T)
        else:
            pre = (t64(p["ff_logit_lstm_b"][0]) + t64(p["ff_logit_prev_b"][0]) + t64(p["ff_logit_ctx_b"][0])).expand(3, -1)
        if readout == "tanh":
            ref = torch.tanh(pre)
        else:
            ref = torch.nn.functional.max_pool1d(pre[:, None, :], 2)[:, 0, :]
    assert out["t"].shape == (3, d.dim_emb)
    assert np.max(np.abs(out["t"] - ref.numpy())) < 1e-14


def test_bos_uses_zero_embedding():
    d, p, m = tiny_model()
    c = O.encode(m, synth.make_source(d.vocab_src, 5, seed=8))
    s = np.tanh(np.random.default_rng(3).standard_normal((1, d.dim_hid)))
    q = dict(p)
    q["Wemb_dec"] = p["Wemb_dec"].copy()
    q["Wemb_dec"][4] = 0.0
    mz = O.Model(d, q)
    a = O.step(m, c, s, [O.BOS])
    b = O.step(mz, O.encode(mz, synth.make_source(d.vocab_src, 5, seed=8)), s, [4])
    assert np.max(np.abs(a["logZ"] - b["logZ"])) < 1e-15


# ------------------------------------------------------------------ log-softmax
def test_log_softmax_matches_scipy_and_normalises():
    d, p, m = tiny_model()
    sess = O.Session(m, synth.make_source(d.vocab_src, 5, seed=2))
    inter = sess.intermediates(0)
    ref = scipy.special.log_softmax(inter["z"])
    got = sess.logprobs_full(0)
    assert np.max(np.abs(got - ref)) < 1e-14
    assert abs(np.exp(got).sum() - 1) < 1e-13
    assert abs(inter["logZ"] - scipy.special.logsumexp(inter["z"])) < 1e-13
    assert inter["argmax"] == int(np.argmax(ref))


# ------------------------------------------------------------------ brute force over a tiny vocabulary
@pytest.mark.parametrize("L", [1, 2, 3])
def test_tiny_vocab_brute_force_sums_to_one(L):
    d, p, m = tiny_model(seed=7)
    V = d.vocab_tgt
    sess = O.Session(m, synth.make_source(d.vocab_src, 4, seed=11))
    frontier = {(): 0}
    cum = {(): 0.0}
    for depth in range(L):
        keys = sorted(frontier)
        parents = [frontier[k] for k in keys]
        offs = list(range(0, V * len(keys) + 1, V))
        lp, ch, _ = sess.score_batch(parents, offs, list(range(V)) * len(keys))
        nxt, ncum = {}, {}
        for i, k in enumerate(keys):
            for w in range(V):
                nxt[k + (w,)] = int(ch[i * V + w])
                ncum[k + (w,)] = cum[k] + lp[i * V + w]
        frontier, cum = nxt, ncum
    total = sum(math.exp(v) for v in cum.values())
    assert len(cum) == V ** L
    assert abs(total - 1.0) < 1e-12
    if L == 2:  # spot-check trie sums against the uncached sequential scorer
        for seq in [(0, 0), (3, 17), (49, 2)]:
            ref, _, _ = O.score_sequence(m, sess.c, seq)
            assert abs(cum[seq] - ref) < 1e-12
    if L == 1:  # argmax by full enumeration
        best = max(range(V), key=lambda w: (cum[(w,)], -w))
        assert sess.nodes[0].argmax == best


# ------------------------------------------------------------------ invariants
def test_prefix_additivity_and_cache_reuse_equals_recomputation():
    d, p, m = tiny_model(seed=13)
    src = synth.make_source(d.vocab_src, 6, seed=4)
    sess = O.Session(m, src)
    rng = np.random.default_rng(5)
    seqs = [tuple(int(x) for x in rng.integers(0, d.vocab_tgt, size=rng.integers(1, 5))) for _ in range(40)]
    # drive the cache with one score_batch per depth, in random interleavings
    for seq in seqs:
        node, acc = 0, 0.0
        for w in seq:
            lp, ch, _ = sess.score_batch([node], [0, 1], [w])
            acc += lp[0]
            node = int(ch[0])
        ref, lps, _ = O.score_sequence(m, sess.c, seq)
        assert abs(acc - ref) < 1e-12
        assert abs(ref - sum(lps)) < 1e-15
    u, v = seqs[0], seqs[1]
    su, _, st = O.score_sequence(m, sess.c, u)
    sv, _, _ = O.score_sequence(m, sess.c, v, s=st, y_prev=u[-1])
    suv, _, _ = O.score_sequence(m, sess.c, u + v)
    assert abs(suv - (su + sv)) < 1e-12


def test_batch_independence_and_duplicates():
    d, p, m = tiny_model()
    c = O.encode(m, synth.make_source(d.vocab_src, 5, seed=2))
    rng = np.random.default_rng(8)
    s = np.tanh(rng.standard_normal((6, d.dim_hid)))
    y = [3, O.BOS, 9, 9, 40, 2]
    full = O.step(m, c, s, y)
    perm = rng.permutation(6)
    pm = O.step(m, c, s[perm], [y[i] for i in perm])
    one = O.step(m, c, s[2:3], y[2:3])
    for k in ("s2", "t", "logZ", "alpha"):
        assert np.max(np.abs(pm[k] - full[k][perm])) < 1e-13
        assert np.max(np.abs(one[k][0] - full[k][2])) < 1e-13
    dup = O.step(m, c, np.stack([s[0], s[0]]), [3, 3])
    assert np.array_equal(dup["t"][0], dup["t"][1])


def test_score_batch_dedup_and_ids():
    d, p, m = tiny_model()
    sess = O.Session(m, synth.make_source(d.vocab_src, 5, seed=2))
    lp, ch, am = sess.score_batch([0, 0], [0, 2, 4], [5, 7, 7, 5])
    assert list(ch) == [1, 2, 2, 1] and lp[0] == lp[3] and lp[1] == lp[2]
    assert sess.rows_per_step == [1]
    lp2, ch2, _ = sess.score_batch([0], [0, 1], [7])  # cache hit: no new step, same id/value
    assert ch2[0] == 2 and lp2[0] == lp[1] and sess.n_steps == 1
    lp3, ch3, am3 = sess.score_batch([1, 0], [0, 0, 1], [9])  # zero-candidate parent is not stepped
    assert am3[0] == -1 and sess.nodes[1].stepped is False
    with pytest.raises(IndexError):
        sess.score_batch([0], [0, 1], [d.vocab_tgt])
    with pytest.raises(KeyError):
        sess.score_batch([999], [0, 1], [3])
    with pytest.raises(ValueError):
        O.encode(m, [])


# ------------------------------------------------------------------ ensemble
def test_ensemble_combine_invariants():
    rng = np.random.default_rng(0)
    L = scipy.special.log_softmax(rng.standard_normal((3, 20)), axis=1)
    single = L[0]
    assert np.max(np.abs(O.ensemble_combine([single] * 4, [0.25] * 4, 0) - single)) < 1e-15
    assert np.max(np.abs(O.ensemble_combine([single] * 4, [0.25] * 4, 1) - single)) < 1e-14
    w = [0.2, 0.5, 0.3]
    a = O.ensemble_combine(list(L), w, 1)
    b = O.ensemble_combine([L[2], L[0], L[1]], [w[2], w[0], w[1]], 1)
    assert np.max(np.abs(a - b)) < 1e-15
    ref = scipy.special.logsumexp(L + np.log(np.array(w))[:, None], axis=0)
    assert np.max(np.abs(a - ref)) < 1e-14


def test_average_params_is_the_elementwise_mean():
    """NMT-k-Avg: identities of the element-wise mean pin the oracle's averaging."""
    d = synth.TINY
    a, b, c = (synth.make_model(d, s) for s in (3, 4, 5))
    one = O.average_params([a])
    assert all(np.array_equal(one[k], a[k].astype(np.float64)) for k in a)          # k = 1: the model itself
    same = O.average_params([a, a, a, a])
    assert all(np.array_equal(same[k], a[k].astype(np.float64)) for k in a)         # identical members
    two = O.average_params([a, b])
    assert all(np.array_equal(two[k], (a[k].astype(np.float64) + b[k]) / 2) for k in a)  # exact in fp64
    p1, p2 = O.average_params([a, b, c]), O.average_params([c, a, b])               # order independent
    assert all(np.max(np.abs(p1[k] - p2[k])) <= 1e-15 * (1 + np.max(np.abs(p1[k]))) for k in a)
    with pytest.raises(ValueError):
        O.average_params([a, {k: v for k, v in b.items() if k != "decoder_U"}])


def test_topk_words_definition():
    """Beam expansion set (NEXT-3): brute force over every k-subset on tiny rows, ties -> lower id."""
    rng = np.random.default_rng(3)
    for trial in range(30):
        v = rng.integers(0, 4, size=7).astype(np.float64)  # many ties
        k = int(rng.integers(1, 7))
        got = list(O.topk_words(v, k))
        # brute force: the lexicographically smallest (by -value, index) k-subset ordering
        best = sorted(range(7), key=lambda i: (-v[i], i))[:k]
        assert got == best
        assert all(v[got[i]] >= v[got[i + 1]] for i in range(k - 1))
        worst_in = min(v[i] for i in got)
        assert all(v[j] <= worst_in for j in set(range(7)) - set(got))   # nothing outside beats the set
    v = rng.standard_normal(50)
    assert O.topk_words(v, 1)[0] == int(np.argmax(v))                    # k = 1 is the argmax
    assert list(O.topk_words(v, 50)) == list(np.argsort(-v))             # k = V is the full ranking


def test_beam_step_matches_full_rows():
    d = synth.TINY
    p = synth.make_model(d, 7)
    sess = O.Session(O.Model(d, p), synth.make_source(d.vocab_src, 4, seed=1))
    w, lp = sess.beam_step([sess.root], 5)
    full = sess.logprobs_full(sess.root)
    assert list(w[0]) == list(np.argsort(-full, kind="stable")[:5])
    assert np.allclose(lp[0], np.sort(full)[::-1][:5], rtol=0, atol=1e-15)


# ------------------------------------------------------------------ Fig. 1 worked example (golden)
def _read_fig1():
    hyps, info = {}, {}
    for ln in open(os.path.join(GOLD, "fig1_forest.txt")):
        ln = ln.strip()
        if not ln or ln.startswith("#"):
            continue
        if ln.startswith("hyp"):
            h, rest = ln[4:].split(":")
            hyps[int(h)] = [tuple(int(w[1:]) for w in ph.split()) for ph in rest.split("|")]
        else:
            k, *v = ln.split()
            info[k] = v
    return hyps, info


def test_fig1_forest_structure_and_scores():
    hyps, info = _read_fig1()
    pairs = [(h, t) for h in sorted(hyps) for t in hyps[h]]
    assert sum(len(t) for _, t in pairs) == int(info["naive_words"][0])
    levels = O.forest_levels(pairs)
    assert [len(l) for l in levels] == [int(x) for x in info["edges_per_depth"]]
    assert len(levels) == int(info["steps"][0])
    # first level rows: E_1 labels and H_0 source nodes in the paper's row order
    assert [f"w{w}" for (_, w) in levels[0]] == info["E1"]
    assert [f"h{src[0]}" for (src, _) in levels[0]] == info["H0"]
    # score through the oracle's state cache: one score_batch per depth, parent-indexed rows
    d, p, m = tiny_model(seed=21)
    sess = O.Session(m, synth.make_source(d.vocab_src, 5, seed=6))
    rng = np.random.default_rng(1)
    hyp_nodes = [sess.inject_state(np.tanh(rng.standard_normal(d.dim_hid)), y) for y in (4, 9)]
    word_id = lambda k: k + 2  # w_k -> token id k+2 (0/1 reserved for EOS/UNK)
    idpairs = [(h, tuple(word_id(w) for w in t)) for h, t in pairs]
    scores = O.score_forest(sess, hyp_nodes, idpairs)
    assert sess.n_steps == int(info["steps"][0])
    assert sess.rows_per_step == [int(x) for x in info["parent_rows_per_depth"]]
    for (h, t) in idpairs:
        n = sess.nodes[hyp_nodes[h]]
        ref, _, _ = O.score_sequence(m, sess.c, t, s=n.s_in, y_prev=n.word)
        assert abs(scores[(h, t)] - ref) < 1e-12


# ------------------------------------------------------------------ params container (synth I/O)
def test_params_container_roundtrip():
    d = TINY
    p = synth.make_model(d, 7)
    blob = synth.params_bytes(d, p)
    d2, q = synth.read_params(blob)
    assert d2 == d and set(q) == set(p)
    for k in p:
        assert np.array_equal(p[k], q[k])
    assert synth.params_bytes(d2, q) == blob
    assert synth.make_model(d, 7)["decoder_U"].tobytes() == p["decoder_U"].tobytes()
