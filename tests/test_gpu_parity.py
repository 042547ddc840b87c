"""GPU (libnmt.so through the C ABI) vs the float64 oracle on identical seeded inputs.

Bounds (BASELINE.json north_star): max |dlogp| <= 1e-3 for NMT_PREC_FP32CLASS, <= 2e-2 for NMT_PREC_BF16;
top-1 identical under the margin rule of DESIGN.md §2 A21 (the GPU's argmax must lie in the oracle's
tie set {w : logp_oracle(w) >= max - 2 tol}); child ids (integer state-cache work) bit-exact."""
import math

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

TOL = {"fp32class": 1e-3, "bf16": 2e-2}


def nmt():
    from paper_1605_04809_b200 import nmt as m
    return m


def check_top1(om_logfull_rows, gpu_argmax, tol):
    """om_logfull_rows: oracle full log-prob rows [n, V] (or z rows)."""
    for row, g in zip(om_logfull_rows, gpu_argmax):
        assert row[g] >= row.max() - 2 * tol, (int(np.argmax(row)), int(g), float(row.max() - row[g]))


# ------------------------------------------------------------------------------------------ tiny (C1)
CONFIGS = [("tanh", "fp32class"), ("tanh", "bf16"), ("maxout", "fp32class"), ("maxout", "bf16")]


@pytest.fixture(scope="module", params=CONFIGS, ids=["-".join(c) for c in CONFIGS])
def tiny(request):
    readout, prec = request.param
    d = synth.Dims(8, 16, 50, 50, readout)
    p = synth.make_model(d, 7)
    return d, p, nmt().Model(synth.params_bytes(d, p), precision=prec), O.Model(d, p), prec


def test_tiny_encoder(tiny):
    d, p, M, om, prec = tiny
    src = synth.make_source(d.vocab_src, 4, seed=1)
    ctx, pctx, s0 = M.encode(src).debug_encoder()
    ref = O.encode(om, src)
    assert np.max(np.abs(ctx - ref.ctx)) < 1e-4
    if prec == "fp32class":
        assert np.max(np.abs(pctx - ref.pctx)) < 1e-4
    else:  # single-pass bf16 keys: both operands rounded to bf16 (2^-9 each), fp32 accumulation
        bound = 2.0 ** -8 * (np.abs(ref.ctx) @ np.abs(p["decoder_Wc_att"])) + 1e-5
        assert np.all(np.abs(pctx - ref.pctx) <= bound)
    assert np.max(np.abs(s0 - ref.s0)) < 1e-4


def test_tiny_intermediates(tiny):
    d, p, M, om, prec = tiny
    src = synth.make_source(d.vocab_src, 4, seed=1)
    c = M.encode(src)
    sess = O.Session(om, src)
    g = c.debug_intermediates(c.root)
    r = sess.intermediates(0)
    tol = {"fp32class": 2e-4, "bf16": 2e-2}[prec]
    for k in ("s1", "alpha", "c", "s2", "t"):
        assert np.max(np.abs(g[k] - r[k])) < tol, k
    assert abs(g["logZ"][0] - r["logZ"]) < TOL[prec]


def test_tiny_c1_batch_and_cache(tiny):
    """C1: 1 source of 5 tokens, 4 parents (root + 3 nodes from a real prior step) x 3 candidates."""
    d, p, M, om, prec = tiny
    src = synth.make_source(d.vocab_src, 4, seed=1)
    c = M.encode(src)
    sess = O.Session(om, src)
    lp1, ch1, am1 = c.score_batch([0], [0, 3], [5, 9, 2])
    rl1, rc1, ra1 = sess.score_batch([0], [0, 3], [5, 9, 2])
    assert list(ch1) == list(rc1)
    assert np.max(np.abs(lp1 - rl1)) < TOL[prec]
    parents = [0] + [int(x) for x in ch1]
    words = [7, 5, 11, 3, 3, 4, 20, 21, 22, 9, 1, 0]
    off = [0, 3, 6, 9, 12]
    lp, ch, am = c.score_batch(parents, off, words)
    rl, rc, ra = sess.score_batch(parents, off, words)
    assert list(ch) == list(rc)
    assert np.max(np.abs(lp - rl)) < TOL[prec]
    assert lp[1] == lp1[0]  # (root, 5) is a cache hit: same child, bit-identical log-prob
    check_top1([sess.logprobs_full(pp) for pp in parents], am, TOL[prec])
    n_nodes, n_stepped = c.stats()
    assert n_nodes == len(sess.nodes) and n_stepped == sum(n.stepped for n in sess.nodes)


def test_tiny_full_row_normalised_and_matches(tiny):
    d, p, M, om, prec = tiny
    src = synth.make_source(d.vocab_src, 4, seed=2)
    c = M.encode(src)
    sess = O.Session(om, src)
    g = c.logprobs_full(c.root)
    r = sess.logprobs_full(0)
    # logZ comes from the (bf16 / bf16x3) vocabulary GEMM, the numerators from the fp32 gather-dot
    assert abs(np.exp(g.astype(np.float64)).sum() - 1) < TOL[prec]
    assert np.max(np.abs(g - r)) < TOL[prec]


def test_tiny_random_trees_vs_oracle(tiny):
    """Random interleaved depth-by-depth scoring with duplicate parents/words in a call: the device
    state cache must assign the oracle's ids and reuse cached states (A13/A14 readings)."""
    d, p, M, om, prec = tiny
    src = synth.make_source(d.vocab_src, 6, seed=3)
    c = M.encode(src)
    sess = O.Session(om, src)
    rng = np.random.default_rng(0)
    frontier = [0]
    worst = 0.0
    for it in range(12):
        k = int(rng.integers(1, 6))
        parents = [int(x) for x in rng.choice(frontier, size=k)]
        counts = rng.integers(0, 4, size=k)
        off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        words = [int(x) for x in rng.integers(0, d.vocab_tgt, size=int(off[-1]))]
        lp, ch, am = c.score_batch(parents, off, words)
        rl, rc, ra = sess.score_batch(parents, off, words)
        assert list(ch) == list(rc)
        assert list(am < 0) == list(ra < 0)
        if len(lp):
            worst = max(worst, float(np.max(np.abs(lp - rl))))
        frontier = sorted(set(frontier) | set(int(x) for x in ch))
    assert worst < TOL[prec]


def test_tiny_errors(tiny):
    d, p, M, om, prec = tiny
    N = nmt()
    with pytest.raises(N.NmtError) as e:
        M.encode([])
    assert e.value.name == "NMT_ERR_EMPTY_SOURCE"
    with pytest.raises(N.NmtError) as e:
        M.encode([1] * 65)
    assert e.value.name == "NMT_ERR_CAPACITY"
    with pytest.raises(N.NmtError) as e:
        M.encode([d.vocab_src])
    assert e.value.name == "NMT_ERR_TOKEN_RANGE"
    c = M.encode([3, 0])
    with pytest.raises(N.NmtError) as e:
        c.score_batch([0], [0, 1], [d.vocab_tgt])
    assert e.value.name == "NMT_ERR_TOKEN_RANGE"
    with pytest.raises(N.NmtError) as e:
        c.score_batch([5], [0, 1], [3])
    assert e.value.name == "NMT_ERR_BAD_STATE"
    lp, ch, am = c.score_batch([0], [0, 0], [])  # zero candidates: nothing stepped
    assert len(lp) == 0 and am[0] == -1 and c.stats() == (1, 0)


# ------------------------------------------------------------------------------------------ En->Ru shape (C2)
@pytest.fixture(scope="module")
def enru():
    d = synth.EN_RU
    p = synth.make_model(d, 2016)
    return d, p, synth.params_bytes(d, p), O.Model(d, p)


@pytest.mark.parametrize("prec", ["bf16", "fp32class"])
def test_enru_ragged_batch_vs_oracle(enru, prec):
    """R = 300 unique parents (2 full 128-row tiles + a ragged tail), Tx = 50, V = 100k, 3 candidates."""
    d, p, blob, om = enru
    M = nmt().Model(blob, precision=prec)
    src = synth.make_source(d.vocab_src, 49, seed=50)
    c = M.encode(src)
    sess = O.Session(om, src)
    g_ctx, g_pctx, g_s0 = c.debug_encoder()
    assert np.max(np.abs(g_ctx - sess.c.ctx)) < 1e-4
    assert np.max(np.abs(g_s0 - sess.c.s0)) < 1e-4
    R = 300
    s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=7)
    y[::17] = -1  # some BOS rows
    gids = c.inject_states(s, y)
    oids = [sess.inject_state(s[i], int(y[i])) for i in range(R)]
    assert list(gids) == oids
    off, words = synth.make_candidates(R, 3, d.vocab_tgt, seed=8)
    lp, ch, am = c.score_batch(gids, off, words)
    rl, rc, ra = sess.score_batch(oids, off, words)
    assert list(ch) == list(rc)
    err = np.abs(lp.astype(np.float64) - rl)
    print(f"\n[parity] En->Ru R={R} {prec}: max|dlogp| = {err.max():.3e}, mean = {err.mean():.3e}")
    assert err.max() < TOL[prec], float(err.max())
    zrows = []
    for i in range(0, R, 10):  # top-1 margin rule on a sample of rows
        n = sess.nodes[oids[i]]
        out = O.step(om, sess.c, n.s_in[None, :], [n.word])
        zrows.append(O.log_softmax(out["z"][0]))
    check_top1(zrows, am[::10], TOL[prec])


@pytest.fixture(scope="module")
def bench_model():
    """Exactly the bench.py model: E 500, H 1024, V_s 50k, V_t 100k, MAXOUT readout, seed 2016."""
    d = synth.Dims(500, 1024, 50000, 100000, "maxout")
    p = synth.make_model(d, 2016)
    return d, p, synth.params_bytes(d, p), O.Model(d, p)


@pytest.mark.parametrize("prec", ["bf16", "fp32class"])
def test_bench_config_sampled(bench_model, prec):
    """The bench.py launch configuration (R = 1024 parents x 3 candidates, maxout, Tx = 50) checked on
    a sample of rows the oracle computes one by one (rows are independent)."""
    d, p, blob, om = bench_model
    M = nmt().Model(blob, precision=prec)
    src = synth.make_source(d.vocab_src, 49, seed=2016)
    c = M.encode(src)
    R = 1024
    s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=2016)
    gids = c.inject_states(s, y)
    off, words = synth.make_candidates(R, 3, d.vocab_tgt, seed=2017)
    lp, ch, am = c.score_batch(gids, off, words)
    ctx = O.encode(om, src)
    rows = list(range(0, R, 37)) + [R - 1]
    out = O.step(om, ctx, s[rows].astype(np.float64), y[rows])
    worst = 0.0
    for j, r in enumerate(rows):
        lsm = O.log_softmax(out["z"][j])
        for i in range(off[r], off[r + 1]):
            worst = max(worst, abs(float(lp[i]) - lsm[words[i]]))
        assert lsm[am[r]] >= lsm.max() - 2 * TOL[prec]
    print(f"\n[parity] bench config R=1024 maxout {prec} (sampled rows): max|dlogp| = {worst:.3e}")
    assert worst < TOL[prec], worst
    assert len(set(ch.tolist())) == len(ch)


def test_tiny_max_source_length(tiny):
    """Tx = max_src_len (64 by default): the longest source the context accepts, encoded and scored
    against the oracle (the attention softmax over 64 positions, the encoder's full smem staging)."""
    d, p, M, om, prec = tiny
    src = synth.make_source(d.vocab_src, 63, seed=64)
    assert len(src) == 64
    c = M.encode(src)
    sess = O.Session(om, src)
    lp, ch, _ = c.score_batch([0], [0, 4], [3, 7, 0, 1])
    rl, rc, _ = sess.score_batch([0], [0, 4], [3, 7, 0, 1])
    assert list(ch) == list(rc)
    assert np.max(np.abs(lp - rl)) < TOL[prec]


@pytest.mark.parametrize("prec", ["bf16"])
def test_enru_large_batch_sampled(enru, prec):
    """R = 8192 unique parents x 2 words at the En->Ru shape (the top of bench's batch sweep): a
    sample of rows against the oracle, every log-prob finite and <= 0, child ids distinct."""
    d, p, blob, om = enru
    M = nmt().Model(blob, precision=prec)
    src = synth.make_source(d.vocab_src, 29, seed=81)
    c = M.encode(src)
    R = 8192
    s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=82)
    ids = c.inject_states(s, y)
    off, words = synth.make_candidates(R, 2, d.vocab_tgt, seed=83)
    lp, ch, am = c.score_batch(ids, off, words)
    assert np.all(np.isfinite(lp)) and np.all(lp <= 0)
    assert len(set(ch.tolist())) == len(ch)
    sess = O.Session(om, src)
    worst = 0.0
    for i in (0, 1, 4095, 4096, 8190, 8191):
        oid = sess.inject_state(s[i], int(y[i]))
        rl, _, _ = sess.score_batch([oid], [0, 2], words[off[i]:off[i + 1]])
        worst = max(worst, float(np.max(np.abs(lp[off[i]:off[i + 1]] - rl))))
    print(f"\n[parity] En->Ru R={R} {prec}: sampled max|dlogp| = {worst:.3e}")
    assert worst < TOL[prec]


# ------------------------------------------------------------------------ irregular shapes (padding)
@pytest.mark.parametrize("readout,prec", CONFIGS, ids=["-".join(c) for c in CONFIGS])
def test_irregular_dims_two_steps(readout, prec):
    """Dimensions that are multiples of nothing (E 13, H 37, V_s 61, V_t 517, Tx 23 and 67 rows): every
    padded extent - Hp, Cp, Ep, ROp, Vp, the E7 operand's rows, the projected-context K range, the encoder's
    units per CTA and its exchange words past H - against the oracle, over a two-step tree."""
    d = synth.Dims(13, 37, 61, 517, readout)
    p = synth.make_model(d, 11)
    om = O.Model(d, p)
    M = nmt().Model(synth.params_bytes(d, p), precision=prec)
    src = synth.make_source(d.vocab_src, 22, seed=5)
    c = M.encode(src)
    sess = O.Session(om, src)
    ctx, _, s0 = c.debug_encoder()
    ref = O.encode(om, src)
    assert np.max(np.abs(ctx - ref.ctx)) < 1e-4 and np.max(np.abs(s0 - ref.s0)) < 1e-4
    rng = np.random.default_rng(3)
    w1 = [int(x) for x in rng.choice(d.vocab_tgt, size=9, replace=False)]
    lp1, ch1, am1 = c.score_batch([0], [0, 9], w1)
    rl1, rc1, _ = sess.score_batch([0], [0, 9], w1)
    assert list(ch1) == list(rc1)
    parents = [int(x) for x in ch1] * 7 + [0]  # 64 parents, duplicates and the (stepped) root
    off = [0]
    words = []
    for _ in parents:
        k = int(rng.integers(1, 5))
        words += [int(x) for x in rng.choice(d.vocab_tgt, size=k, replace=False)]
        off.append(len(words))
    lp, ch, am = c.score_batch(parents, off, words)
    rl, rc, ra = sess.score_batch(parents, off, words)
    assert list(ch) == list(rc)
    err = max(float(np.max(np.abs(lp1 - rl1))), float(np.max(np.abs(lp - rl))))
    print(f"\n[irregular {readout}-{prec}] max|dlogp| = {err:.2e}")
    assert err < TOL[prec]
