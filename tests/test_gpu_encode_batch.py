"""nmt_encode_batch (§8(a) E1-E7 for many sentences at once) against the float64
oracle's per-sentence encoder (oracle.encode, "one context per sentence").

The batched path advances all recurrences together with one tensor-core GEMM per time step, so
sentences of different lengths share GEMMs while each keeps its own backward start (h_{Tx} = 0 at
its own last token).  Bounds: ctx / s0 within 2e-4 (fp32class: bf16x3 operands, fp32 accumulate)
or 3e-2 (bf16: single-pass bf16 recurrence, SURVEY App. A "encoder alone": max|dctx| 9.1e-3);
per-word log-probs of contexts built this way within the north-star tolerance (1e-3 / 2e-2)."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

TOL = {"fp32class": 1e-3, "bf16": 2e-2}
CTX_TOL = {"fp32class": 2e-4, "bf16": 3e-2}


def nmt():
    from paper_1605_04809_b200 import nmt as m
    return m


CONFIGS = [("tanh", "fp32class"), ("tanh", "bf16"), ("maxout", "fp32class"), ("maxout", "bf16")]


@pytest.fixture(scope="module", params=CONFIGS, ids=["-".join(c) for c in CONFIGS])
def tiny(request):
    readout, prec = request.param
    d = synth.Dims(8, 16, 50, 50, readout)
    p = synth.make_model(d, 7)
    return d, p, nmt().Model(synth.params_bytes(d, p), precision=prec), O.Model(d, p), prec


def _sources(vocab, lengths, seed):
    return [synth.make_source(vocab, L - 1, seed=seed + i) for i, L in enumerate(lengths)]


@pytest.mark.parametrize("lengths", [[5, 1, 8, 3, 3, 12, 2, 7, 7, 9, 4, 6],  # batched path (> 8 sentences)
                                     [4, 1, 9]])                             # small-n path (per sentence)
def test_tiny_encode_batch_vs_oracle(tiny, lengths):
    d, p, M, om, prec = tiny
    # ragged, a 1-token source (EOS only), equal lengths
    srcs = _sources(d.vocab_src, lengths, 100)
    cs = M.encode_batch(srcs)
    assert len(cs) == len(srcs)
    for src, c in zip(srcs, cs):
        ref = O.encode(om, src)
        ctx, pctx, s0 = c.debug_encoder()
        assert ctx.shape == ref.ctx.shape
        assert np.max(np.abs(ctx - ref.ctx)) < CTX_TOL[prec]
        assert np.max(np.abs(s0 - ref.s0)) < CTX_TOL[prec]
        # scoring on the batched context: root x 4 words, then one child x 3 words
        sess = O.Session(om, src)
        lp, ch, _ = c.score_batch([0], [0, 4], [3, 7, 0, 1])
        rl, rc, _ = sess.score_batch([0], [0, 4], [3, 7, 0, 1])
        assert list(ch) == list(rc)
        assert np.max(np.abs(lp - rl)) < TOL[prec]
        lp2, _, _ = c.score_batch([int(ch[0])], [0, 3], [5, 9, 2])
        rl2, _, _ = sess.score_batch([int(rc[0])], [0, 3], [5, 9, 2])
        assert np.max(np.abs(lp2 - rl2)) < TOL[prec]


def test_tiny_encode_batch_matches_single(tiny):
    d, p, M, om, prec = tiny
    srcs = _sources(d.vocab_src, [6, 4, 5, 3, 8, 2, 7, 6, 5, 4], 200)  # > 8: the batched path
    cs = M.encode_batch(srcs)
    for src, c in zip(srcs, cs):
        a = c.debug_encoder()
        b = M.encode(src).debug_encoder()
        for x, y in zip(a, b):
            assert np.max(np.abs(x - y)) < 2 * CTX_TOL[prec]


def test_tiny_encode_batch_errors(tiny):
    d, p, M, om, prec = tiny
    N = nmt()
    assert M.encode_batch([]) == []
    with pytest.raises(N.NmtError) as e:
        M.encode_batch([[3, 0], []])
    assert e.value.name == "NMT_ERR_EMPTY_SOURCE" and "sentence 1" in str(e.value)
    with pytest.raises(N.NmtError) as e:
        M.encode_batch([[3, 0], [2, d.vocab_src, 0]])
    assert e.value.name == "NMT_ERR_TOKEN_RANGE"
    with pytest.raises(N.NmtError) as e:
        M.encode_batch([[2] * 65])
    assert e.value.name == "NMT_ERR_CAPACITY"
    # the model still works after the rejected calls
    c = M.encode_batch([[4, 0]])[0]
    assert c.score_batch([0], [0, 1], [3])[1][0] == 1


@pytest.mark.parametrize("prec", ["bf16", "fp32class"])
def test_enru_encode_batch_vs_oracle(prec):
    """300 sentences of U[10, 50] tokens (two 128-row tiles + a ragged tail of GEMM rows, shrinking
    as sentences finish), En->Ru shape (E 500, H 1024, V_s 50k, V_t 100k)."""
    d = synth.EN_RU
    p = synth.make_model(d, 2016)
    om = O.Model(d, p)
    M = nmt().Model(synth.params_bytes(d, p), precision=prec)
    rng = np.random.Generator(np.random.PCG64(3000))
    lengths = [int(x) for x in rng.integers(10, 51, size=300)]
    srcs = _sources(d.vocab_src, lengths, 5000)
    cs = M.encode_batch(srcs)
    worst = 0.0
    for i in range(0, 300, 7):
        ref = O.encode(om, srcs[i])
        ctx, pctx, s0 = cs[i].debug_encoder()
        worst = max(worst, float(np.max(np.abs(ctx - ref.ctx))), float(np.max(np.abs(s0 - ref.s0))))
    print(f"\n[encode_batch] En->Ru n=300 {prec}: max|dctx|,|ds0| = {worst:.3e}")
    assert worst < CTX_TOL[prec]
    err = 0.0
    for i in (0, 77, 299):
        sess = O.Session(om, srcs[i])
        off, words = synth.make_candidates(1, 3, d.vocab_tgt, seed=i)
        lp, _, _ = cs[i].score_batch([0], off, words)
        rl, _, _ = sess.score_batch([0], off, words)
        err = max(err, float(np.max(np.abs(lp - rl))))
    print(f"[encode_batch] root scores max|dlogp| = {err:.3e}")
    assert err < TOL[prec]
