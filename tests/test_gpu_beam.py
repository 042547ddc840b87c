"""Beam step (pure-NMT beam search on the same step) on the GPU
against the float64 oracle.  The k words are chosen from the vocabulary GEMM's logits in the model's
precision, so near-ties may legitimately differ from the float64 ranking: the test checks what is
unique (the exact log-probs of the returned words, order, child ids) and that the returned set is a
valid top-k within the precision bound (no word outside it beats it by more than 2 tol)."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
TOL = {"fp32class": 1e-3, "bf16": 2e-2}


def _check_rows(words, lp, refs, k, tol):
    for q, full in enumerate(refs):
        w = words[q]
        assert len(set(w.tolist())) == k                                  # distinct words
        assert np.all(np.diff(lp[q]) <= 0)                                 # descending log-prob
        assert np.max(np.abs(lp[q] - full[w])) < tol                       # exact scores of the set
        kth = np.sort(full)[::-1][k - 1]
        assert np.all(full[w] >= kth - 2 * tol)                            # a valid top-k set
        outside = np.setdiff1d(np.arange(len(full)), w)
        assert np.all(full[outside] <= full[w].min() + 2 * tol)


@pytest.mark.parametrize("prec", ["fp32class", "bf16"])
@pytest.mark.parametrize("readout", ["tanh", "maxout"])
def test_beam_step_tiny(prec, readout):
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(8, 16, 50, 50, readout)
    p = synth.make_model(d, 31)
    M = nmt.Model(synth.params_bytes(d, p), precision=prec)
    src = synth.make_source(d.vocab_src, 6, seed=2)
    ctx = M.encode(src)
    sess = O.Session(O.Model(d, p), src)
    s, y = synth.make_states(5, d.dim_hid, d.vocab_tgt, seed=9)
    gh = ctx.inject_states(s, y)
    oh = [sess.inject_state(s[i], int(y[i])) for i in range(5)]
    parents = [ctx.root] + list(gh)
    for k in (1, 4, 8):
        words, lp, child = ctx.beam_step(parents, k)
        refs = [sess.logprobs_full(0)] + [sess.logprobs_full(h) for h in oh]
        _check_rows(words, lp, refs, k, TOL[prec])
        # the same (parent, word) through nmt_score_batch: cache hits, bit-identical scores and children
        off = np.arange(0, len(parents) * k + 1, k, dtype=np.int32)
        lp2, ch2, am = ctx.score_batch(parents, off, words.reshape(-1))
        assert np.array_equal(lp2, lp.reshape(-1)) and np.array_equal(ch2, child.reshape(-1))
        if k == 1:  # top-1 is the fused argmax of the step (same logits, lowest index on ties)
            assert np.array_equal(words[:, 0], am)


@pytest.mark.parametrize("prec", ["fp32class", "bf16"])
def test_beam_step_enru_sampled(prec):
    """En->Ru dimensions (V = 100k): 300 injected parents, k = 8; 6 sampled rows against the oracle."""
    from paper_1605_04809_b200 import nmt
    d = synth.EN_RU
    p = synth.make_model(d, 2016)
    M = nmt.Model(synth.params_bytes(d, p), precision=prec)
    src = synth.make_source(d.vocab_src, 20, seed=4)
    ctx = M.encode(src)
    s, y = synth.make_states(300, d.dim_hid, d.vocab_tgt, seed=10)
    gh = ctx.inject_states(s, y)
    words, lp, child = ctx.beam_step(gh, 8)
    sess = O.Session(O.Model(d, p), src)
    rows = [0, 1, 77, 150, 298, 299]
    refs = [sess.logprobs_full(sess.inject_state(s[r], int(y[r]))) for r in rows]
    _check_rows(words[rows], lp[rows], refs, 8, TOL[prec])
    n0 = ctx.stats()
    words2, lp2, child2 = ctx.beam_step(gh, 8)  # everything cached now: same answer, no new nodes
    assert np.array_equal(words2, words) and np.array_equal(lp2, lp) and np.array_equal(child2, child)
    assert ctx.stats() == n0


def test_beam_step_errors():
    from paper_1605_04809_b200 import nmt
    d = synth.TINY
    M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 7)))
    ctx = M.encode(synth.make_source(d.vocab_src, 4, seed=1))
    with pytest.raises(nmt.NmtError) as e:
        ctx.beam_step([ctx.root], 9)
    assert e.value.name == "NMT_ERR_INVALID_ARG"
    with pytest.raises(nmt.NmtError) as e:
        ctx.beam_step([12345], 2)
    assert e.value.name == "NMT_ERR_BAD_STATE"
    w, lp, ch = ctx.beam_step([], 3)
    assert w.shape == (0, 3)
