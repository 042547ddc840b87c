"""ScoreBatch forest driver (Alg. 1) on the GPU path vs the float64 oracle, the Fig. 1 worked
example (tests/golden/fig1_forest.txt), C3-style stack-decoding batches and the
ensemble hook with a single-rank NCCL communicator."""
import os

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = {"fp32class": 1e-3, "bf16": 2e-2}


def _fig1():
    hyps, info = {}, {}
    for ln in open(os.path.join(GOLD, "fig1_forest.txt")):
        ln = ln.strip()
        if not ln or ln.startswith("#"):
            continue
        if ln.startswith("hyp"):
            h, rest = ln[4:].split(":")
            hyps[int(h)] = [tuple(int(w[1:]) + 2 for w in ph.split()) for ph in rest.split("|")]
        else:
            k, *v = ln.split()
            info[k] = v
    return [(h, t) for h in sorted(hyps) for t in hyps[h]], info


def _forest_args(pairs):
    off = np.cumsum([0] + [len(t) for _, t in pairs]).astype(np.int32)
    words = np.array([w for _, t in pairs for w in t], np.int32)
    return off, words


@pytest.mark.parametrize("prec", ["fp32class", "bf16"])
def test_stack_batch_dedup_tiny(prec):
    """C3-style stack through nmt_score_forest: distinct (h, t) expansions over zipf parents, phrase
    lengths 1..5, branching shrinking with depth.  Scores must match the oracle; the
    number of stepped rows is bounded by the edges, and a re-scored stack steps nothing."""
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(8, 16, 50, 50, "maxout")
    p = synth.make_model(d, 1605)
    M = nmt.Model(synth.params_bytes(d, p), precision=prec)
    src = synth.make_source(d.vocab_src, 12, seed=1606)
    ctx = M.encode(src)
    sess = O.Session(O.Model(d, p), src)
    H = 16
    s, y = synth.make_states(H, d.dim_hid, d.vocab_tgt, seed=1607)
    gh = ctx.inject_states(s, y)
    oh = [sess.inject_state(s[i], int(y[i])) for i in range(H)]
    pairs = synth.make_stack_expansions(120, H, d.vocab_tgt, seed=1608)
    off, words = _forest_args(pairs)
    lp, fin, st = ctx.score_forest([gh[h] for h, _ in pairs], off, words)
    ref = O.score_forest(sess, oh, pairs)
    worst = max(abs(lp[i] - ref[k]) / len(k[1]) for i, k in enumerate(pairs))
    assert worst < TOL[prec]
    assert sum(st["rows_per_depth"]) <= sum(st["edges_per_depth"]) <= len(words)
    assert st["steps"] == max(len(t) for _, t in pairs)
    assert st["rows_per_depth"] == sess.rows_per_step
    n0 = ctx.stats()
    lp2, fin2, st2 = ctx.score_forest([gh[h] for h, _ in pairs], off, words)  # cache: no new rows
    assert ctx.stats() == n0 and sum(st2["rows_per_depth"]) == 0
    assert np.array_equal(lp, lp2) and np.array_equal(fin, fin2)


def test_ensemble_single_rank_nccl():
    """nmt_ensemble_combine with one member (NCCL communicator of size 1) reproduces the oracle's
    combine of a single model: mode 0 = weight * logp, mode 1 = log(weight * p)."""
    import torch
    from paper_1605_04809_b200 import nmt
    uid = nmt.Ensemble.unique_id()
    ens = nmt.Ensemble(1, 0, uid, 0)
    rng = np.random.default_rng(0)
    lp = np.log(rng.dirichlet(np.ones(64), size=1)[0]).astype(np.float32)
    d_in = torch.from_numpy(lp).cuda()
    d_out = torch.empty_like(d_in)
    st = torch.cuda.current_stream().cuda_stream
    for mode, w in [(0, 1.0), (0, 0.25), (1, 1.0), (1, 0.5)]:
        ens.combine(d_in.data_ptr(), 64, w, mode, 0, d_out.data_ptr(), st)
        torch.cuda.synchronize()
        ref = O.ensemble_combine([lp.astype(np.float64)], [w], mode)
        assert np.max(np.abs(d_out.cpu().numpy() - ref)) < 1e-5
    ens.close()


@pytest.mark.parametrize("prec", ["fp32class", "bf16"])
def test_native_score_forest_matches_oracle_fig1(prec):
    """nmt_score_forest (native ScoreBatch) == oracle per-pair sums on the Fig. 1 worked example
    (tests/golden/fig1_forest.txt); Fig. 1 step structure (steps, edges per depth, parent rows per
    depth); a second call on the same pairs is served from the state cache (no new rows, identical
    results)."""
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(8, 16, 50, 50, "tanh")
    p = synth.make_model(d, 21)
    M = nmt.Model(synth.params_bytes(d, p), precision=prec)
    src = synth.make_source(d.vocab_src, 5, seed=6)
    rng = np.random.default_rng(1)
    s = np.tanh(rng.standard_normal((2, d.dim_hid))).astype(np.float32)
    pairs, info = _fig1()
    hs_idx = [h for h, _ in pairs]
    off = np.cumsum([0] + [len(t) for _, t in pairs]).astype(np.int32)
    words = np.array([w for _, t in pairs for w in t], np.int32)
    ctx = M.encode(src)
    hyps = ctx.inject_states(s, [4, 9])
    lp, stt, st = ctx.score_forest([hyps[h] for h in hs_idx], off, words)
    assert st["steps"] == int(info["steps"][0])
    assert st["edges_per_depth"] == [int(x) for x in info["edges_per_depth"]]
    assert st["rows_per_depth"] == [int(x) for x in info["parent_rows_per_depth"]]
    sess = O.Session(O.Model(d, p), src)
    oh = [sess.inject_state(s[i], y) for i, y in enumerate([4, 9])]
    ref = O.score_forest(sess, oh, pairs)
    for i, k in enumerate(pairs):
        assert abs(lp[i] - ref[k]) < TOL[prec] * len(k[1])
    lp2, st2, s2 = ctx.score_forest([hyps[h] for h in hs_idx], off, words)
    assert s2["rows_per_depth"] == [0, 0, 0, 0] and np.array_equal(lp, lp2) and np.array_equal(stt, st2)
    with pytest.raises(nmt.NmtError) as e:
        ctx.score_forest([hyps[0]], [0, 0], np.zeros(0, np.int32))
    assert "empty expansion" in str(e.value)


def test_native_score_forest_c3_stack_tiny():
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(8, 16, 50, 50, "maxout")
    p = synth.make_model(d, 1605)
    M = nmt.Model(synth.params_bytes(d, p), precision="fp32class")
    src = synth.make_source(d.vocab_src, 12, seed=1606)
    ctx = M.encode(src)
    sess = O.Session(O.Model(d, p), src)
    H = 16
    s, y = synth.make_states(H, d.dim_hid, d.vocab_tgt, seed=1607)
    gh = ctx.inject_states(s, y)
    oh = [sess.inject_state(s[i], int(y[i])) for i in range(H)]
    pairs = synth.make_stack_expansions(200, H, d.vocab_tgt, seed=1609)
    off = np.cumsum([0] + [len(t) for _, t in pairs]).astype(np.int32)
    words = np.array([w for _, t in pairs for w in t], np.int32)
    lp, _, st = ctx.score_forest([gh[h] for h, _ in pairs], off, words)
    ref = O.score_forest(sess, oh, pairs)
    worst = max(abs(lp[i] - ref[k]) / len(k[1]) for i, k in enumerate(pairs))
    assert worst < TOL["fp32class"]
    assert st["rows_per_depth"] == sess.rows_per_step


@pytest.mark.parametrize("prec", ["fp32class", "bf16"])
def test_score_sequences_nbest_vs_oracle(prec):
    """n-best forced rescoring (nmt_score_sequences, §8(f) NEXT-1): sequences longer than
    a phrase (up to 27 words + EOS) sharing prefixes, scored from the root in one forest; each total
    equals the oracle's chained sequence score (oracle.score_sequence), and the returned state
    continues exactly like the oracle state after the sequence."""
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(8, 16, 50, 50, "tanh")
    p = synth.make_model(d, 7)
    M = nmt.Model(synth.params_bytes(d, p), precision=prec)
    om = O.Model(d, p)
    src = synth.make_source(d.vocab_src, 6, seed=3)
    c = M.encode(src)
    oc = O.encode(om, src)
    rng = np.random.Generator(np.random.PCG64(9))
    base = [int(x) for x in rng.integers(2, d.vocab_tgt, size=27)]
    nbest = [base + [0], base[:20] + [5, 6, 0], base[:20] + [5, 7, 0], base[:3] + [0], [4, 0],
             [int(x) for x in rng.integers(2, d.vocab_tgt, size=18)] + [0]]
    lp, st = c.score_sequences(nbest)
    tol = 1e-3 if prec == "fp32class" else 2e-2
    for seq, g in zip(nbest, lp):
        ref, _, _ = O.score_sequence(om, oc, seq)
        assert abs(g - ref) < tol * len(seq) ** 0.5, (len(seq), g, ref)
    # shared prefixes were collapsed: the arena holds one node per distinct prefix (+ the root)
    prefixes = {tuple(s[:k]) for s in nbest for k in range(1, len(s) + 1)}
    assert c.stats()[0] == 1 + len(prefixes)
    # continuing from a returned state: same as the oracle from the state after the sequence
    lp2, _, _ = c.score_batch([int(st[4])], [0, 2], [3, 9])
    _, _, s_after = O.score_sequence(om, oc, nbest[4])
    out = O.step(om, oc, s_after[None, :], [nbest[4][-1]])
    ref2 = O.log_softmax(out["z"][0])[[3, 9]]
    assert np.max(np.abs(lp2 - ref2)) < tol
