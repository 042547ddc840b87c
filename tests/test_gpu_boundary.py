"""GPU tests of the remaining SURVEY §8(b) boundary calls: nmt_save_params / nmt_params_bytes
(byte-identical round trip), nmt_create_random (the library's generator, checked by
exporting its container to the float64 oracle), nmt_debug_vocab (D8 + D9 alone on given t, bounded
by the operand rounding of the vocabulary GEMM) and nmt_score_batch_multi (several sentences per
call, identical to per-context nmt_score_batch)."""
import os
import tempfile

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

TOL = {"fp32class": 1e-3, "bf16": 2e-2}
CONFIGS = [("tanh", "fp32class"), ("tanh", "bf16"), ("maxout", "fp32class"), ("maxout", "bf16")]


def nmt():
    from paper_1605_04809_b200 import nmt as m
    return m


@pytest.mark.parametrize("readout", ["tanh", "maxout"])
def test_save_params_round_trip(readout):
    d = synth.Dims(8, 16, 50, 60, readout)
    blob = synth.params_bytes(d, synth.make_model(d, 3))
    M = nmt().Model(blob, precision="bf16")
    assert M.params_bytes() == blob
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "m.params")
        M.save_params(path)
        assert open(path, "rb").read() == blob
        M2 = nmt().Model(path, precision="bf16")  # and the saved file loads again
        assert M2.params_bytes() == blob
    with pytest.raises(nmt().NmtError) as e:
        M.save_params("/nonexistent-dir/x.params")
    assert e.value.name == "NMT_ERR_IO"


@pytest.mark.parametrize("readout,prec", CONFIGS)
def test_create_random_vs_oracle(readout, prec):
    N = nmt()
    M = N.Model.create_random(8, 16, 50, 50, readout, seed=21, logit_std=1.5, precision=prec)
    blob = M.params_bytes()
    assert blob == N.random_params(8, 16, 50, 50, readout, seed=21, logit_std=1.5)
    d, p = synth.read_params(blob)
    om = O.Model(d, p)
    src = synth.make_source(d.vocab_src, 6, seed=4)
    c = M.encode(src)
    sess = O.Session(om, src)
    lp, ch, _ = c.score_batch([0], [0, 5], [2, 3, 4, 0, 1])
    rl, rc, _ = sess.score_batch([0], [0, 5], [2, 3, 4, 0, 1])
    assert list(ch) == list(rc)
    assert np.max(np.abs(lp - rl)) < TOL[prec]
    parents = [int(x) for x in ch]
    off = [0, 2, 4, 6, 8, 10]
    words = [5, 6, 7, 8, 9, 10, 11, 12, 13, 14]
    lp2, _, _ = c.score_batch(parents, off, words)
    rl2, _, _ = sess.score_batch(parents, off, words)
    assert np.max(np.abs(lp2 - rl2)) < TOL[prec]


def _vocab_case(d, p, M, prec, R, n_cand, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    scale = 1.0 if d.readout == "tanh" else 1.7
    t = (np.tanh(rng.standard_normal((R, d.dim_emb))) * scale).astype(np.float32)
    off = (np.arange(R + 1) * n_cand).astype(np.int32)
    words = rng.integers(0, d.vocab_tgt, size=R * n_cand).astype(np.int32)
    lp, lz, am = M.debug_vocab(t, off, words)
    W = p["ff_logit_W"].astype(np.float64)
    b = p["ff_logit_b"][0].astype(np.float64)
    t64 = t.astype(np.float64)
    z = t64 @ W + b
    ref_lz = O.logsumexp(z)
    # operand-rounding bound of the GEMM: bf16 t and W (2^-9 relative each) -> 2^-8 sum|t||W|;
    # bf16x3 (fp32class) drops the lo.lo term: ~2^-16 relative
    rel = 2.0 ** -8 if prec == "bf16" else 2.0 ** -15
    B = rel * (np.abs(t64) @ np.abs(W)) + 2e-5
    Bmax = B.max(axis=1)
    assert np.all(np.abs(lz - ref_lz) <= Bmax + 1e-4), float(np.max(np.abs(lz - ref_lz) - Bmax))
    for r in range(R):
        assert z[r, am[r]] >= z[r].max() - 2 * Bmax[r], r
    rows = np.repeat(np.arange(R), n_cand)
    ref = z[rows, words] - ref_lz[rows]
    err = np.abs(lp.astype(np.float64) - ref)
    assert np.all(err <= B[rows, words] + Bmax[rows] + 1e-4), float(err.max())
    return float(err.max()) if err.size else 0.0


@pytest.mark.parametrize("readout,prec", CONFIGS)
def test_debug_vocab_tiny(readout, prec):
    d = synth.Dims(8, 16, 50, 50, readout)
    p = synth.make_model(d, 7)
    M = nmt().Model(synth.params_bytes(d, p), precision=prec)
    _vocab_case(d, p, M, prec, 5, 4, seed=1)
    _vocab_case(d, p, M, prec, 1, 0, seed=2)  # no candidates: logZ / argmax only


@pytest.mark.parametrize("prec", ["bf16", "fp32class"])
def test_debug_vocab_enru(prec):
    """D8 + D9 at the north-star shape (K = 500, V = 100k) on 300 rows (2 tiles + a ragged tail)."""
    d = synth.EN_RU
    p = synth.make_model(d, 2016)
    M = nmt().Model(synth.params_bytes(d, p), precision=prec)
    err = _vocab_case(d, p, M, prec, 300, 3, seed=3)
    print(f"\n[debug_vocab] En->Ru {prec}: max|dlogp| = {err:.3e}")
    assert err < TOL[prec]


@pytest.mark.parametrize("readout,prec", CONFIGS)
def test_score_batch_multi(readout, prec):
    d = synth.Dims(8, 16, 50, 50, readout)
    p = synth.make_model(d, 7)
    om = O.Model(d, p)
    N = nmt()
    M = N.Model(synth.params_bytes(d, p), precision=prec)
    srcs = [synth.make_source(d.vocab_src, L, seed=30 + L) for L in (3, 7, 5)]
    cs = [M.encode(s) for s in srcs]
    sess = [O.Session(om, s) for s in srcs]
    # call 1: the three roots, interleaved with a repeated parent
    ctxs = [cs[1], cs[0], cs[2], cs[1]]
    par = [0, 0, 0, 0]
    off = [0, 2, 5, 6, 8]
    words = [4, 5, 6, 7, 8, 9, 4, 10]
    lp, ch, am = N.score_batch_multi(ctxs, par, off, words)
    idx = {id(c): i for i, c in enumerate(cs)}
    for k, c in enumerate(ctxs):
        s = sess[idx[id(c)]]
        rl, rc, ra = s.score_batch([par[k]], [0, off[k + 1] - off[k]], words[off[k]:off[k + 1]])
        assert list(ch[off[k]:off[k + 1]]) == list(rc)
        assert np.max(np.abs(lp[off[k]:off[k + 1]] - rl)) < TOL[prec]
    assert lp[0] == lp[6] and ch[0] == ch[6]  # same (ctx, parent, word): same handle, same bits
    # the same request streams through per-context nmt_score_batch on fresh contexts: identical
    # child ids and argmax; log-probs equal up to fp32 summation order (the fused step's split-K
    # factors and vocabulary runs depend on its total row count) in fp32class; in bf16 up to the
    # operand rounding of the two D5-D7 forms (single context: alpha . (ctx . W) with bf16 alpha and
    # ctx . W; multi-context: c . W with bf16 c, reading A30)
    fresh = [M.encode(s) for s in srcs]
    f1 = fresh[1].score_batch([0, 0], [0, 2, 4], [4, 5, 4, 10])
    f0 = fresh[0].score_batch([0], [0, 3], [6, 7, 8])
    f2 = fresh[2].score_batch([0], [0, 1], [9])
    at = 1e-4 if prec == "fp32class" else TOL[prec] / 4
    assert np.allclose(f1[0], lp[[0, 1, 6, 7]], atol=at) and np.array_equal(f1[1], ch[[0, 1, 6, 7]])
    assert np.allclose(f0[0], lp[2:5], atol=at) and np.allclose(f2[0], lp[5:6], atol=at)
    assert list(am) == [f1[2][0], f0[2][0], f2[2][0], f1[2][1]]
    # call 2: children of call 1 across contexts, against the oracle
    ctxs2 = [cs[0], cs[2], cs[1], cs[0]]
    par2 = [int(ch[2]), int(ch[5]), int(ch[0]), int(ch[3])]
    off2 = [0, 3, 4, 6, 9]
    words2 = [1, 2, 3, 4, 5, 6, 7, 8, 9]
    lp2, ch2, _ = N.score_batch_multi(ctxs2, par2, off2, words2)
    for k, c in enumerate(ctxs2):
        s = sess[idx[id(c)]]
        rl, rc, _ = s.score_batch([par2[k]], [0, off2[k + 1] - off2[k]], words2[off2[k]:off2[k + 1]])
        assert list(ch2[off2[k]:off2[k + 1]]) == list(rc)
        assert np.max(np.abs(lp2[off2[k]:off2[k + 1]] - rl)) < TOL[prec]
    with pytest.raises(N.NmtError) as e:
        N.score_batch_multi([cs[0]], [99], [0, 1], [3])
    assert e.value.name == "NMT_ERR_BAD_STATE"


@pytest.mark.parametrize("readout,prec", CONFIGS)
def test_score_batch_multi_many_contexts(readout, prec):
    """20 sentences in one fused step: ragged parent counts (groups padded to 4 rows), repeated and
    already-stepped parents (dead rows), parents without candidates; against the oracle."""
    d = synth.Dims(8, 16, 50, 50, readout)
    p = synth.make_model(d, 7)
    om = O.Model(d, p)
    N = nmt()
    M = N.Model(synth.params_bytes(d, p), precision=prec)
    rng = np.random.Generator(np.random.PCG64(44))
    srcs = [synth.make_source(d.vocab_src, int(rng.integers(1, 12)), seed=400 + i) for i in range(20)]
    cs = M.encode_batch(srcs)
    sess = [O.Session(om, s) for s in srcs]
    frontier = [[0] for _ in cs]
    worst = 0.0
    for call in range(3):
        ctxs, par, counts = [], [], []
        for _ in range(60):
            i = int(rng.integers(0, len(cs)))
            ctxs.append(i)
            par.append(int(rng.choice(frontier[i])))
            counts.append(int(rng.integers(0, 4)))
        off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        words = rng.integers(0, d.vocab_tgt, size=int(off[-1])).astype(np.int32)
        lp, ch, am = N.score_batch_multi([cs[i] for i in ctxs], par, off, words)
        # oracle: each context's entries as ONE nmt_score_batch-style call (the multi semantics)
        for i in sorted(set(ctxs), key=ctxs.index):
            ks = [k for k, j in enumerate(ctxs) if j == i]
            goff = np.concatenate([[0], np.cumsum([counts[k] for k in ks])]).astype(np.int32)
            gw = np.concatenate([words[off[k]:off[k + 1]] for k in ks]).astype(np.int32)
            rl, rc, ra = sess[i].score_batch([par[k] for k in ks], goff, gw)
            glp = np.concatenate([lp[off[k]:off[k + 1]] for k in ks])
            gch = np.concatenate([ch[off[k]:off[k + 1]] for k in ks])
            assert list(gch) == list(rc)
            assert [am[k] < 0 for k in ks] == list(ra < 0)
            if len(rl):
                worst = max(worst, float(np.max(np.abs(glp - rl))))
            frontier[i] = sorted(set(frontier[i]) | set(int(x) for x in rc))
    assert worst < TOL[prec], worst


@pytest.mark.parametrize("prec", ["bf16", "fp32class"])
def test_score_batch_multi_enru(prec):
    """8 En->Ru sentences x 40 injected parents x 2 words in one fused step, against the oracle on a
    sample of parents (every sentence)."""
    d = synth.EN_RU
    p = synth.make_model(d, 2016)
    om = O.Model(d, p)
    N = nmt()
    M = N.Model(synth.params_bytes(d, p), precision=prec)
    rng = np.random.Generator(np.random.PCG64(45))
    srcs = [synth.make_source(d.vocab_src, int(rng.integers(10, 50)), seed=500 + i) for i in range(8)]
    cs = M.encode_batch(srcs)
    s, y = synth.make_states(40, d.dim_hid, d.vocab_tgt, seed=46)
    ids = [c.inject_states(s, y) for c in cs]
    ctxs, par = [], []
    for k in range(40):
        for i in range(8):
            ctxs.append(cs[i])
            par.append(int(ids[i][k]))
    off, words = synth.make_candidates(len(par), 2, d.vocab_tgt, seed=47)
    lp, ch, am = N.score_batch_multi(ctxs, par, off, words)
    worst = 0.0
    for i in range(8):
        sess = O.Session(om, srcs[i])
        oid = [sess.inject_state(s[k], int(y[k])) for k in range(40)]
        for k in (0, 17, 39):
            q = k * 8 + i
            rl, rc, _ = sess.score_batch([oid[k]], [0, 2], words[off[q]:off[q + 1]])
            worst = max(worst, float(np.max(np.abs(lp[off[q]:off[q + 1]] - rl))))
    print(f"\n[score_batch_multi] En->Ru 8 x 40 {prec}: max|dlogp| = {worst:.3e}")
    assert worst < TOL[prec]


@pytest.mark.parametrize("prec", ["fp32class", "bf16"])
def test_vocab_shards_emulated(prec):
    """Vocab-parallel path (NEXT-2) emulated on one GPU: n slices of the vocabulary computed as ranks
    0..n-1 and merged by the post-all-gather combine give the unsharded logZ (fp32 summation order)
    and argmax, and logZ stays within the GEMM operand-rounding bound of the float64 oracle."""
    d = synth.Dims(16, 32, 60, 1000, "maxout")  # Vp = 1024: 4 tiles of 256 columns
    p = synth.make_model(d, 5)
    M = nmt().Model(synth.params_bytes(d, p), precision=prec)
    rng = np.random.Generator(np.random.PCG64(8))
    t = (np.tanh(rng.standard_normal((37, d.dim_emb))) * 1.7).astype(np.float32)
    _, lz_full, am_full = M.debug_vocab(t, np.zeros(38, np.int32), np.zeros(0, np.int32))
    z = t.astype(np.float64) @ p["ff_logit_W"].astype(np.float64) + p["ff_logit_b"][0]
    rel = 2.0 ** -8 if prec == "bf16" else 2.0 ** -15
    B = (rel * (np.abs(t.astype(np.float64)) @ np.abs(p["ff_logit_W"].astype(np.float64)))).max(axis=1) + 1e-4
    for n in (1, 2, 3, 4):
        lz, am = M.debug_vocab_shards(t, n)
        assert np.allclose(lz, lz_full, atol=1e-5, rtol=1e-6), n
        assert np.array_equal(am, am_full), n
        assert np.all(np.abs(lz - O.logsumexp(z)) <= B), n
    with pytest.raises(nmt().NmtError):
        M.debug_vocab_shards(t, 5)  # more slices than 256-column tiles


def test_vocab_shards_emulated_enru():
    d = synth.EN_RU
    p = synth.make_model(d, 2016)
    M = nmt().Model(synth.params_bytes(d, p), precision="bf16")
    rng = np.random.Generator(np.random.PCG64(9))
    t = (np.tanh(rng.standard_normal((300, d.dim_emb))) * 1.7).astype(np.float32)
    _, lz_full, am_full = M.debug_vocab(t, np.zeros(301, np.int32), np.zeros(0, np.int32))
    for n in (2, 8):
        lz, am = M.debug_vocab_shards(t, n)
        assert np.allclose(lz, lz_full, atol=1e-5, rtol=1e-6), n
        assert np.array_equal(am, am_full), n


def test_vocab_shard_single_rank_and_errors():
    """world == 1 (single-rank NCCL communicator) keeps the full vocabulary; mismatched rank/world is
    rejected."""
    N = nmt()
    d = synth.Dims(8, 16, 50, 50, "tanh")
    p = synth.make_model(d, 7)
    M = N.Model(synth.params_bytes(d, p), precision="fp32class")
    uid = N.Ensemble.unique_id()
    comm = N.Ensemble(1, 0, uid, 0)
    src = synth.make_source(d.vocab_src, 4, seed=1)
    ref = M.encode(src).score_batch([0], [0, 3], [5, 9, 2])[0]
    M.vocab_shard(0, 1, comm)
    got = M.encode(src).score_batch([0], [0, 3], [5, 9, 2])[0]
    assert np.array_equal(ref, got)
    with pytest.raises(N.NmtError) as e:
        M.vocab_shard(1, 2, comm)  # the communicator has one rank
    assert e.value.name == "NMT_ERR_INVALID_ARG"
    with pytest.raises(N.NmtError):
        M.vocab_shard(2, 2, None)
    comm.close()


@pytest.mark.parametrize("readout,prec", CONFIGS)
def test_score_forest_multi_vs_oracle(readout, prec):
    """nmt_score_forest_multi: expansions of 5 sentences (shared prefixes, lengths 1-20) in one call;
    each summed log-prob equals the oracle's forest score of its sentence, final states continue like
    the oracle's, and per-context node counts equal the distinct prefixes."""
    d = synth.Dims(8, 16, 50, 50, readout)
    p = synth.make_model(d, 7)
    om = O.Model(d, p)
    N = nmt()
    M = N.Model(synth.params_bytes(d, p), precision=prec)
    rng = np.random.Generator(np.random.PCG64(61))
    srcs = [synth.make_source(d.vocab_src, int(rng.integers(2, 9)), seed=600 + i) for i in range(5)]
    cs = M.encode_batch(srcs)
    sess = [O.Session(om, s) for s in srcs]
    ctxs, hyps, phrases = [], [], []
    for i in range(5):
        base = [int(x) for x in rng.integers(0, d.vocab_tgt, size=20)]
        for L in (1, 3, 3, 7, 20):
            ph = base[:L] if L != 3 or not phrases or phrases[-1] != base[:3] else base[:2] + [5]
            ctxs.append(cs[i])
            hyps.append(0)
            phrases.append(ph)
    off = np.concatenate([[0], np.cumsum([len(x) for x in phrases])]).astype(np.int32)
    words = np.concatenate(phrases).astype(np.int32)
    order = rng.permutation(len(phrases))  # interleave the sentences
    lp, st = N.score_forest_multi([ctxs[k] for k in order], [hyps[k] for k in order],
                                  np.concatenate([[0], np.cumsum([len(phrases[k]) for k in order])]).astype(np.int32),
                                  np.concatenate([phrases[k] for k in order]).astype(np.int32))
    tol = TOL[prec]
    for j, k in enumerate(order):
        i = [id(c) for c in cs].index(id(ctxs[k]))
        ref, _, _ = O.score_sequence(om, sess[i].c, phrases[k])
        assert abs(lp[j] - ref) < tol * len(phrases[k]) ** 0.5, (k, lp[j], ref)
    for i in range(5):
        prefixes = {tuple(ph[:L]) for k, ph in enumerate(phrases) if ctxs[k] is cs[i] for L in range(1, len(ph) + 1)}
        assert cs[i].stats()[0] == 1 + len(prefixes)
