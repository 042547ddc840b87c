"""Multi-rank paths on ONE GPU through the in-process ("local") communicator of the library: every
rank or ensemble member is its own model instance driven by its own host thread, and the exchange
runs through the same collective (all-gather) and the same kernels as the NCCL transport.

* Ensemble combine with M = 4 members (PAPER.md:92 separately weighted features; SURVEY §8(c) C4:
  "the combined output of one C2 batch, both combine modes") against oracle.ensemble_combine of the
  oracle's per-member log-probs.
* Vocab-parallel scoring (nmt_vocab_shard) with world = 2, 3, 4 ranks: the real
  run_step branch (slice GEMM -> all-gather of (max, sum exp, argmax) partials -> rank-order combine)
  against the unsharded model and the oracle."""
import threading

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
TOL = {"fp32class": 1e-3, "bf16": 2e-2}


def nmt():
    from paper_1605_04809_b200 import nmt as m
    return m


def run_ranks(fn, n):
    """fn(rank) in n threads (ctypes releases the GIL in library calls); re-raise the first error."""
    out, err = [None] * n, []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if err:
        raise err[0]
    assert not any(t.is_alive() for t in ts), "a rank thread hung"
    return out


def _combine_members(models, scorer, weights, modes, n_members):
    """Each member scores (scorer(rank, model) -> host log-probs), then every mode is combined to root 0
    over the local communicator; returns (member log-probs, {mode: combined})."""
    import torch
    comms = nmt().Ensemble.local(n_members)
    res = {}

    def member(r):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        lp = scorer(r, models[r])
        with torch.cuda.stream(st):
            d_in = torch.from_numpy(lp).cuda()
            out = {}
            for mode in modes:
                d_out = torch.full_like(d_in, float("nan")) if r == 0 else None
                comms[r].combine(d_in.data_ptr(), len(lp), weights[r], mode, 0,
                                 d_out.data_ptr() if d_out is not None else None, st.cuda_stream)
                if r == 0:
                    out[mode] = d_out
        st.synchronize()
        if r == 0:
            res.update({k: v.cpu().numpy() for k, v in out.items()})
        return lp

    lps = run_ranks(member, n_members)
    for c in comms:
        c.close()
    return lps, res


@pytest.mark.parametrize("prec", ["fp32class", "bf16"])
def test_local_ensemble_m4_tiny(prec):
    """4 different tiny members (C1 shapes), unequal weights, both modes, combined on the device vs the
    oracle's combine of the oracle's member log-probs; M identical members reduce to the single model."""
    d = synth.Dims(8, 16, 50, 50, "maxout")
    ps = [synth.make_model(d, 7 + m) for m in range(4)]
    models = [nmt().Model(synth.params_bytes(d, p), precision=prec) for p in ps]
    src = synth.make_source(d.vocab_src, 6, seed=2)
    par, off, words = [0], [0, 6], [5, 9, 2, 0, 1, 33]
    w = [0.4, 0.3, 0.2, 0.1]

    def scorer(r, M):
        c = M.encode(src)
        lp, _, _ = c.score_batch(par, off, words)
        # a second depth from real children (the cache and child states are per member)
        ch = c.score_batch(par, off, words)[1]
        lp2, _, _ = c.score_batch([int(ch[0]), int(ch[1])], [0, 2, 4], [3, 4, 5, 6])
        return np.concatenate([lp, lp2]).astype(np.float32)

    lps, comb = _combine_members(models, scorer, w, (0, 1), 4)
    ref_members = []
    for p in ps:
        sess = O.Session(O.Model(d, p), src)
        rl, rc, _ = sess.score_batch(par, off, words)
        rl2, _, _ = sess.score_batch([int(rc[0]), int(rc[1])], [0, 2, 4], [3, 4, 5, 6])
        ref_members.append(np.concatenate([rl, rl2]))
    for r in range(4):
        assert np.max(np.abs(lps[r] - ref_members[r])) < TOL[prec]
    for mode in (0, 1):
        ref = O.ensemble_combine(ref_members, w, mode)
        err = float(np.max(np.abs(comb[mode] - ref)))
        print(f"\n[ensemble m4 tiny {prec}] mode {mode}: max|d| = {err:.2e}")
        assert err < TOL[prec], (mode, err)
        # the device combine itself is exact up to fp32 output rounding on the members' own values
        own = O.ensemble_combine([x.astype(np.float64) for x in lps], w, mode)
        assert np.max(np.abs(comb[mode] - own)) < 1e-6
    # identical members with sum(w) = 1 combine to the single model (oracle invariant)
    same = [models[0]] * 4
    lps2, comb2 = _combine_members(same, scorer, [0.25] * 4, (0, 1), 4)
    for mode in (0, 1):
        assert np.max(np.abs(comb2[mode] - lps2[0])) < 1e-6


def test_local_ensemble_mode1_no_underflow():
    """Mode 1 is max-shifted: log-probs far below the fp32 exp range (-150) still combine exactly."""
    import torch
    comms = nmt().Ensemble.local(2)
    base = np.array([-150.0, -300.0, -1.0, -104.0], np.float32)
    vals = [base, base - 2.0]
    outs = {}

    def member(r):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            d_in = torch.from_numpy(vals[r]).cuda()
            d_out = torch.empty_like(d_in) if r == 0 else None
            comms[r].combine(d_in.data_ptr(), 4, 0.5, 1, 0, d_out.data_ptr() if r == 0 else None, st.cuda_stream)
        st.synchronize()
        if r == 0:
            outs[0] = d_out.cpu().numpy()

    run_ranks(member, 2)
    ref = O.ensemble_combine([v.astype(np.float64) for v in vals], [0.5, 0.5], 1)
    assert np.all(np.isfinite(outs[0]))
    assert np.max(np.abs(outs[0] - ref)) < 1e-4
    for c in comms:
        c.close()


@pytest.fixture(scope="module")
def c4_members():
    """C4: 4 members of the C2 bench model (maxout, E 500, H 1024, V 100k), seeds 2016..2019."""
    d = synth.Dims(500, 1024, 50000, 100000, "maxout")
    ps = [synth.make_model(d, 2016 + m) for m in range(4)]
    return d, ps


def test_c4_ensemble_m4_enru_sampled(c4_members):
    """C4: one C2 batch (R = 1024 parents x 3 candidates, Tx = 50) scored by 4 members
    on one GPU, combined with lambda = 1/4 (mode 0) and pi = 1/4 (mode 1); the combined log-probs of a
    sample of rows against the oracle ensemble of the four float64 models."""
    d, ps = c4_members
    models = [nmt().Model(synth.params_bytes(d, p), precision="bf16") for p in ps]
    src = synth.make_source(d.vocab_src, 49, seed=2016)
    R = 1024
    s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=2016)
    off, words = synth.make_candidates(R, 3, d.vocab_tgt, seed=2017)

    def scorer(r, M):
        c = M.encode(src)
        ids = c.inject_states(s, y)
        lp, _, _ = c.score_batch(ids, off, words)
        return lp

    lps, comb = _combine_members(models, scorer, [0.25] * 4, (0, 1), 4)
    rows = list(range(0, R, 97)) + [R - 1]
    ref_members = []
    for p in ps:
        om = O.Model(d, p)
        out = O.step(om, O.encode(om, src), s[rows].astype(np.float64), y[rows])
        ref_members.append(np.concatenate([O.log_softmax(out["z"][j])[words[off[r]:off[r + 1]]]
                                           for j, r in enumerate(rows)]))
    idx = np.concatenate([np.arange(off[r], off[r + 1]) for r in rows])
    for mode in (0, 1):
        ref = O.ensemble_combine(ref_members, [0.25] * 4, mode)
        err = float(np.max(np.abs(comb[mode][idx] - ref)))
        print(f"\n[C4 ensemble m4 En->Ru bf16] mode {mode}: sampled max|d| = {err:.2e} over {len(idx)} words")
        assert err < TOL["bf16"], (mode, err)


def _shard_run(blob, prec, world, src, s, y, off, words):
    models = [nmt().Model(blob, precision=prec) for _ in range(world)]
    comms = nmt().Ensemble.local(world)

    def rank(r):
        M = models[r]
        M.vocab_shard(r, world, comms[r])
        c = M.encode(src)
        ids = c.inject_states(s, y)
        lp, ch, am = c.score_batch(ids, off, words)
        lp2, ch2, am2 = c.score_batch(ch[: len(ch) // 2], np.arange(0, len(ch) // 2 + 1, dtype=np.int32),
                                      words[: len(ch) // 2])  # a second depth from real children
        return lp, ch, am, lp2, am2

    out = run_ranks(rank, world)
    for c in comms:
        c.close()
    return out


@pytest.mark.parametrize("prec", ["fp32class", "bf16"])
def test_vocab_shard_local_ranks_tiny(prec):
    """world = 2, 3, 4 vocab-parallel ranks on one GPU (V = 1000, Vp = 1024: 4 tiles) through the real
    step: every rank returns bit-identical results; they equal the unsharded model's (argmax, child
    ids) up to fp32 summation order (log-probs), and the oracle within the precision's bound."""
    d = synth.Dims(16, 32, 60, 1000, "maxout")
    p = synth.make_model(d, 5)
    blob = synth.params_bytes(d, p)
    src = synth.make_source(d.vocab_src, 9, seed=3)
    R = 37
    s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=4)
    off, words = synth.make_candidates(R, 3, d.vocab_tgt, seed=5)
    ref = _shard_run(blob, prec, 1, src, s, y, off, words)[0]
    sess = O.Session(O.Model(d, p), src)
    oids = [sess.inject_state(s[i], int(y[i])) for i in range(R)]
    rl, rc, ra = sess.score_batch(oids, off, words)
    for world in (2, 3, 4):
        outs = _shard_run(blob, prec, world, src, s, y, off, words)
        for r in range(1, world):
            for a, b in zip(outs[0], outs[r]):
                assert np.array_equal(a, b), (world, r)
        lp, ch, am, lp2, am2 = outs[0]
        assert np.array_equal(ch, ref[1]) and np.array_equal(am, ref[2]) and np.array_equal(am2, ref[4])
        assert np.max(np.abs(lp - ref[0])) < 1e-5 and np.max(np.abs(lp2 - ref[3])) < 1e-5
        assert np.array_equal(ch, rc)
        assert np.max(np.abs(lp - rl)) < TOL[prec]


def test_vocab_shard_local_ranks_enru():
    """4 vocab-parallel ranks at the En->Ru shape (V = 100k: 391 tiles, 97-98 per rank), R = 300 ragged
    batch, bf16: identical across ranks, argmax equal to the unsharded model, sampled oracle rows."""
    d = synth.EN_RU
    p = synth.make_model(d, 2016)
    blob = synth.params_bytes(d, p)
    src = synth.make_source(d.vocab_src, 49, seed=50)
    R = 300
    s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=7)
    off, words = synth.make_candidates(R, 3, d.vocab_tgt, seed=8)
    ref = _shard_run(blob, "bf16", 1, src, s, y, off, words)[0]
    outs = _shard_run(blob, "bf16", 4, src, s, y, off, words)
    for r in range(1, 4):
        assert all(np.array_equal(a, b) for a, b in zip(outs[0], outs[r]))
    lp, ch, am = outs[0][:3]
    assert np.array_equal(ch, ref[1]) and np.array_equal(am, ref[2])
    assert np.max(np.abs(lp - ref[0])) < 1e-4
    om = O.Model(d, p)
    rows = [0, 1, 150, 255, 256, 299]
    out = O.step(om, O.encode(om, src), s[rows].astype(np.float64), y[rows])
    worst = max(float(np.max(np.abs(lp[off[r]:off[r + 1]] - O.log_softmax(out["z"][j])[words[off[r]:off[r + 1]]])))
                for j, r in enumerate(rows))
    print(f"\n[vocab shard 4 ranks En->Ru bf16] sampled max|dlogp| = {worst:.2e}")
    assert worst < TOL["bf16"]
