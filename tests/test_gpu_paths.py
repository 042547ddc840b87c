"""The paths the bench numbers come from, checked against the oracle (VERDICT r01 "Next round" 2):

* the device-resident calls bench.py times (nmt_encode_dev -> nmt_inject_states_dev ->
  nmt_score_batch_dev) equal the host C ABI bit for bit on the same inputs, and the oracle on a sample;
* run-to-run determinism on fresh models and contexts (SURVEY §8(b) "Identical call sequences give
  bit-identical outputs"; PAPER.md:263 rescoring "the same as if they were produced at decode-time");
* C3 at its real shape (Ru->En, V_s 100k, V_t 50k; a 4096-expansion stack through nmt_score_forest,
  PAPER.md:187, :260) with sampled pairs against the oracle's uncached sequential scorer."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
TOL = {"fp32class": 1e-3, "bf16": 2e-2}


def nmt():
    from paper_1605_04809_b200 import nmt as m
    return m


@pytest.fixture(scope="module")
def bench_model():
    """The bench.py model: E 500, H 1024, V_s 50k, V_t 100k, maxout, seed 2016."""
    d = synth.Dims(500, 1024, 50000, 100000, "maxout")
    p = synth.make_model(d, 2016)
    return d, p, synth.params_bytes(d, p)


def _c2_inputs(d, seed, R=1024, cands=3, Tx=50):
    src = synth.make_source(d.vocab_src, Tx - 1, seed=seed)
    s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=seed + 1)
    off, words = synth.make_candidates(R, cands, d.vocab_tgt, seed=seed + 2)
    return src, s, y, off, words


def _dev_step(M, src, s, y, off, words):
    """Exactly bench.py's timed step: device-resident inputs, nmt_*_dev calls on the model stream."""
    import torch
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        dsrc, ds, dy = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (src, s, y))
        doff, dw = torch.from_numpy(off).cuda(), torch.from_numpy(words).cuda()
        R, nc = len(y), len(words)
        ids = torch.empty(R, dtype=torch.int32, device="cuda")
        lp = torch.empty(nc, dtype=torch.float32, device="cuda")
        ch = torch.empty(nc, dtype=torch.int32, device="cuda")
        am = torch.empty(R, dtype=torch.int32, device="cuda")
    st.synchronize()
    ctx = M.encode_dev(dsrc.data_ptr(), len(src))
    ctx.inject_states_dev(R, ds.data_ptr(), dy.data_ptr(), ids.data_ptr())
    ctx.score_batch_dev(R, ids.data_ptr(), doff.data_ptr(), nc, dw.data_ptr(), lp.data_ptr(), ch.data_ptr(),
                        am.data_ptr())
    ctx.check()  # waits for the model stream, reports device-side validation errors
    out = lp.cpu().numpy(), ch.cpu().numpy().astype(np.int64), am.cpu().numpy(), ids.cpu().numpy()
    ctx.close()
    return out


def _host_step(M, src, s, y, off, words):
    c = M.encode(src)
    ids = c.inject_states(s, y)
    lp, ch, am = c.score_batch(ids, off, words)
    c.close()
    return lp, ch, am, ids


@pytest.mark.parametrize("prec", ["bf16", "fp32class"])
def test_dev_path_equals_host_path_and_oracle(bench_model, prec):
    d, p, blob = bench_model
    M = nmt().Model(blob, precision=prec, max_src_len=64)
    src, s, y, off, words = _c2_inputs(d, 4242)
    dlp, dch, dam, dids = _dev_step(M, src, s, y, off, words)
    hlp, hch, ham, hids = _host_step(M, src, s, y, off, words)
    assert np.array_equal(dids, hids)
    assert np.array_equal(dch, hch) and np.array_equal(dam, ham)
    assert np.array_equal(dlp.view(np.uint32), hlp.view(np.uint32)), "device path differs from the host path"
    om = O.Model(d, p)
    rows = list(range(0, len(y), 61)) + [len(y) - 1]
    out = O.step(om, O.encode(om, src), s[rows].astype(np.float64), y[rows])
    worst = 0.0
    for j, r in enumerate(rows):
        lsm = O.log_softmax(out["z"][j])
        worst = max(worst, float(np.max(np.abs(dlp[off[r]:off[r + 1]] - lsm[words[off[r]:off[r + 1]]]))))
        assert lsm[dam[r]] >= lsm.max() - 2 * TOL[prec]
    print(f"\n[dev path {prec}] sampled max|dlogp| = {worst:.2e}")
    assert worst < TOL[prec]


def test_run_to_run_determinism_fresh_models(bench_model):
    """Two fresh models (fresh arenas, fresh workspaces) and a reused pooled context: the C2 batch gives
    bit-identical log-probs, child ids and argmax."""
    d, p, blob = bench_model
    src, s, y, off, words = _c2_inputs(d, 777)
    runs = []
    for _ in range(2):
        M = nmt().Model(blob, precision="bf16")
        runs.append(_dev_step(M, src, s, y, off, words))
        runs.append(_dev_step(M, src, s, y, off, words))  # pooled arena reused
        runs.append(_host_step(M, src, s, y, off, words))
        M.close()
    for r in runs[1:]:
        assert np.array_equal(r[0].view(np.uint32), runs[0][0].view(np.uint32))
        assert np.array_equal(r[1], runs[0][1]) and np.array_equal(r[2], runs[0][2])


def test_c3_full_shape_stack_sampled():
    """C3 Ru->En (E 500, H 1024, V_s 100k, V_t 50k, tanh readout, seed 1605): one sentence, a stack of
    4096 distinct (hypothesis, phrase) expansions over 1024 hypothesis states in ONE nmt_score_forest
    call (<= 5 depths, shared prefixes collapsed).  Sampled pairs are rescored by the oracle's uncached
    sequential scorer; the dedup law naive words >= edges >= rows holds per depth."""
    d = synth.RU_EN
    p = synth.make_model(d, 1605)
    M = nmt().Model(synth.params_bytes(d, p), precision="bf16")
    om = O.Model(d, p)
    src = synth.make_source(d.vocab_src, 37, seed=1605)
    c = M.encode(src)
    n_h = 1024
    s, y = synth.make_states(n_h, d.dim_hid, d.vocab_tgt, seed=3000)
    pairs = synth.make_stack_expansions(4096, n_h, d.vocab_tgt, seed=4000)
    assert len(pairs) == 4096
    hs = c.inject_states(s, y)
    off = np.cumsum([0] + [len(t) for _, t in pairs]).astype(np.int32)
    words = np.array([w for _, t in pairs for w in t], np.int32)
    lp, fin, st = c.score_forest(hs[[h for h, _ in pairs]], off, words)
    assert st["steps"] == max(len(t) for _, t in pairs) <= 5
    assert all(r <= e for r, e in zip(st["rows_per_depth"], st["edges_per_depth"]))
    assert sum(st["edges_per_depth"]) <= len(words)
    assert np.all(np.isfinite(lp)) and np.all(lp <= 0)
    oc = O.encode(om, src)
    rng = np.random.default_rng(0)
    sample = sorted(rng.choice(len(pairs), 24, replace=False).tolist()) + [len(pairs) - 1]
    worst = 0.0
    for i in sample:
        h, t = pairs[i]
        ref, _, _ = O.score_sequence(om, oc, t, s=s[h].astype(np.float64), y_prev=int(y[h]))
        worst = max(worst, abs(float(lp[i]) - ref) / len(t))
    print(f"\n[C3 full shape] {len(words)} naive words, edges {st['edges_per_depth']}, rows {st['rows_per_depth']}, "
          f"sampled max|dlogp| per word = {worst:.2e}")
    assert worst < TOL["bf16"]


@pytest.mark.parametrize("prec", ["bf16", "fp32class"])
def test_projected_and_explicit_context_forms(bench_model, prec):
    """Both forms of D5-D7 (reading A31) on the same source and requests: a context from
    nmt_encode takes the projected single-context step (c . W = alpha . (ctx . W), K = Tx), a context from
    the batched encoder (nmt_encode_batch of > 8 sentences) the explicit one (c formed by the attention,
    K = 2H); the batched encoder's own arithmetic differs within the precision (reading A27).  Both against the oracle, and
    against each other within the precisions' operand rounding."""
    d, p, blob = bench_model
    M = nmt().Model(blob, precision=prec)
    src, s, y, off, words = _c2_inputs(d, seed=71, R=96, cands=3, Tx=37)
    c_proj = M.encode(src)
    others = [synth.make_source(d.vocab_src, 20 + k, seed=900 + k) for k in range(9)]
    batch = M.encode_batch([src] + others)  # (> 8 sentences: the batched encoder, contexts without cw)
    c_expl = batch[0]
    ids_p = c_proj.inject_states(s, y)
    ids_e = c_expl.inject_states(s, y)
    lp_p, ch_p, am_p = c_proj.score_batch(ids_p, off, words)
    lp_e, ch_e, am_e = c_expl.score_batch(ids_e, off, words)
    assert np.array_equal(ch_p - ch_p.min(), ch_e - ch_e.min())
    om = O.Model(d, p)
    rows = list(range(0, 96, 12))
    out = O.step(om, O.encode(om, src), s[rows].astype(np.float64), y[rows])
    rl = np.concatenate([O.log_softmax(out["z"][j])[words[off[r]:off[r + 1]]] for j, r in enumerate(rows)])
    got_p = np.concatenate([lp_p[off[r]:off[r + 1]] for r in rows])
    got_e = np.concatenate([lp_e[off[r]:off[r + 1]] for r in rows])
    err_p, err_e = float(np.max(np.abs(got_p - rl))), float(np.max(np.abs(got_e - rl)))
    print(f"\n[A31 forms] {prec}: projected {err_p:.2e}, explicit {err_e:.2e}, "
          f"between {np.max(np.abs(lp_p - lp_e)):.2e}")
    assert err_p < TOL[prec] and err_e < TOL[prec]
    assert np.max(np.abs(lp_p - lp_e)) < (5e-4 if prec == "fp32class" else TOL[prec])
