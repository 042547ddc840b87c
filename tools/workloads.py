"""Secondary workloads of BASELINE.json:configs (not the bench.py headline line):

  c3     Ru->En shape (V_t 50k, V_s 100k): per sentence (L ~ U[10,50]) one stack of 4096 distinct
         (hypothesis, phrase) expansions over 1024 hypothesis states, scored with the ScoreBatch
         forest driver (one nmt_score_batch per depth) - word-scores/s, rows/s and the dedup ratio
         naive words : collapsed edges (word-scores) : stepped rows.
  sweep  C2 model (V_t 100k): hypothesis batch-size sweep R in 64..16384 (x3 candidates) through the
         device-resident C ABI - word-scores/s and the vocabulary GEMM's TFLOP/s / fraction of the
         measured bf16 peak per R (HBM-bound W_o stream at small R, tensor-bound at large R).
  beam   C2 model: nmt_beam_step over R fresh injected parents, k = 8 -
         expansions/s (R x k per call, host C ABI, synchronised) for R in 256..4096.
  avg    NMT-k-Avg vs the k-ensemble ("four times smaller and four times faster"):
         one C2 batch (R = 1024 x 3) scored by 4 member models in turn (+ log-linear combine on
         the host) vs by their nmt_params_average model, on one GPU.
  encb   nmt_encode_batch vs a loop of nmt_encode: n sentences of L ~ U[10,50] (+EOS) tokens, En->Ru
         encoder (H 1024) - sentences/s, source tokens/s and the recurrence+pctx TFLOP/s per n.
  c5     cube-pruning workload: sentences L ~ U[10,50]; per sentence one batched
         encode (nmt_encode_batch over a chunk of sentences), B injected hypothesis states, then L
         stacks, each a ScoreBatch (nmt_score_forest) of B (hypothesis, phrase) pairs with phrase
         lengths 1..4 w.p. .4/.3/.2/.1 (rows per depth ~ B [1, .6, .3, .1]); stack s+1 expands the
         final states of stack s.  Sweep B in 64..16384; the sentence count of a point is cut to a
         fixed row budget (recorded).  Sentences are sharded over ranks by greedy LPT on L x B
         under torchrun (no collective on the data path; max-over-ranks time).
  ens    C4 ensemble: member m = rank (seed 2016 + m) scores the same C2 batch (R = 1024 x 3) and
         the per-word scores are combined by nmt_ensemble_combine (NCCL reduce to rank 0, log-linear,
         lambda = 1/M) - combined word-scores/s and the reduce's microseconds.  One GPU per member.
Prints one JSON line per measurement point.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def peaks():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    return json.load(open(p)) if os.path.exists(p) else {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}


def c3(a):
    import torch
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(500, 1024, 100000, 50000, a.readout)
    M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 1605)), precision=a.precision)
    rng = np.random.default_rng(1605)
    tot_t = tot_e = tot_r = tot_n = 0
    per = []
    WARM = 3  # warm-up sentences (arena growth to steady-state capacity)
    for k in range(a.sentences + WARM):
        L = int(rng.integers(10, 51))
        src = synth.make_source(d.vocab_src, L, seed=1605 + k)
        s, y = synth.make_states(1024, d.dim_hid, d.vocab_tgt, seed=3000 + k)
        pairs = synth.make_stack_expansions(4096, 1024, d.vocab_tgt, seed=4000 + k)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        off = np.cumsum([0] + [len(t) for _, t in pairs]).astype(np.int32)
        words = np.array([w for _, t in pairs for w in t], np.int32)
        hidx = np.array([h for h, _ in pairs], np.int64)
        ctx = M.encode(src)
        ctx.reserve(1024 + len(words) + 1, len(words))  # (pooled arena: grows during warm-up only)
        hyps = ctx.inject_states(s, y)
        lp, fin, st = ctx.score_forest(hyps[hidx], off, words)  # native ScoreBatch (one call)
        ctx.close()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if k < WARM:
            continue  # warm-up sentences
        tot_t += dt
        tot_e += sum(st["edges_per_depth"])
        tot_r += sum(st["rows_per_depth"])
        tot_n += len(words)
        per.append(sum(st["edges_per_depth"]) / dt)
        print(json.dumps({"workload": "c3", "sentence": k, "src_len": L + 1, "ms": 1000 * dt,
                          "steps": st["steps"], "edges_per_depth": st["edges_per_depth"],
                          "rows_per_depth": st["rows_per_depth"], "naive_words": int(len(words))}), flush=True)
    print(json.dumps({"workload": "c3 summary", "precision": a.precision, "readout": a.readout,
                      "sentences": a.sentences, "word_scores_per_s": tot_e / tot_t, "rows_per_s": tot_r / tot_t,
                      "median_word_scores_per_s": float(np.median(per)),
                      "dedup naive:edges:rows": [1.0, tot_e / tot_n, tot_r / tot_n],
                      "timing": "host wall clock around nmt_encode + nmt_inject_states + nmt_score_forest "
                                "(host C ABI, inputs and outputs on the host), synchronized"}), flush=True)


def sweep(a):
    import torch
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(500, 1024, 50000, 100000, a.readout)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016)), precision=a.precision, stream=st.cuda_stream)
    pk = peaks()
    src = torch.from_numpy(synth.make_source(d.vocab_src, 49, seed=1)).cuda()
    flush = torch.empty(256 * 2**20 // 4, device="cuda")
    vi = nmt.STAGES.index("vocab_gemm_lse")
    for R in [64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384]:
        s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=R)
        off, w = synth.make_candidates(R, 3, d.vocab_tgt, seed=R + 1)
        ds, dy, doff, dw = (torch.from_numpy(x).cuda() for x in (s, y, off, w))
        ids = torch.empty(R, dtype=torch.int32, device="cuda")
        lp = torch.empty(3 * R, device="cuda")
        ch = torch.empty(3 * R, dtype=torch.int32, device="cuda")
        ctx = M.encode_dev(src.data_ptr(), 50)
        n_inj = 1 + 3 + a.iters  # injections of R parents into this context (+ their 3R children)
        ctx.reserve(4 * R * n_inj + 1, 2 * R * n_inj)  # steady state: no arena growth while timed
        ctx.inject_states_dev(R, ds.data_ptr(), dy.data_ptr(), ids.data_ptr())

        def score():  # re-score fresh parents every iteration: inject new nodes each time
            ctx.inject_states_dev(R, ds.data_ptr(), dy.data_ptr(), ids.data_ptr())
            ctx.score_batch_dev(R, ids.data_ptr(), doff.data_ptr(), 3 * R, dw.data_ptr(), lp.data_ptr(),
                                ch.data_ptr(), None)
        for _ in range(3):
            score()
        M.profile(1)
        M.profile_read()
        ev = []
        for _ in range(a.iters):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            score()
            e1.record(st)
            ev.append((e0, e1))
        torch.cuda.synchronize()
        ms, cnt = M.profile_read()
        M.profile(0)
        t = sum(e0.elapsed_time(e1) for e0, e1 in ev) / a.iters
        vms = ms[vi] / cnt[vi]
        tf = 2 * R * d.vocab_tgt * d.dim_emb / (vms / 1000) / 1e12
        wo_gbs = 2 * 512 * 100096 / (vms / 1000) / 1e9
        ctx.close()
        print(json.dumps({"workload": "sweep", "R": R, "ms_per_batch": t, "word_scores_per_s": 3 * R / (t / 1000),
                          "rows_per_s": R / (t / 1000), "vocab_ms": vms, "vocab_tflops": tf,
                          "vocab_frac_bf16_peak": tf / pk["bf16_tflops"], "W_o_stream_GBps": wo_gbs,
                          "W_o_frac_hbm": wo_gbs / pk["hbm_gbs"],
                          "note": "per batch: inject R parents + nmt_score_batch_dev (no encode), L2 flushed, "
                                  "arena reserved up front (no growth while timed)"}),
              flush=True)


def beam(a):
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(500, 1024, 50000, 100000, a.readout)
    M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016)), precision=a.precision)
    src = synth.make_source(d.vocab_src, 49, seed=1)
    for R in [256, 1024, 4096]:
        s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=R)
        ctx = M.encode(src)
        n_inj = 3 + a.iters
        ctx.reserve(9 * R * n_inj + 1, 2 * R * n_inj)  # steady state: no arena growth while timed
        for _ in range(3):  # warm-up
            ctx.beam_step(ctx.inject_states(s, y), 8)
        ts = []
        for _ in range(a.iters):
            hy = ctx.inject_states(s, y)
            t0 = time.perf_counter()
            ctx.beam_step(hy, 8)
            ts.append(time.perf_counter() - t0)
        ctx.close()
        t = float(np.median(ts))
        print(json.dumps({"workload": "beam", "R": R, "k": 8, "precision": a.precision, "ms_per_call": 1000 * t,
                          "expansions_per_s": R * 8 / t, "rows_per_s": R / t,
                          "timing": "host wall clock around nmt_beam_step (parents injected outside), median"}),
              flush=True)


def avg(a):
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(500, 1024, 50000, 100000, a.readout)
    blobs = [synth.params_bytes(d, synth.make_model(d, 2016 + i)) for i in range(4)]
    members = [nmt.Model(b, precision=a.precision) for b in blobs]
    avg_model = nmt.Model(nmt.params_average(blobs), precision=a.precision)
    src = synth.make_source(d.vocab_src, 49, seed=1)
    s, y = synth.make_states(1024, d.dim_hid, d.vocab_tgt, seed=5)
    off, w = synth.make_candidates(1024, 3, d.vocab_tgt, seed=6)

    def run(models):
        out = []
        for M in models:
            ctx = M.encode(src)
            lp, _, _ = ctx.score_batch(ctx.inject_states(s, y), off, w, with_argmax=False)
            ctx.close()
            out.append(lp)
        return np.mean(np.stack(out), axis=0) if len(out) > 1 else out[0]  # log-linear, lambda = 1/4
    for _ in range(2):
        run(members)
        run([avg_model])
    te, ta = [], []
    for _ in range(a.iters):
        t0 = time.perf_counter()
        run(members)
        te.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        run([avg_model])
        ta.append(time.perf_counter() - t0)
    e, v = float(np.median(te)), float(np.median(ta))
    print(json.dumps({"workload": "avg", "members": 4, "precision": a.precision,
                      "ensemble_ms_per_batch": 1000 * e, "average_ms_per_batch": 1000 * v,
                      "speedup_average_vs_ensemble": e / v,
                      "batch": "1 source (Tx=50) + 1024 injected parents x 3 words, host C ABI, one GPU",
                      "note": "PAPER.md:305 reports the averaged model four times faster than the 4-ensemble"}),
          flush=True)


ENC_FLOP_PER_TOKEN = 2 * 2 * 1024 * 3072 + 2 * 2048 * 2048  # E3/E4 recurrence + E7 pctx
ENC_FLOP_PER_SENTENCE = 2 * 2048 * 1024                   # E6 s0


def encb(a):
    import torch
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(500, 1024, 50000, 100000, a.readout)
    M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016)), precision=a.precision, max_src_len=64)
    rng = np.random.default_rng(3000)
    for n in [1, 16, 64, 256, 1024, 3000]:
        srcs = [synth.make_source(d.vocab_src, int(rng.integers(10, 51)), seed=7000 + i) for i in range(n)]
        ntok = sum(len(x) for x in srcs)
        for _ in range(2):
            for c in M.encode_batch(srcs):
                c.close()
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(1, a.iters // 2)):
            t0 = time.perf_counter()
            cs = M.encode_batch(srcs)
            cs[0].check()  # synchronises the model stream
            ts.append(time.perf_counter() - t0)
            for c in cs:
                c.close()
        tb = float(np.median(ts))
        m_loop = min(n, 64)  # the single-sentence kernel, over the first sentences
        for c in [M.encode(x) for x in srcs[:2]]:
            c.close()
        t0 = time.perf_counter()
        cs = [M.encode(x) for x in srcs[:m_loop]]
        cs[-1].check()
        tl = (time.perf_counter() - t0) / m_loop
        for c in cs:
            c.close()
        flop = ntok * ENC_FLOP_PER_TOKEN + n * ENC_FLOP_PER_SENTENCE
        print(json.dumps({"workload": "encb", "n": n, "tokens": ntok, "precision": a.precision,
                          "batch_ms": 1000 * tb, "sentences_per_s": n / tb, "tokens_per_s": ntok / tb,
                          "tflops": flop / tb / 1e12, "single_encode_ms_per_sentence": 1000 * tl,
                          "speedup_vs_single": tl * n / tb,
                          "timing": "host wall clock around nmt_encode_batch + stream sync (median)"}), flush=True)


def _dist():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
        return rank, world, dist
    return 0, 1, None


def lpt_shard(costs, world):
    """Greedy LPT: sentences in descending cost to the least-loaded rank (deterministic)."""
    load = [0.0] * world
    out = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        r = min(range(world), key=lambda r: (load[r], r))
        out[r].append(i)
        load[r] += costs[i]
    return [sorted(x) for x in out]


def c5(a):
    import torch
    from paper_1605_04809_b200 import nmt
    rank, world, dist = _dist()
    d = synth.Dims(500, 1024, 50000, 100000, a.readout)
    M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016)), precision=a.precision, max_src_len=64)
    rng = np.random.default_rng(3000)
    lens = [int(x) for x in rng.integers(10, 51, size=3000)]
    Bs = [int(x) for x in a.batches.split(",")]
    for B in Bs:
        n_sent = max(world, min(3000, int(a.row_budget // (2.0 * B * 30))))
        costs = [lens[i] * B for i in range(n_sent)]
        mine = lpt_shard(costs, world)[rank]

        s_st, y_st = synth.make_states(B, d.dim_hid, d.vocab_tgt, seed=50000 + B)  # one stack's states

        def run(sents, count):
            edges = rows = naive = stacks = 0
            for c0 in range(0, len(sents), a.enc_chunk):
                chunk = sents[c0:c0 + a.enc_chunk]
                srcs = [synth.make_source(d.vocab_src, lens[i], seed=9000 + i) for i in chunk]
                ctxs = M.encode_batch(srcs)
                for i, ctx in zip(chunk, ctxs):
                    g = np.random.default_rng(100000 * B + i)
                    n_stk = lens[i] + 1  # one stack per target position (~L)
                    L = g.choice(4, size=(n_stk, B), p=[.4, .3, .2, .1]).astype(np.int32) + 1
                    words_all = synth.zipf_ids(g, int(L.sum()), d.vocab_tgt)
                    ctx.reserve(int(L.sum()) + B + 1, int(L.sum()))
                    hyps = ctx.inject_states(s_st, y_st)
                    w0 = 0
                    for stk in range(n_stk):
                        off = np.zeros(B + 1, np.int32)
                        off[1:] = np.cumsum(L[stk])
                        words = words_all[w0:w0 + off[-1]]
                        w0 += int(off[-1])
                        lp, fin, st = ctx.score_forest(hyps, off, words)
                        hyps = fin
                        if count:
                            edges += sum(st["edges_per_depth"])
                            rows += sum(st["rows_per_depth"])
                            naive += int(off[-1])
                            stacks += 1
                    ctx.close()
            return edges, rows, naive, stacks
        tcall = [0.0]  # seconds inside nmt_score_batch_multi (host wall, synchronised calls)
        tphase = [0.0, 0.0, 0.0]  # encode_batch, reserve, inject
        max_tot = [0]  # words of the largest sentence of this point (arena reservation)

        def prep_multi(sents):
            """synthetic requests of each chunk (outside the timed region): phrase lengths and words"""
            out = []
            for c0 in range(0, len(sents), a.concurrent):
                chunk = sents[c0:c0 + a.concurrent]
                S = len(chunk)
                g = np.random.default_rng(100000 * B + chunk[0])
                nstk = np.array([lens[i] + 1 for i in chunk])
                T = int(nstk.max())
                L_all = (g.choice(4, size=(S, T, B), p=[.4, .3, .2, .1]) + 1).astype(np.int32)
                L_all[np.arange(T)[None, :] >= nstk[:, None]] = 0  # sentences with fewer stacks
                W_all = synth.zipf_ids(g, S * T * B * 4, d.vocab_tgt).reshape(S, T, B, 4)
                srcs = [synth.make_source(d.vocab_src, lens[i], seed=9000 + i) for i in chunk]
                max_tot[0] = max(max_tot[0], int(L_all.sum(axis=(1, 2)).max()))
                out.append((chunk, nstk, L_all, W_all, srcs))
            return out

        def run_multi(prepped, count):
            """a.concurrent sentences at a time: each (stack, depth) is ONE nmt_score_batch_multi over
            all of them (rows of different sentences share the fused decoder step)."""
            edges = stacks = 0
            tcall[0] = 0.0
            tphase[:] = [0.0, 0.0, 0.0]
            for chunk, nstk, L_all, W_all, srcs in prepped:
                S, T = L_all.shape[0], L_all.shape[1]
                tp0 = time.perf_counter()
                ctxs = M.encode_batch(srcs)
                tphase[0] += time.perf_counter() - tp0
                hnd_pair = np.repeat(np.array([c.handle for c in ctxs], np.int64), B)
                cur_h = np.empty(S * B, np.int64)
                tp0 = time.perf_counter()
                for ctx in ctxs:  # every arena sized for the largest sentence of the point: pooled arenas
                    ctx.reserve(max_tot[0] + B + 1, max_tot[0])  # never grow inside the timed region
                tp1 = time.perf_counter()
                for q, ctx in enumerate(ctxs):
                    cur_h[q * B:(q + 1) * B] = ctx.inject_states(s_st, y_st)
                tp2 = time.perf_counter()
                tphase[1] += tp1 - tp0
                tphase[2] += tp2 - tp1
                for stk in range(T):
                    L = L_all[:, stk, :].reshape(-1)
                    Wst = W_all[:, stk, :, :].reshape(-1, 4)
                    cur = cur_h.copy()
                    for dep in range(4):
                        sel = np.nonzero(L > dep)[0]
                        if len(sel) == 0:
                            break
                        off = np.arange(len(sel) + 1, dtype=np.int32)
                        tc0 = time.perf_counter()
                        lp, ch, _ = nmt.score_batch_multi(hnd_pair[sel], cur[sel], off, Wst[sel, dep],
                                                          with_argmax=False)
                        tcall[0] += time.perf_counter() - tc0
                        cur[sel] = ch
                        if count:
                            edges += len(sel)
                    live = L > 0
                    cur_h[live] = cur[live]  # the stack's hypotheses: the phrase-final states
                    if count:
                        stacks += int((nstk > stk).sum())
                for ctx in ctxs:
                    ctx.close()
            # one candidate per parent and every parent a fresh node: naive words = edges = rows
            return edges, edges, edges, stacks

        if a.concurrent > 1:
            work = prep_multi(mine)
            warm = prep_multi(mine[:min(len(mine), a.concurrent)])
            run_multi(warm, False)  # warm-up (workspaces, arenas at the point's largest reservation)
            runner = lambda: run_multi(work, True)
        else:
            run(mine[:min(len(mine), 2)], False)  # warm-up (workspaces)
            runner = lambda: run(mine, True)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        import bench  # (nvidia-smi clock / throttle sampler of the bench contract)
        with bench.ClockSampler(torch.cuda.current_device()) as clk:
            t0 = time.perf_counter()
            e, r, nv, ns = runner()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        clocks = clk.summary()
        tot = torch.tensor([e, r, nv, ns, len(mine)], dtype=torch.float64, device="cuda")
        tmax = torch.tensor([dt], dtype=torch.float64, device="cuda")
        if dist:
            dist.all_reduce(tot)
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        e, r, nv, ns, nsent = (float(x) for x in tot.tolist())
        dt = float(tmax.item())
        if rank == 0:
            print(json.dumps({"workload": "c5", "B": B, "gpus": world, "precision": a.precision,
                              "concurrent_sentences": a.concurrent,
                              "seconds_in_score_calls": tcall[0] if a.concurrent > 1 else None,
                              "seconds_encode_reserve_inject": list(tphase) if a.concurrent > 1 else None,
                              "clocks": clocks,
                              "sentences": int(nsent), "stacks": int(ns), "word_scores_per_s": e / dt,
                              "rows_per_s": r / dt, "naive_words": int(nv), "edges": int(e), "rows": int(r),
                              "seconds": dt, "row_budget": a.row_budget,
                              "timing": ("host wall clock (max over ranks) around encode_batch + reserve + inject + "
                                         "L+1 stacks x depth <= 4 nmt_score_batch_multi calls over concurrent sentences "
                                         "(host C ABI, synchronized; request generation outside the timed region)")
                              if a.concurrent > 1 else
                              ("host wall clock (max over ranks) around encode_batch + reserve + inject "
                               "+ L+1 stacks of nmt_score_forest per sentence (host C ABI, synchronized; "
                               "the synthetic request generation is inside the timed region)")}),
                  flush=True)


def ens(a):
    import torch
    from paper_1605_04809_b200 import nmt
    rank, world, dist = _dist()
    dev = torch.cuda.current_device()
    d = synth.Dims(500, 1024, 50000, 100000, a.readout)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016 + rank)), precision=a.precision,
                  stream=st.cuda_stream)
    if dist:
        obj = [nmt.Ensemble.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    else:
        uid = nmt.Ensemble.unique_id()
    E = nmt.Ensemble(world, rank, uid, dev)
    R, Cn = 1024, 3
    src = torch.from_numpy(synth.make_source(d.vocab_src, 49, seed=1)).cuda()
    s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=5)
    off, w = synth.make_candidates(R, Cn, d.vocab_tgt, seed=6)
    ds, dy, doff, dw = (torch.from_numpy(x).cuda() for x in (s, y, off, w))
    ids = torch.empty(R, dtype=torch.int32, device="cuda")
    lp = torch.empty(R * Cn, device="cuda")
    ch = torch.empty(R * Cn, dtype=torch.int32, device="cuda")
    out = torch.empty(R * Cn, device="cuda")

    def step(combine=True):
        ctx = M.encode_dev(src.data_ptr(), 50)
        ctx.inject_states_dev(R, ds.data_ptr(), dy.data_ptr(), ids.data_ptr())
        ctx.score_batch_dev(R, ids.data_ptr(), doff.data_ptr(), R * Cn, dw.data_ptr(), lp.data_ptr(),
                            ch.data_ptr(), None)
        if combine:
            E.combine(lp.data_ptr(), R * Cn, 1.0 / world, 0, 0, out.data_ptr(), st.cuda_stream)
        ctx.close()
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    e0.record(st)
    for _ in range(a.iters):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(st)
    for _ in range(100):
        E.combine(lp.data_ptr(), R * Cn, 1.0 / world, 0, 0, out.data_ptr(), st.cuda_stream)
    c1.record(st)
    torch.cuda.synchronize()
    red_us = 1000 * c0.elapsed_time(c1) / 100
    t = torch.tensor([ms, red_us], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, red_us = (float(x) for x in t.tolist())
    if rank == 0:
        print(json.dumps({"workload": "ens", "members": world, "gpus": world, "precision": a.precision,
                          "ms_per_batch": ms, "combined_word_scores_per_s": R * Cn / (ms / 1000),
                          "reduce_us": red_us, "message_bytes": 4 * R * Cn,
                          "batch": "encode Tx=50 + 1024 injected parents x 3 words per member, device C ABI",
                          "timing": "CUDA events on the model stream, max over ranks"}), flush=True)
    E.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["c3", "sweep", "beam", "avg", "encb", "c5", "ens"])
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--readout", default="tanh")
    ap.add_argument("--sentences", type=int, default=10)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--batches", default="64,256,1024,4096,16384")
    ap.add_argument("--row_budget", type=float, default=2e6)
    ap.add_argument("--enc_chunk", type=int, default=64)
    ap.add_argument("--concurrent", type=int, default=1, help="c5: sentences per fused multi-context step")
    a = ap.parse_args()
    {"c3": c3, "sweep": sweep, "beam": beam, "avg": avg, "encb": encb, "c5": c5, "ens": ens}[a.what](a)
