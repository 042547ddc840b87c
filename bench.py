#!/usr/bin/env python
"""bench.py - hypothesis word-scores/s of the batched cGRU scorer on B200 (BASELINE.json metric).

One step = one pass of the whole hot path (SURVEY §8(a) E1-E7 + D0-D9) over one batch of the C2
En->Ru workload (BASELINE.json configs[1]): encode one synthetic source sentence (Tx = 50 incl. EOS),
inject R = 1024 synthetic parent states, and score R x 3 candidate words (3072 word-scores) through
nmt_score_batch (device planner -> GRU1 -> attention -> GRU2 -> readout -> vocab GEMM + fused
log-softmax -> gather).  `value` times the device-resident C-ABI path (nmt_*_dev, inputs already in
HBM); `e2e` times the host API (pinned host inputs copied in, results copied out) every step.
Variants in the same line (`variants`): the primary C2 with 1 candidate per row, and the FP32CLASS
precision (bf16x3, bound 1e-3), each with its own in-run parity against the float64 oracle.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--ensemble M]
  N > 1: one rank per GPU.  Without torchrun in the environment (WORLD_SIZE unset) bench.py starts
  torchrun itself.  Sentences are sharded over ranks (weak scaling, no collective on the data path).
  --ensemble M: C4, an M-member ensemble (seeds 2016..) whose per-word log-probs are combined to rank 0
  of each member group (one member per GPU over NCCL when N >= M, groups of M ranks; all M members on
  the one GPU over the in-process communicator when N == 1).
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "hypothesis word-scores/sec at 100k vocab, 1/2/4/8 B200; % tensor-pipe peak"
UNIT = "word-scores/s"


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32class"])
    ap.add_argument("--readout", default="maxout", choices=["maxout", "tanh"])
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--cands", type=int, default=3)
    ap.add_argument("--src-len", type=int, default=50)
    ap.add_argument("--ensemble", type=int, default=0, help="C4: number of ensemble members (0: single model)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--stages", action="store_true", help="add a per-stage CUDA-event breakdown (untimed pass)")
    return ap.parse_args(argv)


def model_dims(readout: str) -> synth.Dims:
    return synth.Dims(500, 1024, 50000, 100000, readout)


def workload_config(a, n_gpus: int) -> dict:
    c = {"workload": f"C2 En->Ru: encode 1 source (Tx={a.src_len}) + score {a.rows} injected parents x "
                     f"{a.cands} candidate words per step",
         "dim_emb": 500, "dim_hid": 1024, "vocab_tgt": 100000, "src_len": a.src_len, "rows": a.rows,
         "cands_per_row": a.cands, "precision": a.precision, "readout": a.readout,
         "l2": "flushed before every timed step (256 MiB write)",
         "parallelism": f"{n_gpus} GPU(s), sentence sharding, no collective on the data path"}
    if a.ensemble:
        c["workload"] = (f"C4 En->Ru ensemble of {a.ensemble} members: per member encode 1 source (Tx={a.src_len}) "
                         f"+ score {a.rows} parents x {a.cands} words, combined log-probs (mode 0, lambda = 1/M)")
        c["members"] = a.ensemble
        c["l2"] = "not flushed: each step reads the weights of all members (> 4 x 0.3 GB), larger than L2"
        c["parallelism"] = (f"{n_gpus} GPU(s): " + ("one member per GPU, NCCL all-gather + combine on the group's "
                                                    "rank 0" if n_gpus >= a.ensemble else
                                                    f"all {a.ensemble} members on one GPU (in-process communicator)"))
    return c


def shard_seed(rank: int, step: int) -> int:
    """Sentence (and batch) seed for a rank/step: disjoint shards per rank (weak scaling)."""
    return 100_003 * (rank + 1) + step


def reduce_max(value: float, dist) -> float:
    """Max over ranks (the slowest rank defines the job time)."""
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(value: float, dist) -> float:
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def step_flops(rows: int, src_len: int, d: synth.Dims) -> dict:
    """Algorithmic dense work of one bench step (multiply-add = 2 flops), SURVEY §8(a)/(d):
    per decoder row: GRU1 s.[U|Ux] 2*H*3H, query s1.W_comb_att 2*H*2H, attention energies + context
    4*Tx*2H, GRU2 2*(H+2H)*2H + 2*H*H + 2*2H*H, readout 2*(2H+H)*RO (RO = 2E maxout, E tanh), vocabulary
    2*E*V; per source token: input projections 2*E*3H*2, recurrence 2*H*3H*2, keys pctx 2*2H*2H; per
    sentence s0 2*2H*H.  (The embedding projections the library precomputes at load are counted.)"""
    E, H, V = d.dim_emb, d.dim_hid, d.vocab_tgt
    RO = 2 * E if d.readout == "maxout" else E
    row = (2 * H * 3 * H + 2 * H * 2 * H + 4 * src_len * 2 * H + 2 * 3 * H * 2 * H + 2 * H * H + 2 * 2 * H * H
           + 2 * 3 * H * RO + 2 * E * V + 2 * E * 3 * H + 2 * E * RO)
    enc = src_len * (2 * E * 3 * H * 2 + 2 * H * 3 * H * 2 + 2 * 2 * H * 2 * H) + 2 * 2 * H * H
    # the dense work the library executes per step (reading A31): the embedding projections are
    # precomputed at load (Ex, Eproj, EncIn: gathers per step), and c . W (GRU2 gates, readout) is computed as
    # alpha . (ctx . W) with ctx . W once per sentence (K = Tx instead of 2H per row)
    xrow = (2 * H * 3 * H + 2 * H * 2 * H + 2 * src_len * 2 * H + 2 * H * 3 * H + 2 * src_len * 3 * H
            + 2 * H * RO + 2 * src_len * RO + 2 * E * V)
    xenc = src_len * (2 * H * 3 * H * 2 + 2 * 2 * H * 2 * H + 2 * 2 * H * (3 * H + RO)) + 2 * 2 * H * H
    return {"per_row": row, "encoder": enc, "per_step": rows * row + enc, "executed_per_step": rows * xrow + xenc}


# ------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling DURING the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self) -> dict:
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for ln in fh:
                parts = [x.strip() for x in ln.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if num(r[1])]
        mx = [num(r[2]) for r in rows if num(r[2])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        loaded = [s for s in sm if s and s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded or sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------------- oracle (CPU)
def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(n[0])
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


def oracle_sample(om, d, a, rows: int, seed: int, cands: int | None = None) -> tuple:
    """One bounded sample of the step on the host: encode 1 source + `rows` parents x cands."""
    import oracle as O
    cands = a.cands if cands is None else cands
    src = synth.make_source(d.vocab_src, a.src_len - 1, seed=seed)
    s, y = synth.make_states(rows, d.dim_hid, d.vocab_tgt, seed=seed + 1)
    off, words = synth.make_candidates(rows, cands, d.vocab_tgt, seed=seed + 2)
    t0 = time.perf_counter()
    sess = O.Session(om, src)
    ids = [sess.inject_state(s[i], int(y[i])) for i in range(rows)]
    lp, _, am = sess.score_batch(ids, off, words)
    dt = time.perf_counter() - t0
    assert np.all(np.isfinite(lp))
    oracle_sample.last = (src, s, y, off, words, lp, am, sess, ids)  # (inputs and results, for the parity check)
    return dt, rows * cands


def run_reference(a, rank: int, world: int) -> None:
    """--impl reference: the float64 oracle on the host cores, bounded samples of the same workload."""
    if rank != 0:
        return
    import oracle as O
    try:  # the box's host cores (torchrun sets OMP_NUM_THREADS=1 per rank)
        from threadpoolctl import threadpool_limits
        threadpool_limits(len(os.sched_getaffinity(0)))
    except Exception:
        pass
    d = model_dims(a.readout)
    om = O.Model(d, synth.make_model(d, 2016))
    rows = 96  # per step: 1 encode + 96 parents x cands (~1 s of CPU work)
    for w in range(a.warmup):
        oracle_sample(om, d, a, rows, seed=shard_seed(0, w))
    tot_t, tot_n = 0.0, 0
    for k in range(a.steps):
        dt, n = oracle_sample(om, d, a, rows, seed=shard_seed(0, 1000 + k))
        tot_t += dt
        tot_n += n
    v = tot_n / tot_t
    cores = cpu_threads()
    sample = f"per step: encode 1 source (Tx={a.src_len}) + {rows} injected parents x {a.cands} words (float64 numpy)"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1000 * tot_t / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload_config(a, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def parity_vs_oracle(M, om, d, a, rows: int, seeds, cands: int, tol: float) -> tuple:
    """(oracle seconds, word-scores, parity dict): oracle samples through the host C ABI and the oracle."""
    t, n = 0.0, 0
    worst, cnt, top_same, top_rows, top_tie_ok = 0.0, 0, 0, 0, True
    for sd in seeds:
        dt, m = oracle_sample(om, d, a, rows, seed=sd, cands=cands)
        t += dt
        n += m
        src, s, y, off, words, ref, ref_am, sess, oids = oracle_sample.last
        ctx = M.encode(src)
        lp, _, am = ctx.score_batch(ctx.inject_states(s, y), off, words)
        ctx.close()
        worst = max(worst, float(np.max(np.abs(lp.astype(np.float64) - ref))))
        cnt += len(lp)
        same = am == ref_am
        top_same += int(same.sum())
        top_rows += len(am)
        for i in np.nonzero(~same)[0]:  # a different top-1 must lie in the oracle's tie set (A21)
            row = sess.logprobs_full(oids[i])
            top_tie_ok = top_tie_ok and bool(row[am[i]] >= row.max() - 2 * tol)
    par = {"max_abs_dlogp": worst, "tol": tol, "ok": worst < tol and top_tie_ok, "word_scores": cnt,
           "top1_identical": f"{top_same}/{top_rows}", "top1_in_oracle_tie_set": top_tie_ok,
           "vs": "float64 oracle, same inputs through the host C ABI"}
    return t, n, par


def cpu_baseline(a, M=None) -> tuple:
    """(cpu_baseline dict, parity dict or None): the oracle timed on two full steps of the workload;
    the same two steps through the GPU path (host C ABI) give the run's own max |dlogp|."""
    import oracle as O
    d = model_dims(a.readout)
    om = O.Model(d, synth.make_model(d, 2016))
    oracle_sample(om, d, a, 16, seed=7)  # warm BLAS
    tol = 2e-2 if a.precision == "bf16" else 1e-3
    if M is None:
        t, n = 0.0, 0
        for k in range(2):
            dt, m = oracle_sample(om, d, a, a.rows, seed=shard_seed(0, 5000 + k))
            t, n = t + dt, n + m
        par = None
    else:
        t, n, par = parity_vs_oracle(M, om, d, a, a.rows, [shard_seed(0, 5000 + k) for k in range(2)], a.cands, tol)
    base = {"value": n / t, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
            "sample": f"2 full steps of the workload (encode Tx={a.src_len} + {a.rows} parents x {a.cands} words), "
                      f"float64 numpy oracle, {t:.1f} s"}
    return base, par, om


# ------------------------------------------------------------------------------------- GPU arm
def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return {"bf16_tflops": j.get("bf16_tflops"), "bf16_tflops_sustained": j.get("bf16_tflops_sustained"),
                "hbm_gbs": j.get("hbm_gbs"), "source": "measured (MEASURED_PEAKS.json)"}
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": None, "hbm_gbs": 6650.0,
            "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic() -> tuple:
    """dram read + write bytes per launch of the vocab GEMM from the committed `ncu --set full` summary
    (ncu cannot run inside the timed bench; the file names the capture)."""
    for p in (os.path.join(ROOT, "profiles", "r02", "vocab_ncu.json"), os.path.join(ROOT, "profiles", "vocab_gemm_ncu.json")):
        if os.path.exists(p):
            with open(p) as f:
                j = json.load(f)
            return j.get("dram_bytes_per_launch"), os.path.relpath(p, ROOT)
    return None, None


class Workload:
    """Seeded device-resident inputs of a rank's shard (NSETS batches) and the timed step."""
    NSETS = 4

    def __init__(self, M, d, a, rank, cands, torch):
        self.M, self.d, self.R, self.Cn, self.Tx = M, d, a.rows, cands, a.src_len
        self.srcs, self.states, self.ys, self.words, self.off = [], [], [], [], None
        for i in range(self.NSETS):
            sd = shard_seed(rank, i)
            self.srcs.append(synth.make_source(d.vocab_src, self.Tx - 1, seed=sd))
            s, y = synth.make_states(self.R, d.dim_hid, d.vocab_tgt, seed=sd + 1)
            off, w = synth.make_candidates(self.R, cands, d.vocab_tgt, seed=sd + 2)
            self.states.append(s)
            self.ys.append(y)
            self.words.append(w)
            self.off = off
        cu = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
        self.dsrc = [cu(x) for x in self.srcs]
        self.dstates = [cu(x) for x in self.states]
        self.dy = [cu(x) for x in self.ys]
        self.dwords = [cu(x) for x in self.words]
        self.doff = cu(self.off)
        R, nc = self.R, self.R * cands
        self.ids = torch.empty(R, dtype=torch.int32, device="cuda")
        self.logp = torch.empty(nc, dtype=torch.float32, device="cuda")
        self.child = torch.empty(nc, dtype=torch.int32, device="cuda")
        self.amax = torch.empty(R, dtype=torch.int32, device="cuda")

    def step_dev(self, i: int) -> None:
        j = i % self.NSETS
        ctx = self.M.encode_dev(self.dsrc[j].data_ptr(), self.Tx)
        ctx.inject_states_dev(self.R, self.dstates[j].data_ptr(), self.dy[j].data_ptr(), self.ids.data_ptr())
        ctx.score_batch_dev(self.R, self.ids.data_ptr(), self.doff.data_ptr(), self.R * self.Cn,
                            self.dwords[j].data_ptr(), self.logp.data_ptr(), self.child.data_ptr(),
                            self.amax.data_ptr())
        ctx.close()

    def step_host(self, j: int, pinned) -> tuple:
        ctx = self.M.encode(pinned["src"][j])
        pids = ctx.inject_states(pinned["s"][j], pinned["y"][j])
        out = ctx.score_batch(pids, pinned["off"], pinned["w"][j])
        ctx.close()
        return out


def timed_dev(wl, a, stream, flush, dist, torch, nmt):
    """W warm-up steps, then K steps bracketed by barrier + synchronize, per-step CUDA events on the
    model stream with an L2 flush (outside the events) before each step."""
    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(a.warmup):
        wl.step_dev(i)
    torch.cuda.synchronize()
    assert torch.isfinite(wl.logp).all().item(), "non-finite log-probs"
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    barrier()
    n0 = nmt.launch_count()
    for i in range(a.steps):
        flush.zero_()
        ev[i][0].record(stream)
        wl.step_dev(i)
        ev[i][1].record(stream)
    barrier()
    launches = nmt.launch_count() - n0
    t_local = sum(e0.elapsed_time(e1) for e0, e1 in ev) / 1000.0
    return t_local, launches


def run_ours(a, rank: int, world: int, dist) -> None:
    import torch
    from paper_1605_04809_b200 import nmt

    dev = int(os.environ.get("LOCAL_RANK", 0))
    if dev >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{dev} but only {torch.cuda.device_count()} GPU(s) exist")
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    d = model_dims(a.readout)
    params = synth.params_bytes(d, synth.make_model(d, 2016))
    M = nmt.Model(params, precision=a.precision, device=dev, max_src_len=64, stream=stream.cuda_stream)
    R, Cn, Tx = a.rows, a.cands, a.src_len
    wl = Workload(M, d, a, rank, Cn, torch)
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")
    # ---------------- timed region (value): per-step CUDA events on the model stream, L2 flushed between steps
    M.profile(0)
    with ClockSampler(dev) as clk:
        t_local, launches = timed_dev(wl, a, stream, flush, dist, torch, nmt)
    last_set = (a.steps - 1) % Workload.NSETS
    dev_logp = wl.logp.cpu().numpy().copy()  # the last timed step's output (compared with the host path below)
    # ---------------- the same W + K steps again with CUDA events around every vocab-GEMM launch (on the model
    # stream): the dominant kernel's live duration for the roofline.  Events between PDL-chained kernels
    # serialise them (measured +13 us per step), so they stay out of the region that gives `value`.
    M.profile(1)
    M.profile_read()
    t_local_ev, _ = timed_dev(wl, a, stream, flush, dist, torch, nmt)
    stage_ms, stage_cnt = M.profile_read()
    M.profile(0)
    t_max = reduce_max(t_local, dist)
    total_scores = reduce_sum(float(R * Cn * a.steps), dist)
    value = total_scores / t_max
    clocks = clk.summary()
    # roofline of the dominant kernel (vocabulary GEMM + fused log-sum-exp), live from the timed region
    vi = nmt.STAGES.index("vocab_gemm_lse")
    vocab_ms = stage_ms[vi] / max(1, stage_cnt[vi])
    flops = 2.0 * R * d.vocab_tgt * d.dim_emb
    achieved = flops / (vocab_ms / 1000.0) / 1e12 if vocab_ms > 0 else float("nan")
    peaks = measured_peaks()
    traffic, traffic_src = ncu_traffic()
    roof = {"kernel": "k_gemm<256,6,EPI_LSE,pair> (CTA-pair vocab GEMM + online log-sum-exp)", "bound": "tensor",
            "achieved": achieved, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
            "frac": achieved / peaks["bf16_tflops"], "traffic": traffic,
            "traffic_source": f"ncu --set full capture summarised in {traffic_src} (not measured in this run)",
            "peak_source": peaks["source"] + " bf16 burst", "algorithmic_flops_per_launch": flops,
            "avg_launch_ms": vocab_ms, "share_of_step": vocab_ms / (1000.0 * t_local_ev / a.steps),
            "timing": "CUDA events around each launch on the model stream over a second pass of the same W + K "
                      "steps (events there cost the PDL overlap: ms_per_step_with_events)",
            "ms_per_step_with_events": 1000.0 * t_local_ev / a.steps}
    sf = step_flops(R, Tx, d)
    ms_step = 1000.0 * t_max / a.steps
    step_roof = {"algorithmic_flops_per_step": sf["per_step"], "per_row": sf["per_row"], "encoder": sf["encoder"],
                 "achieved_tflops": sf["per_step"] / (ms_step / 1000.0) / 1e12,
                 "frac_of_bf16_peak": sf["per_step"] / (ms_step / 1000.0) / 1e12 / peaks["bf16_tflops"],
                 "executed_flops_per_step": sf["executed_per_step"],
                 "executed_tflops": sf["executed_per_step"] / (ms_step / 1000.0) / 1e12,
                 "note": "whole step (encoder + decoder + vocabulary) against the dense bf16 burst peak; "
                         "algorithmic = the method's contractions as written (SURVEY 8(a)), executed = what the "
                         "library computes (projections precomputed at load, c.W as alpha.(ctx.W), DESIGN A31)"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16" if a.precision == "bf16" else "bf16x3",
            "data": "synthetic (seeded random-init cGRU weights, Zipf ids, injected parent states)",
            "config": workload_config(a, world), "roofline": roof, "step_roofline": step_roof,
            "gpu_launches": int(launches), "gpu_launches_per_step": launches / a.steps, "clocks": clocks,
            "rows_per_s": value / Cn}  # unique decoder steps (rows) per second
    if dist is not None:
        line["comm"] = comm_info(dist, torch)
    # ---------------- optional per-stage breakdown (separate untimed pass)
    if a.stages:
        M.profile(2)
        M.profile_read()
        for i in range(10):
            wl.step_dev(i)
        ms, cnt = M.profile_read()
        M.profile(0)
        line["stages_ms_per_step"] = {n: ms[k] / 10 for k, n in enumerate(nmt.STAGES) if cnt[k]}
    # ---------------- e2e: the host C-ABI (pinned host inputs in, results out, every step)
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
    pinned = {"src": [pin(x) for x in wl.srcs], "s": [pin(x) for x in wl.states], "y": [pin(x) for x in wl.ys],
              "w": [pin(x) for x in wl.words], "off": pin(wl.off)}
    host_lp = wl.step_host(last_set, pinned)[0]
    line["dev_vs_host"] = {"bitwise_equal": bool(np.array_equal(dev_logp.view(np.uint32), host_lp.view(np.uint32))),
                           "what": "log-probs of the last timed device step vs the host C ABI on the same inputs"}
    if not a.no_e2e:
        for i in range(a.warmup):
            wl.step_host(i % Workload.NSETS, pinned)
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        for i in range(a.steps):
            flush.zero_()
            ev2[i][0].record(stream)
            wl.step_host(i % Workload.NSETS, pinned)
            ev2[i][1].record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t2 = reduce_max(sum(e0.elapsed_time(e1) for e0, e1 in ev2) / 1000.0, dist)
        h2d = Tx * 4 + R * d.dim_hid * 4 + R * 4 + R * 8 + (R + 1) * 4 + R * Cn * 4
        d2h = R * 8 + R * Cn * 4 + R * Cn * 8 + R * 4
        line["e2e"] = {"value": total_scores / t2, "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h,
                       "path": "nmt_encode + nmt_inject_states + nmt_score_batch (host arrays, pinned)"}
    om = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"], line["parity"], om = cpu_baseline(a, M)
    # ---------------- variants: primary C2 (1 candidate per row) and FP32CLASS, each with its own parity
    if not a.no_variants:
        line["variants"] = variants(a, M, params, d, rank, world, dist, stream, flush, torch, nmt, om)
    M.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


def variants(a, M, params, d, rank, world, dist, stream, flush, torch, nmt, om) -> dict:
    import copy
    out = {}
    steps = max(3, min(a.steps, 10))
    for name, prec, cands in (("c2_1cand_bf16", "bf16", 1), ("fp32class", "fp32class", a.cands)):
        if prec == a.precision and cands == a.cands:
            continue
        va = copy.copy(a)
        va.steps, va.warmup, va.cands, va.precision = steps, max(3, min(a.warmup, 5)), cands, prec
        Mv = M if prec == a.precision else nmt.Model(params, precision=prec, device=torch.cuda.current_device(),
                                                       max_src_len=64, stream=stream.cuda_stream)
        wl = Workload(Mv, d, va, rank, cands, torch)
        t_local, launches = timed_dev(wl, va, stream, flush, dist, torch, nmt)
        t_max = reduce_max(t_local, dist)
        v = reduce_sum(float(va.rows * cands * steps), dist) / t_max
        r = {"value": v, "unit": UNIT, "rows_per_s": v / cands, "ms_per_step": 1000.0 * t_max / steps,
             "steps": steps, "warmup": va.warmup, "precision": prec, "cands_per_row": cands,
             "dtype": "bf16" if prec == "bf16" else "bf16x3"}
        if om is not None and rank == 0:
            tol = 2e-2 if prec == "bf16" else 1e-3
            _, _, r["parity"] = parity_vs_oracle(Mv, om, d, va, 256, [shard_seed(0, 7000)], cands, tol)
            r["parity"]["sample"] = "256 parents of one step"
        out[name] = r
        if Mv is not M:
            Mv.close()
    return out


def comm_info(dist, torch) -> dict:
    """What the process group really is (rank count from the communicator, NCCL version, init lines)."""
    info = {"backend": dist.get_backend(), "world_size": dist.get_world_size()}
    try:
        v = torch.cuda.nccl.version()
        info["nccl_version"] = ".".join(str(x) for x in v) if isinstance(v, tuple) else str(v)
    except Exception:
        pass
    lines = []
    for f in sorted(glob.glob(os.environ.get("NMT_NCCL_LOG_GLOB", "/tmp/nmt_bench_nccl.*.log"))):
        try:
            lines += [ln.strip() for ln in open(f) if "nranks" in ln or "Init COMPLETE" in ln]
        except OSError:
            pass
    info["nccl_init_lines"] = lines[:16]
    return info


# ------------------------------------------------------------------------------------- C4 ensemble
def run_ensemble(a, rank: int, world: int, dist) -> None:
    """C4: M members (seeds 2016..2016+M-1) score the same C2 batch; per-word log-probs are combined
    (mode 0, lambda = 1/M) on member 0.  N >= M GPUs: groups of M ranks, one member per GPU, NCCL;
    N == 1: all members on the GPU, one host thread each, in-process communicator."""
    import torch
    from paper_1605_04809_b200 import nmt
    Mn = a.ensemble
    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    d = model_dims(a.readout)
    if world == 1:
        members, group = list(range(Mn)), 0
    elif world % Mn == 0:
        members, group = [rank % Mn], rank // Mn
    else:
        raise SystemExit(f"--ensemble {Mn} needs 1 GPU or a multiple of {Mn} GPUs (got {world})")
    streams = [torch.cuda.Stream(device=dev) for _ in members]
    models = [nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016 + m)), precision=a.precision, device=dev,
                        max_src_len=64, stream=streams[i].cuda_stream) for i, m in enumerate(members)]
    if world == 1:
        comms = nmt.Ensemble.local(Mn)
    else:
        obj = [None] * world  # every group leader makes its NCCL id; the group's ranks take their leader's
        dist.all_gather_object(obj, nmt.Ensemble.unique_id() if rank % Mn == 0 else None)
        ids = obj[group * Mn]
        comms = [nmt.Ensemble(Mn, rank % Mn, ids, dev)]
    wls = []
    for i, m in enumerate(members):
        with torch.cuda.stream(streams[i]):
            wls.append(Workload(models[i], d, a, group, a.cands, torch))  # the group's shard: same batch per member
    nc = a.rows * a.cands
    out = torch.empty(nc, dtype=torch.float32, device="cuda")

    def member_steps(i, k0, n):
        for k in range(k0, k0 + n):
            wls[i].step_dev(k)
            comms[i].combine(wls[i].logp.data_ptr(), nc, 1.0 / Mn, 0, 0,
                             out.data_ptr() if comms[i].rank == 0 else None, streams[i].cuda_stream)

    def run_all(k0, n):
        if len(members) == 1:
            member_steps(0, k0, n)
            return
        err = []

        def body(i):
            try:
                torch.cuda.set_device(dev)
                member_steps(i, k0, n)
            except BaseException as e:  # noqa: BLE001
                err.append(e)
        ts = [threading.Thread(target=body, args=(i,)) for i in range(len(members))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if err:
            raise err[0]

    run_all(0, a.warmup)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in members]
    ends = [torch.cuda.Event(enable_timing=True) for _ in members]
    n0 = nmt.launch_count()
    with ClockSampler(dev) as clk:
        for i in range(len(members)):
            starts[i].record(streams[i])
        run_all(a.warmup, a.steps)
        for i in range(len(members)):
            ends[i].record(streams[i])
        torch.cuda.synchronize()
    launches = nmt.launch_count() - n0
    t_local = max(starts[0].elapsed_time(e) for e in ends) / 1000.0
    t_max = reduce_max(t_local, dist)
    groups = max(1, world // Mn)
    total = float(groups * nc * a.steps)
    value = total / t_max
    ms_step = 1000.0 * t_max / a.steps
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16" if a.precision == "bf16" else "bf16x3",
            "data": "synthetic (seeded random-init cGRU weights, Zipf ids, injected parent states)",
            "config": workload_config(a, world), "gpu_launches": int(launches), "clocks": clk.summary(),
            "combined_word_scores": "value counts each combined (parent, word) log-prob once",
            "member_word_scores_per_s": value * Mn}
    if dist is not None:
        line["comm"] = comm_info(dist, torch)
    if rank == 0 and not a.no_cpu_baseline:
        line["parity"] = ensemble_parity(a, models, comms, members, streams, d, torch, nmt) if world == 1 else None
    for c in comms:
        c.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


def ensemble_parity(a, models, comms, members, streams, d, torch, nmt) -> dict:
    """The combined log-probs of 64 rows of a batch vs the oracle ensemble (float64 members)."""
    import oracle as O
    Mn = len(members)
    R = 64
    src = synth.make_source(d.vocab_src, a.src_len - 1, seed=9000)
    s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=9001)
    off, words = synth.make_candidates(R, a.cands, d.vocab_tgt, seed=9002)
    nc = len(words)
    res = {}

    def body(i):
        torch.cuda.set_device(torch.cuda.current_device())
        c = models[i].encode(src)
        lp, _, _ = c.score_batch(c.inject_states(s, y), off, words)
        c.close()
        with torch.cuda.stream(streams[i]):
            dl = torch.from_numpy(lp).cuda()
            o = torch.empty_like(dl)
            comms[i].combine(dl.data_ptr(), nc, 1.0 / Mn, 0, 0, o.data_ptr() if i == 0 else None, streams[i].cuda_stream)
        streams[i].synchronize()
        if i == 0:
            res["out"] = o.cpu().numpy()

    ts = [threading.Thread(target=body, args=(i,)) for i in range(Mn)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    refs = []
    for m in members:
        om = O.Model(d, synth.make_model(d, 2016 + m))
        sess = O.Session(om, src)
        ids = [sess.inject_state(s[i], int(y[i])) for i in range(R)]
        refs.append(sess.score_batch(ids, off, words)[0])
    ref = O.ensemble_combine(refs, [1.0 / Mn] * Mn, 0)
    tol = 2e-2 if a.precision == "bf16" else 1e-3
    err = float(np.max(np.abs(res["out"] - ref)))
    return {"max_abs_dlogp_combined": err, "tol": tol, "ok": err < tol, "word_scores": nc,
            "vs": f"float64 oracle ensemble of the {Mn} members (mode 0), 64 parents of one batch"}


# ------------------------------------------------------------------------------------- launcher
def relaunch_under_torchrun(a, argv) -> int:
    """`python bench.py --gpus N` without torchrun: start N ranks with torchrun (one per GPU) and
    relay rank 0's JSON line."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]
    env = dict(os.environ)
    env["NMT_BENCH_LAUNCHED"] = "1"
    return subprocess.call(cmd, env=env)


def main(argv=None) -> None:
    argv = sys.argv[1:] if argv is None else argv
    a = parse_args(argv)
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        sys.exit(relaunch_under_torchrun(a, argv))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")
    dist = None
    if world > 1 and a.impl == "ours":
        import torch
        import torch.distributed as tdist
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/nmt_bench_nccl.%h.%p.log")
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
        dist = tdist
        dist.barrier()
    if a.impl == "reference":
        run_reference(a, rank, world)
    elif a.ensemble:
        run_ensemble(a, rank, world, dist)
    else:
        run_ours(a, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
