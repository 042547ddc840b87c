#!/usr/bin/env python
"""bench.py - hypothesis word-scores/s of the batched cGRU scorer on B200 (BASELINE.json metric).

One step = one pass of the whole hot path (SURVEY §8(a) E1-E7 + D0-D9) over one batch of the C2
En->Ru workload (BASELINE.json configs[1]): encode one synthetic source sentence (Tx = 50 incl. EOS),
inject R = 1024 synthetic parent states, and score R x 3 candidate words (3072 word-scores) through
nmt_score_batch (device planner -> GRU1 -> attention -> GRU2 -> readout -> vocab GEMM + fused
log-softmax -> gather).  `value` times the device-resident C-ABI path (nmt_*_dev, inputs already in
HBM); `e2e` times the host API (pinned host inputs copied in, results copied out) every step.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  N > 1: torchrun, one rank per GPU, sentences sharded (weak scaling, no collective on the data path).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--stages", action="store_true", help="add a per-stage CUDA-event breakdown (untimed pass)")
    return ap.parse_args(argv)


def model_dims(readout: str) -> synth.Dims:
    return synth.Dims(500, 1024, 50000, 100000, readout)


def workload_config(a, n_gpus: int) -> dict:
    return {"workload": f"C2 En->Ru: encode 1 source (Tx={a.src_len}) + score {a.rows} injected parents x "
                        f"{a.cands} candidate words per step",
            "dim_emb": 500, "dim_hid": 1024, "vocab_tgt": 100000, "src_len": a.src_len, "rows": a.rows,
            "cands_per_row": a.cands, "precision": a.precision, "readout": a.readout,
            "l2": "flushed before every timed step (256 MiB write)",
            "parallelism": f"{n_gpus} GPU(s), sentence sharding, no collective on the data path"}


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
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
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


def oracle_sample(om, d, a, rows: int, seed: int) -> tuple:
    """One bounded sample of the step on the host: encode 1 source + `rows` parents x cands."""
    import oracle as O
    src = synth.make_source(d.vocab_src, a.src_len - 1, seed=seed)
    s, y = synth.make_states(rows, d.dim_hid, d.vocab_tgt, seed=seed + 1)
    off, words = synth.make_candidates(rows, a.cands, d.vocab_tgt, seed=seed + 2)
    t0 = time.perf_counter()
    sess = O.Session(om, src)
    ids = [sess.inject_state(s[i], int(y[i])) for i in range(rows)]
    lp, _, am = sess.score_batch(ids, off, words)
    dt = time.perf_counter() - t0
    assert np.all(np.isfinite(lp))
    oracle_sample.last = (src, s, y, off, words, lp, am, sess, ids)  # (inputs and results, for the parity check)
    return dt, rows * a.cands


def run_reference(a, rank: int, world: int) -> None:
    """--impl reference: the float64 oracle on the host cores, bounded samples of the same workload."""
    if rank != 0:
        return
    import oracle as O
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


def cpu_baseline(a, M=None) -> tuple:
    """(cpu_baseline dict, parity dict or None): the oracle timed on two full steps of the workload;
    the same two steps through the GPU path (host C ABI) give the run's own max |dlogp|."""
    import oracle as O
    d = model_dims(a.readout)
    om = O.Model(d, synth.make_model(d, 2016))
    oracle_sample(om, d, a, 16, seed=7)  # warm BLAS
    rows = a.rows
    t, n = 0.0, 0
    worst, cnt, top_same, top_rows, top_tie_ok = 0.0, 0, 0, 0, True
    tol = 2e-2 if a.precision == "bf16" else 1e-3
    for k in range(2):
        dt, m = oracle_sample(om, d, a, rows, seed=shard_seed(0, 5000 + k))
        t += dt
        n += m
        if M is not None:  # (untimed) the same inputs through the CUDA path
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
    base = {"value": n / t, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
            "sample": f"2 full steps of the workload (encode Tx={a.src_len} + {rows} parents x {a.cands} words), "
                      f"float64 numpy oracle, {t:.1f} s"}
    par = None
    if M is not None:
        par = {"max_abs_dlogp": worst, "tol": tol, "ok": worst < tol and top_tie_ok, "word_scores": cnt,
               "top1_identical": f"{top_same}/{top_rows}", "top1_in_oracle_tie_set": top_tie_ok,
               "vs": "float64 oracle on the cpu_baseline sample (same inputs), host C ABI"}
    return base, par


# ------------------------------------------------------------------------------------- GPU arm
def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return {"bf16_tflops": j.get("bf16_tflops"), "hbm_gbs": j.get("hbm_gbs"), "source": "measured"}
    return {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic() -> float | None:
    p = os.path.join(ROOT, "profiles", "vocab_gemm_ncu.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j.get("dram_bytes_per_launch")
    return None


def run_ours(a, rank: int, world: int, dist) -> None:
    import torch
    from paper_1605_04809_b200 import nmt

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    d = model_dims(a.readout)
    params = synth.params_bytes(d, synth.make_model(d, 2016))
    M = nmt.Model(params, precision=a.precision, device=dev, max_src_len=64, stream=stream.cuda_stream)
    del params
    R, Cn, Tx = a.rows, a.cands, a.src_len
    NSETS = 4
    # device-resident inputs (value leg): NSETS seeded batches of this rank's shard
    srcs, states, ys, words = [], [], [], []
    for i in range(NSETS):
        sd = shard_seed(rank, i)
        srcs.append(synth.make_source(d.vocab_src, Tx - 1, seed=sd))
        s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=sd + 1)
        off, w = synth.make_candidates(R, Cn, d.vocab_tgt, seed=sd + 2)
        states.append(s)
        ys.append(y)
        words.append(w)
    dsrc = [torch.from_numpy(x).cuda() for x in srcs]
    dstates = [torch.from_numpy(x).cuda() for x in states]
    dy = [torch.from_numpy(x).cuda() for x in ys]
    dwords = [torch.from_numpy(x).cuda() for x in words]
    doff = torch.from_numpy(off).cuda()
    ids = torch.empty(R, dtype=torch.int32, device="cuda")
    logp = torch.empty(R * Cn, dtype=torch.float32, device="cuda")
    child = torch.empty(R * Cn, dtype=torch.int32, device="cuda")
    amax = torch.empty(R, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")

    def step_dev(i: int) -> None:
        j = i % NSETS
        ctx = M.encode_dev(dsrc[j].data_ptr(), Tx)
        ctx.inject_states_dev(R, dstates[j].data_ptr(), dy[j].data_ptr(), ids.data_ptr())
        ctx.score_batch_dev(R, ids.data_ptr(), doff.data_ptr(), R * Cn, dwords[j].data_ptr(), logp.data_ptr(),
                            child.data_ptr(), amax.data_ptr())
        ctx.close()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(a.warmup):
        step_dev(i)
    torch.cuda.synchronize()
    assert torch.isfinite(logp).all().item(), "non-finite log-probs"
    # ---------------- timed region (value): per-step CUDA events on the model stream, L2 flushed between steps
    M.profile(1)
    M.profile_read()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    barrier()
    n0 = nmt.launch_count()
    with ClockSampler(dev) as clk:
        for i in range(a.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step_dev(i)
            ev[i][1].record(stream)
        barrier()
    launches = nmt.launch_count() - n0
    stage_ms, stage_cnt = M.profile_read()
    M.profile(0)
    t_local = sum(e0.elapsed_time(e1) for e0, e1 in ev) / 1000.0
    t_max = reduce_max(t_local, dist)
    total_scores = reduce_sum(float(R * Cn * a.steps), dist)
    value = total_scores / t_max
    clocks = clk.summary()
    # roofline of the dominant kernel (vocabulary GEMM + fused log-sum-exp), live from the timed region
    vocab_ms = stage_ms[nmt.STAGES.index("vocab_gemm_lse")] / max(1, stage_cnt[nmt.STAGES.index("vocab_gemm_lse")])
    flops = 2.0 * R * d.vocab_tgt * d.dim_emb
    achieved = flops / (vocab_ms / 1000.0) / 1e12
    peaks = measured_peaks()
    roof = {"kernel": "k_gemm<256,6,EPI_LSE,pair> (CTA-pair vocab GEMM + online log-sum-exp)", "bound": "tensor",
            "achieved": achieved, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
            "frac": achieved / peaks["bf16_tflops"], "traffic": ncu_traffic(),
            "peak_source": peaks["source"] + " bf16 burst", "algorithmic_flops_per_launch": flops,
            "avg_launch_ms": vocab_ms, "share_of_step": vocab_ms / (1000.0 * t_local / a.steps)}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1000.0 * t_max / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16" if a.precision == "bf16" else "bf16x3",
            "data": "synthetic (seeded random-init cGRU weights, Zipf ids, injected parent states)",
            "config": workload_config(a, world), "roofline": roof, "gpu_launches": int(launches),
            "gpu_launches_per_step": launches / a.steps, "clocks": clocks,
            "rows_per_s": value / a.cands}  # unique decoder steps (rows) per second
    # ---------------- optional per-stage breakdown (separate untimed pass)
    if a.stages:
        M.profile(2)
        M.profile_read()
        for i in range(10):
            step_dev(i)
        ms, cnt = M.profile_read()
        M.profile(0)
        line["stages_ms_per_step"] = {n: ms[k] / 10 for k, n in enumerate(nmt.STAGES) if cnt[k]}
    # ---------------- e2e: the host C-ABI (pinned host inputs in, results out, every step)
    if not a.no_e2e:
        pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
        hsrc = [pin(x) for x in srcs]
        hstates = [pin(x) for x in states]
        hy = [pin(x) for x in ys]
        hwords = [pin(x) for x in words]
        hoff = pin(off)

        def step_host(i: int) -> int:
            j = i % NSETS
            ctx = M.encode(hsrc[j])
            pids = ctx.inject_states(hstates[j], hy[j])
            lp, ch, am = ctx.score_batch(pids, hoff, hwords[j])
            ctx.close()
            return int(np.isfinite(lp).sum())

        for i in range(a.warmup):
            step_host(i)
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        barrier()
        for i in range(a.steps):
            flush.zero_()
            ev2[i][0].record(stream)
            step_host(i)
            ev2[i][1].record(stream)
        barrier()
        t2 = reduce_max(sum(e0.elapsed_time(e1) for e0, e1 in ev2) / 1000.0, dist)
        h2d = Tx * 4 + R * d.dim_hid * 4 + R * 4 + R * 8 + (R + 1) * 4 + R * Cn * 4
        d2h = R * 8 + R * Cn * 4 + R * Cn * 8 + R * 4
        line["e2e"] = {"value": total_scores / t2, "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h,
                       "path": "nmt_encode + nmt_inject_states + nmt_score_batch (host arrays, pinned)"}
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"], line["parity"] = cpu_baseline(a, M)
    if rank == 0:
        print(json.dumps(line), flush=True)


def main(argv=None) -> None:
    a = parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        if a.impl == "ours":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
            tdist.init_process_group("nccl")
            dist = tdist
    if a.impl == "reference":
        run_reference(a, rank, world)
    else:
        run_ours(a, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
