"""Kernel timeline of bench steps (CUPTI activity records via torch.profiler): start / end of every kernel
relative to the step's first kernel, with its stream, so that overlap between the encoder stream and the
model stream (and PDL overlap between consecutive kernels) is visible.
  python tools/timeline.py [--steps 3] [--rows 1024]"""
import argparse
import json
import os
import re
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1605_04809_b200 import nmt  # noqa: E402


def short(name: str) -> str:
    m = re.search(r"(k_\w+)(<[^>]*>)?", name)
    if not m:
        return name[:40]
    return m.group(1) + (m.group(2).replace("(int)", "").replace("(bool)", "") if m.group(1) == "k_gemm" and m.group(2) else "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--cands", type=int, default=3)
    args = ap.parse_args()
    a = bench.parse_args(["--rows", str(args.rows), "--cands", str(args.cands)])
    d = bench.model_dims(a.readout)
    M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016)), precision=a.precision)
    wl = bench.Workload(M, d, a, 0, a.cands, torch)
    for i in range(5):
        wl.step_dev(i)
    torch.cuda.synchronize()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for i in range(args.steps):
            flush.fill_(float(i))  # (as bench.py: L2 flushed before each step)
            wl.step_dev(i)
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    steps, cur = [], []
    for e in ev:
        if "fill" in e["name"] or "elementwise" in e["name"].lower():
            if cur:
                steps.append(cur)
            cur = []
            continue
        cur.append(e)
    if cur:
        steps.append(cur)
    for k, st in enumerate(steps):
        t0 = st[0]["ts"]
        t_end = max(e["ts"] + e["dur"] for e in st)
        print(f"== step {k}: {len(st)} kernels, first start -> last end {t_end - t0:.1f} us")
        for e in st:
            print(f"  stream {e['args'].get('stream', '?'):>3}  {e['ts'] - t0:8.1f} .. {e['ts'] + e['dur'] - t0:8.1f}"
                  f"  ({e['dur']:6.1f})  {short(e['name'])}")


if __name__ == "__main__":
    main()
