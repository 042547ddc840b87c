"""Diagnose the vocab GEMM's in-step vs isolated gap (VERDICT r01 "Next round" 8): the CTA-pair
LSE kernel alone at the bench shape (M = 1024, V = 100k -> 100096, K = 512), back to back with W_o
L2-warm, and with a 256 MiB L2 flush before every launch (W_o cold from HBM, as in the bench step).
Needs the diagnostic build (python -m paper_1605_04809_b200.build --diag)."""
import json
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["NMT_LIB_PATH"] = os.path.join(HERE, "paper_1605_04809_b200", "libnmt_diag.so")
sys.path.insert(0, HERE)
from paper_1605_04809_b200 import nmt  # noqa: E402

peak = json.load(open(os.path.join(HERE, "MEASURED_PEAKS.json")))["bf16_tflops"] if os.path.exists(
    os.path.join(HERE, "MEASURED_PEAKS.json")) else 1590.0
for R in (1024, 4096):
    fl = 2.0 * R * 100000 * 500
    for flush in (False, True):
        if flush:
            os.environ["NMT_BENCH_FLUSH"] = "1"
        else:
            os.environ.pop("NMT_BENCH_FLUSH", None)
        ms = nmt.bench_gemm(R, 100096, 512, epi=4, iters=30)
        print(json.dumps({"R": R, "l2": "flushed before every launch" if flush else "warm (back to back)",
                          "us": ms * 1e3, "tflops": fl / (ms * 1e-3) / 1e12, "frac": fl / (ms * 1e-3) / 1e12 / peak}),
              flush=True)
