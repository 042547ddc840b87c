"""Per-step phase breakdown of the encoder recurrence (NMT_ENC_TRACE diagnostic, CTA 0 thread 0)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1605_04809_b200 import nmt  # noqa: E402

d = synth.Dims(500, 1024, 50000, 100000, "maxout")
M = nmt.Model(synth.params_bytes(d, synth.make_model(d, 2016)), precision="bf16")
src = synth.make_source(d.vocab_src, 49, seed=1)
for _ in range(3):
    M.encode(src).close()
if "--plain" in sys.argv:  # (for ncu: no trace stamps)
    M.encode(src).close()
    sys.exit(0)
os.environ["NMT_ENC_TRACE"] = "1"
for _ in range(3):
    M.encode(src).close()
