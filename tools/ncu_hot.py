"""Top warp-stall SASS lines of an ncu report (source page), optionally grouped by CUDA source line.
  python tools/ncu_hot.py REPORT [N] [--inst]   (--inst: rank by instructions executed instead)"""
import csv
import subprocess
import sys
from collections import defaultdict

args = [a for a in sys.argv[1:] if not a.startswith("--")]
rep, n = args[0], int(args[1]) if len(args) > 1 else 30
COL = "Instructions Executed" if "--inst" in sys.argv else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, cur_line, cur_src = "", 0, ""
by_line = defaultdict(float)
sass = []
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        i_s = r.index(COL)
        continue
    if hdr is None or len(r) <= i_s:
        continue
    k = i_s + (len(r) - len(hdr))  # (unescaped quotes in a source line split it into extra columns)
    if r[0].strip():  # a source line row (aggregated over its instructions)
        cur_line, cur_src = r[0], r[1]
        if r[k] not in ("", "-"):
            by_line[(cur_file, cur_line, cur_src.strip()[:80])] += float(r[k])
    elif r[2].startswith("0x") and r[k] not in ("", "-"):  # an instruction row
        sass.append((float(r[k]), cur_file, cur_line, r[3][:70]))
tot = sum(by_line.values())
print(f"total samples {tot:.0f}")
print("-- by source line")
for (f, ln, src), v in sorted(by_line.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{100 * v / tot:5.1f}%  {f}:{ln}  {src}")
print("-- by SASS")
for v, f, ln, ins in sorted(sass, reverse=True)[:n // 2]:
    print(f"{100 * v / tot:5.1f}%  {f}:{ln}  {ins}")
