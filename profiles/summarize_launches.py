"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of bench.py into per-step shares.
The list is cold-cache and serialised: compare SHARES of the step, not absolute times."""
import csv
import json
import re
import sys
from collections import OrderedDict


def short(name: str) -> str:
    m = re.search(r"nmt::(k_\w+)(<[^>]*>)?", name)
    if not m:
        return "torch:" + re.sub(r"\(.*", "", name)[-40:]
    base = m.group(1)
    if base == "k_gemm":
        base += m.group(2).replace("(int)", "")
    if base == "k_enc_recur":
        base = "k_enc_recur"
    return base


def main(path: str, out_json: str) -> None:
    lines = [ln for ln in open(path) if ln.startswith('"')]  # drop ==PROF== / ==WARNING== lines
    rows = list(csv.DictReader(lines))
    launches = [(short(r["Kernel Name"]), float(r["Metric Value"]) / 1000.0) for r in rows
                if r["Metric Name"] == "gpu__time_duration.sum"]
    # a step starts at k_enc_gather; keep the last complete step
    starts = [i for i, (n, _) in enumerate(launches) if n.startswith("k_enc_recur")]
    i0 = starts[-2] if len(starts) >= 2 else starts[-1]
    i1 = starts[-1] if len(starts) >= 2 else len(launches)
    if "--step" in sys.argv:  # the k-th step of the list (bench.py appends its variants' steps after the headline's)
        k = int(sys.argv[sys.argv.index("--step") + 1])
        i0, i1 = starts[k], starts[k + 1]
    # a step = the launches from one encoder recurrence to the next (encode + inject + score)
    step = [x for x in launches[i0 - 1:i1 - 1] if not x[0].startswith("torch:")]
    tot = sum(t for _, t in step)
    agg = OrderedDict()
    for n, t in step:
        agg.setdefault(n, [0.0, 0])
        agg[n][0] += t
        agg[n][1] += 1
    table = [{"kernel": n, "launches": c, "us": round(t, 2), "share": round(t / tot, 4)} for n, (t, c) in agg.items()]
    res = {"source": path, "step_kernels": len(step), "step_us_serialised": round(tot, 1), "table": table,
           "sequence": [[n, round(t, 2)] for n, t in step]}
    json.dump(res, open(out_json, "w"), indent=1)
    for r in sorted(table, key=lambda r: -r["us"]):
        print(f'{r["kernel"]:34s} {r["launches"]:3d} {r["us"]:9.2f} us  {100 * r["share"]:5.1f} %')
    print(f"step: {len(step)} launches, {tot:.1f} us serialised")
    if "--seq" in sys.argv:
        for n, t in step:
            print(f"  {n:34s} {t:8.2f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])  # [--seq]: also print the step's launches in order; [--step k]: the k-th step
