"""Summarise one `ncu --set full` capture (raw page) into a small JSON: duration, DRAM traffic,
L2->SM traffic, tensor/XU pipe and issue utilisation, top stall reasons."""
import csv
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "l2_to_sm_GB": "l1tex__m_xbar2l1tex_read_bytes.sum",
    "l2_to_sm_pct_peak": "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed",
    "tensor_mem_cycles_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "tensor_mem_cycles_pct_elapsed": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "hmma_subpipe_active_cycles_realtime": "TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}


def main(rep, out, label):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader([ln for ln in raw.splitlines() if ln.startswith('"')]))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    res = {"kernel": d.get("Kernel Name", label), "label": label, "source": rep}
    for k, m in KEYS.items():
        v = d.get(m)
        try:
            v = float(v)
        except (TypeError, ValueError):
            pass
        res[k] = v
    # normalise byte units to MB / GB
    for k, m, scale in [("dram_read_MB", "dram__bytes_read.sum", "Mbyte"), ("dram_write_MB", "dram__bytes_write.sum", "Mbyte"),
                        ("l2_to_sm_GB", "l1tex__m_xbar2l1tex_read_bytes.sum", "Gbyte")]:
        unit = u.get(m, "")
        f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        target = {"Mbyte": 1e6, "Gbyte": 1e9}[scale]
        if isinstance(res[k], float):
            res[k] = res[k] * f / target
    res["dram_bytes_per_launch"] = (res["dram_read_MB"] + res["dram_write_MB"]) * 1e6
    st = sorted(((float(v), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                 for k, v in d.items() if "issue_stalled" in k and k.endswith("per_issue_active.ratio")
                 and v.replace(".", "", 1).isdigit()), reverse=True)
    res["top_stalls"] = {k: round(v, 3) for v, k in st[:5]}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
