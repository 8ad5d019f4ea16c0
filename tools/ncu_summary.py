"""Summarise an ncu report (--set full) into profiles/<name>.json: one entry per profiled kernel launch."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]


def summarise(rep: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append({k: (d[k] + (" " + u[k] if u.get(k) else "")) for k in KEYS if k in d})
    return out


if __name__ == "__main__":
    rep, dst = sys.argv[1], sys.argv[2]
    res = summarise(rep)
    json.dump({"report": rep, "command": sys.argv[3] if len(sys.argv) > 3 else None, "launches": res},
              open(dst, "w"), indent=1)
    for l in res:
        print(json.dumps(l))
