"""Per-point DRAM bytes of the C5 sweep, for ncu.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file gpurun_out/sweep_dram.csv python tools/sweep_dram_ncu.py run
    python tools/sweep_dram_ncu.py parse gpurun_out/sweep_dram.csv > profiles/r2_sweep_dram.json

`run` launches every sweep point with T in {1e7, 1e8} once, each followed by a marker fill
kernel; `parse` attributes the libaolb200 kernels between markers to their point and sums
their DRAM bytes (compared in bench.py with the point's 128 B line floor)."""
import csv
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

TS = (10 ** 7, 10 ** 8)


def points():
    import bench
    sw = bench.SweepWorkload.__new__(bench.SweepWorkload)
    out = []
    for m in bench.SweepWorkload.POINTS_M:
        for kind in ("dense", "overlap", "gaps", "strided", "rowstride"):
            if kind in ("overlap", "strided", "rowstride") and m == 1:
                continue
            for T in TS:
                if (sw._geometry(m, kind, T)[0] + T * m) * 4 <= bench.SweepWorkload.MAX_FOOTPRINT:
                    out.append((m, kind, T))
    return sw, out


def run():
    import torch
    from paper_1105_4424_b200 import _capi
    sw, pts = points()
    sw.torch, sw.device = torch, torch.device("cuda", 0)
    marker = torch.empty(1024, device="cuda")        # no kernel: fills are the only markers
    st = int(torch.cuda.current_stream().cuda_stream)
    for i, (m, kind, T) in enumerate(pts):
        t = sw._make(m, kind, T)
        torch.cuda.synchronize()
        marker.fill_(float(i))
        _capi.launch(t["task"], 0, T, t["ptrs"], (), st)
        torch.cuda.synchronize()
        print(m, kind, T, t["plan"], flush=True)
        del t
        torch.cuda.empty_cache()
    marker.fill_(-1.0)
    torch.cuda.synchronize()


def parse(path):
    import bench
    sw, pts = points()
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    iid, iname, imet, ival = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    kern = {}
    order = []
    for r in rows[1:]:
        k = int(r[iid])
        if k not in kern:
            kern[k] = {"name": r[iname]}
            order.append(k)
        kern[k][r[imet]] = float(r[ival].replace(",", ""))
    out, cur = [], -1
    acc = None
    fills = [k for k in order if "fill" in kern[k]["name"].lower() or "FillFunctor" in kern[k]["name"]]
    if len(fills) == len(pts) + 2:        # an older run created the marker with torch.zeros (one more fill)
        order = order[order.index(fills[0]) + 1:]
    for k in order:
        d = kern[k]
        if "fill" in d["name"].lower() or "FillFunctor" in d["name"]:
            if acc is not None:
                out.append(acc)
            cur += 1
            if cur >= len(pts):
                acc = None
                continue
            m, kind, T = pts[cur]
            acc = {"m": m, "paving": kind, "T": T, "kernels": [], "dram_bytes": 0.0, "ns": 0.0}
            continue
        if acc is None or "aol::" not in d["name"]:     # inputs of the next point are made in between
            continue
        acc["kernels"].append(d["name"].split("(")[0])
        acc["dram_bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        acc["ns"] += d.get("gpu__time_duration.sum", 0)
    for a in out:
        a["floor_bytes"] = sw.line_floor_bytes(a["m"], a["paving"], a["T"])
        a["algorithmic_bytes"] = (sw._geometry(a["m"], a["paving"], a["T"])[1] + a["T"] * a["m"]) * 4
        a["dram_over_floor"] = a["dram_bytes"] / a["floor_bytes"]
        a["dram_over_algorithmic"] = a["dram_bytes"] / a["algorithmic_bytes"]
    print(json.dumps({"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                                "--clock-control none (one launch per point, cold-ish L2, serialised)",
                      "points": out}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        parse(sys.argv[2])
