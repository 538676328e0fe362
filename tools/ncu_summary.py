#!/usr/bin/env python
"""Summarise ncu artefacts brought back from the GPU box.

    python tools/ncu_summary.py launches gpurun_out/launches_<tag>.csv
    python tools/ncu_summary.py full gpurun_out/prof_<tag>.ncu-rep [--hot N]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "smsp__inst_executed.sum",
           "lts__t_bytes.sum", "l1tex__t_bytes.sum",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[hi + 1:]:
        d[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    out = []
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": k[:100], "launches": len(v), "avg_us": sum(v) / len(v) / 1e3,
                    "share": sum(v) / tot})
    return out


def full(path, hot=0):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, vals = rows[0], rows[1], rows[2:]
    res = []
    for v in vals:
        e = {"kernel": v[h.index("Kernel Name")][:100]}
        for m in METRICS:
            if m in h:
                e[m] = v[h.index(m)] + " " + units[h.index(m)]
        res.append(e)
    if hot:
        src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                              "sass"], capture_output=True, text=True).stdout
        srows = list(csv.reader(io.StringIO(src)))
        sh = srows[1]
        wi, ii, si = (sh.index("Warp Stall Sampling (All Samples)"),
                      sh.index("Instructions Executed"), sh.index("Source"))
        data = []
        for r in srows[2:]:
            try:
                data.append((int(r[wi]), int(r[ii]), r[si].strip()))
            except (ValueError, IndexError):
                pass
        tot = sum(d[0] for d in data) or 1
        res.append({"hot_sass": [f"{d[0] / tot:6.1%} {d[1]:>10} {d[2][:70]}"
                                 for d in sorted(data, key=lambda d: -d[0])[:hot]]})
    return res


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    hot = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[3] == "--hot" else 0
    out = launches(path) if kind == "launches" else full(path, hot)
    print(json.dumps(out, indent=1))
