#!/usr/bin/env python
"""Stall breakdown (warps stalled per issued instruction) per kernel of an ncu report.

    python tools/ncu_stalls.py gpurun_out/prof_<tag>.ncu-rep
"""
import csv
import io
import subprocess
import sys

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
pre = "smsp__average_warps_issue_stalled_"
for row in rows[2:]:
    d = dict(zip(h, row))
    vals = []
    for n, v in d.items():
        if n.startswith(pre):
            try:
                vals.append((float(v.replace(",", "")), n[len(pre):].replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    vals.sort(reverse=True)
    print(d.get("Kernel Name", "")[:40], " ".join(f"{n}={v:.2f}" for v, n in vals[:7]))
