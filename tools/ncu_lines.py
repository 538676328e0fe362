#!/usr/bin/env python
"""Per-CUDA-source-line instruction counts and stall samples from an ncu report
(needs -lineinfo):  python tools/ncu_lines.py gpurun_out/prof_<tag>.ncu-rep [N]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kfilter = sys.argv[3:4]
txt = subprocess.run(["ncu", "-i", rep] + (["-k", "regex:" + kfilter[0]] if kfilter else []) + ["--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = defaultdict(lambda: [0, 0, ""])
cur = ("?", "?")
fname = "?"
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a CUDA source line row
        cur = (fname, r[0])
        agg[cur][2] = r[1].strip()[:80]
    try:
        w = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        n = int(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    agg[cur][0] += n
    agg[cur][1] += w
ti = sum(v[0] for v in agg.values()) or 1
tw = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {ti / 1e6:.1f}M, stall samples {tw}")
for (f, ln), (n, w, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{n / 1e6:7.2f}M {100 * n / ti:5.1f}%i {100 * w / tw:5.1f}%s {f}:{ln:>4} {s}")
