#!/usr/bin/env python
"""Per-CUDA-source-line instructions and stall samples of one kernel in an ncu report.

    python tools/ncu_lines_src.py gpurun_out/prof_<tag>.ncu-rep <kernel-substring> [top]
"""
import csv
import io
import subprocess
import sys

rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = fn = None
out = {}
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if fn and kname in fn and r[0].isdigit():
        try:
            out[(cur, int(r[0]))] = (int(r[4]), int(r[7]), r[1][:80])
        except (ValueError, IndexError):
            pass
ts = sum(v[0] for v in out.values()) or 1
ti = sum(v[1] for v in out.values()) or 1
print(f"stall samples {ts}, warp instructions {ti}")
for k, v in sorted(out.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]}:{k[1]:<5} stall {v[0] / ts:6.1%}  inst {v[1]:>10} {v[1] / ti:6.1%}  {v[2]}")
