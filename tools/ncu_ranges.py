#!/usr/bin/env python
"""Warp instructions of one kernel grouped by source-line ranges.
   python tools/ncu_ranges.py <rep> <kernel-substring> <file> name:lo-hi [name:lo-hi ...]"""
import csv, io, subprocess, sys
rep, kname, fname = sys.argv[1:4]
ranges = [(a.split(":")[0], *map(int, a.split(":")[1].split("-"))) for a in sys.argv[4:]]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = fn = None
tot = {r[0]: 0 for r in ranges}; tot["other"] = 0; allv = 0
for r in csv.reader(io.StringIO(txt)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": fn = r[1]; continue
    if fn and kname in fn and r[0].isdigit():
        try: v = int(r[7])
        except (ValueError, IndexError): continue
        allv += v
        ln = int(r[0]); hit = False
        if cur == fname:
            for name, lo, hi in ranges:
                if lo <= ln <= hi: tot[name] += v; hit = True; break
        if not hit: tot["other"] += v
for k, v in tot.items(): print(f"{k:12s} {v/1e6:8.2f}M  {100*v/max(allv,1):5.1f}%")
print(f"{'total':12s} {allv/1e6:8.2f}M")
