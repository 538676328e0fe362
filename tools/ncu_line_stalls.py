#!/usr/bin/env python
"""Per-CUDA-line stall samples by reason for one kernel.
   python tools/ncu_line_stalls.py <rep> <kernel-substring> [top]"""
import csv, io, subprocess, sys
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr = None; fn = None; cur = None; out = []
for r in csv.reader(io.StringIO(txt)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": fn = r[1]; continue
    if r[0] == "Line No": hdr = r; continue
    if fn and kname in fn and hdr and r[0].isdigit():
        d = dict(zip(hdr, r))
        try: tot = int(d["Warp Stall Sampling (All Samples)"])
        except ValueError: continue
        reasons = sorted(((int(v), h[6:]) for h, v in d.items() if h.startswith("stall_") and "Not Issued" not in h and v.isdigit() and int(v) > 0), reverse=True)
        out.append((tot, cur, int(r[0]), r[1][:70], reasons[:3]))
T = sum(o[0] for o in out) or 1
print("total samples", T)
for tot, f, ln, src, rs in sorted(out, reverse=True)[:top]:
    print(f"{f}:{ln:<5} {100*tot/T:5.1f}%  {' '.join(f'{n}={100*v/T:.1f}' for v, n in rs):45s} {src}")
