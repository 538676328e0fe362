#!/usr/bin/env python
"""Per-step memory traffic of the bench step's kernels (run under gpurun).

    python tools/traffic.py C2 [C3 ...]   -> profiles/r2_traffic.json

One `ncu` pass per config over a short bench run (ncu flushes the caches before
every kernel, so DRAM reads are cold-L2 reads). Per kernel of one step: DRAM bytes
read / written and the bytes the kernel writes into L2 (lts__t_sectors_srcunit_tex
_op_write x 32: every store leaves the SM; the DRAM write counter misses whatever
is still dirty in the 126 MB L2 when the kernel ends). Step totals are the sums
over the step's kernels (the last launch of each name).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
           "gpu__time_duration.sum"]
KERNELS = "regex:k_w2|k_encode|k_rcll16|k_r16|k_xy|k_scan|k_sweep|k_pack"


def capture(cfg):
    cmd = ["ncu", "--metrics", ",".join(METRICS), "-k", KERNELS, "--csv", "--page", "raw",
           sys.executable, "bench.py", "--config", cfg, "--steps", "1", "--warmup", "3",
           "--no-cpu-baseline", "--e2e-steps", "0"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout
    lines = [l for l in out.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    last = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].split("::")[-1]
        last[name] = d
    ker = {}
    for name, d in last.items():
        f = lambda m: float(d[m].replace(",", ""))  # noqa: E731
        ker[name] = {"dram_read": f("dram__bytes_read.sum"), "dram_write": f("dram__bytes_write.sum"),
                     "l2_write": 32 * f("lts__t_sectors_srcunit_tex_op_write.sum"),
                     "l2_read": 32 * f("lts__t_sectors_srcunit_tex_op_read.sum"),
                     "ns": f("gpu__time_duration.sum")}
    tot = {k: sum(v[k] for v in ker.values()) for k in ("dram_read", "dram_write", "l2_write",
                                                         "l2_read", "ns")}
    return dict(tot, kernels=ker)


def main():
    commit = os.environ.get("COMMIT") or subprocess.run(
        ["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True,
        cwd=ROOT).stdout.strip() or None
    res = {"commit": commit, "how": "ncu --metrics " + ",".join(METRICS) +
           " on bench.py --steps 1 --warmup 3; last launch of each kernel; cold L2",
           "configs": {}}
    for cfg in sys.argv[1:]:
        res["configs"][f"{cfg}_fp16"] = capture(cfg)
        print(cfg, {k: round(v / 1e6, 2) if k != "ns" else v for k, v in res["configs"][f"{cfg}_fp16"].items() if k != "kernels"})
    with open(os.path.join(ROOT, "profiles", "r2_traffic.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
