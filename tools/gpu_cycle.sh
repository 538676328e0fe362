#!/bin/bash
# One GPU iteration (run under gpurun): parity tests, bench, profile.
#   tools/gpu_cycle.sh <tag> [--no-profile]
TAG=$1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; tail -4 gpurun_out/pytest_${TAG}.log
python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python - "$TAG" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/bench_{t}.json"))
    print("value", f"{d['value']:.4g}", "breakdown", {k: round(v * 1e3, 1) for k, v in d["breakdown_ms"].items()},
          "frac", round(d["roofline"]["frac"], 4), "parity", d["parity"]["bit_exact_vs_reference_hash"],
          "e2e_ms", round(d["e2e"]["ms_per_step"], 3))
except Exception as e:
    print("bench failed", e)
    print(open(f"gpurun_out/bench_{t}.err").read()[-2000:])
PY
if [ "$2" != "--no-profile" ]; then bash tools/profile.sh "$TAG"; fi
