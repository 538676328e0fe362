#!/bin/bash
# Quick iteration on the 2-D tiled path (under gpurun): GPU tests for the 2-D
# suites, the C2 bench line, launch times of the tiled kernels, one ncu capture.
#   tools/t2cycle.sh <tag> [--all-tests] [--no-ncu]
TAG=$1; shift
mkdir -p gpurun_out
SEL="tests/test_gpu_parity.py tests/test_dense.py tests/test_multigpu.py tests/test_core_api.py"
case " $* " in *" --all-tests "*) SEL="tests";; esac
timeout 900 python -m pytest $SEL -m gpu -x -q 2>&1 | tail -4
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/b_${TAG}.json 2> gpurun_out/b_${TAG}.err
python - "$TAG" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/b_{t}.json"))
    print("value", f"{d['value']:.4g}", {k: round(v * 1e3, 1) for k, v in d["breakdown_ms"].items()},
          "parity", d["parity"]["bit_exact_vs_reference_hash"])
except Exception as e:
    print("bench failed", e, open(f"gpurun_out/b_{t}.err").read()[-1500:])
PY
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_t2 -c 6 --csv \
  python bench.py --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>/dev/null | grep k_t2 | \
  python -c "
import csv,sys
for r in csv.reader(sys.stdin): print(r[4][:40], r[-3], r[-1])"
case " $* " in *" --no-ncu "*) exit 0;; esac
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_t2_(count|fill)" -s 2 -c 2 \
  -o gpurun_out/prof_${TAG} python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls gpurun_out/prof_${TAG}*
