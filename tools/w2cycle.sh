#!/bin/bash
# GPU iteration for the windowed 2-D path: tools/w2cycle.sh <tag> [--full] [--ncu]
TAG=$1; shift
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_window2.py -x -q > gpurun_out/pytest_w2_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_w2_${TAG}.log
case " $* " in *" --full "*) timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_${TAG}.log;; esac
for C in C2; do
  timeout 300 python bench.py --config $C --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${TAG}_${C}.json 2> gpurun_out/bench_${TAG}_${C}.err
  python - "$TAG" "$C" <<'PY'
import json, sys
t, c = sys.argv[1], sys.argv[2]
try:
    d = json.load(open(f"gpurun_out/bench_{t}_{c}.json"))
    print(c, "value", f"{d['value']:.4g}", {k: round(v * 1e3, 1) for k, v in d["breakdown_ms"].items()},
          "frac", round(d["roofline"]["frac"], 4), "parity", d["parity"]["bit_exact_vs_reference_hash"])
except Exception as e:
    print(c, "bench failed", e, open(f"gpurun_out/bench_{t}_{c}.err").read()[-1500:])
PY
done
case " $* " in *" --ncu "*)
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_w2" -s 6 -c 2 \
    -o gpurun_out/prof_${TAG} python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/ncu_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_${TAG}.log;;
esac
