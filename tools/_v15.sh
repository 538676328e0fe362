timeout 300 python bench.py --config C2 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_v15_C2.json 2> gpurun_out/bench_v15_C2.err
python -c "import json; d=json.load(open('gpurun_out/bench_v15_C2.json')); print(d['value'], d['breakdown_ms'], d['parity']); print(json.dumps(d['e2e'])); print(d['config'])" || tail -20 gpurun_out/bench_v15_C2.err
COMMIT=5d646f3 timeout 900 python tools/traffic.py C2 C3 > gpurun_out/traffic_v15.log 2>&1; tail -3 gpurun_out/traffic_v15.log
cp profiles/r2_traffic.json gpurun_out/r2_traffic.json
