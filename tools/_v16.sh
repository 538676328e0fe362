timeout 600 python -m pytest tests/test_core_api.py tests/test_abi.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --config C2 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_v16_C2.json 2> gpurun_out/bench_v16_C2.err
python -c "import json; d=json.load(open('gpurun_out/bench_v16_C2.json')); print(d['value'], d['parity']['bit_exact_vs_reference_hash']); print(json.dumps(d['e2e']))" || tail -20 gpurun_out/bench_v16_C2.err
