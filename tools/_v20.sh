timeout 600 python -m pytest tests/test_window2.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for O in lattice shuffled sorted; do
  timeout 600 python bench.py --order $O --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_v20_$O.json 2> gpurun_out/bench_v20_$O.err
  python -c "import json; d=json.load(open('gpurun_out/bench_v20_$O.json')); print('$O', d['value'], {k: round(v*1e3,1) for k,v in d['breakdown_ms'].items()}, d['parity']['bit_exact_vs_reference_hash'])"
done
