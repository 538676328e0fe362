bash tools/w2cycle.sh v8 --ncu
SPHX_W2BT=256 timeout 300 python bench.py --config C2 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_v8b_C2.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_v8b_C2.json')); print('BT256', d['value'], d['breakdown_ms'], d['parity']['bit_exact_vs_reference_hash'])"
