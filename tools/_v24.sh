timeout 900 python -m pytest tests/test_gradient.py tests/test_window2.py -x -q 2>&1 | tail -2
for BT in 128 256; do
SPHX_W2BT=$BT timeout 300 python bench.py --config C2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_v24_$BT.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_v24_$BT.json')); print('BT$BT', d['value'], {k: round(v*1e3,1) for k,v in d['breakdown_ms'].items()}, 'frac', round(d['roofline']['frac'],4), 'pipe', round(d['roofline']['pipeline']['frac'],4), d['parity']['bit_exact_vs_reference_hash'])"
done
