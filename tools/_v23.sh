timeout 900 python -m pytest tests/test_gradient.py tests/test_window2.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --op grad --config C2 --no-cpu-baseline > gpurun_out/bench_v23_grad.json 2> gpurun_out/bench_v23_grad.err
python -c "import json; d=json.load(open('gpurun_out/bench_v23_grad.json')); print('grad', d['value'], d['ms_per_step'], d.get('parity'))" || tail -5 gpurun_out/bench_v23_grad.err
