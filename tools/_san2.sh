# compute-sanitizer over the gradient / step / drop-in stream tests (round 2, final code)
mkdir -p gpurun_out/san
timeout 1200 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gradient.py -x -q -m gpu > gpurun_out/san/memcheck_gradient.log 2>&1; tail -3 gpurun_out/san/memcheck_gradient.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -x -q -k "stream or small_case_tables" > gpurun_out/san/memcheck_stream.log 2>&1; tail -3 gpurun_out/san/memcheck_stream.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 python -m pytest tests/test_gradient.py -x -q -m gpu > gpurun_out/san/racecheck_gradient.log 2>&1; tail -3 gpurun_out/san/racecheck_gradient.log
