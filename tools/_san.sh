mkdir -p gpurun_out/san
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_window2.py -x -q > gpurun_out/san/memcheck_window2.log 2>&1; tail -3 gpurun_out/san/memcheck_window2.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 python -m pytest tests/test_window2.py -x -q -k "small or golden or dense or orders" > gpurun_out/san/racecheck_window2.log 2>&1; tail -3 gpurun_out/san/racecheck_window2.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 5 python -m pytest tests/test_window2.py -x -q -k "small or golden or dense" > gpurun_out/san/synccheck_window2.log 2>&1; tail -3 gpurun_out/san/synccheck_window2.log
timeout 900 compute-sanitizer --tool initcheck --print-limit 5 python -m pytest tests/test_window2.py -x -q -k "small or golden" > gpurun_out/san/initcheck_window2.log 2>&1; tail -3 gpurun_out/san/initcheck_window2.log
