#!/bin/bash
# Round-end measurement pass (run under gpurun, one GPU):
#   tools/final_cycle.sh <tag> [--all]   (--all: also C4, C5, the step and grad ops, smoke)
# parity tests, the default bench line (C2, with the CPU baseline), C3, the
# reference arm, and the launch list + ncu capture of C2 and C3.
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -c 600 gpurun_out/bench_${TAG}.json
timeout 900 python bench.py --config C3 > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err; tail -c 300 gpurun_out/bench_${TAG}_c3.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_reference.json 2> gpurun_out/bench_${TAG}_reference.err; tail -c 300 gpurun_out/bench_${TAG}_reference.json
bash tools/profile.sh "$TAG"
bash tools/profile.sh "${TAG}_c3" --config C3
if [ "$2" = "--all" ]; then
  for C in C4 C5; do
    timeout 900 python bench.py --config $C --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_${TAG}_$C.json 2> gpurun_out/bench_${TAG}_$C.err
    tail -c 200 gpurun_out/bench_${TAG}_$C.json
  done
  for C in C2 C3; do
    timeout 600 python bench.py --op step --config $C --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_step_$C.json 2> gpurun_out/bench_${TAG}_step_$C.err
    timeout 600 python bench.py --op grad --config $C --no-cpu-baseline > gpurun_out/bench_${TAG}_grad_$C.json 2> gpurun_out/bench_${TAG}_grad_$C.err
  done
  timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
fi
