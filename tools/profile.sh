#!/bin/bash
# GPU-box profiling recipe (run under gpurun, one GPU):
#   tools/profile.sh <tag> [extra bench.py args]
# 1) launch list with per-launch device time (cold-cache, serialised: compare shares)
# 2) one `ncu --set full` capture of the dominant sweep kernel (read here with ncu -i)
set -u
mkdir -p gpurun_out
TAG=$1
shift
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on \
    -k regex:"k_(w2|rcll16|r16_test|r16_emit|encode_rows|encode_xy)" -s 6 -c 3 \
    -o gpurun_out/prof_${TAG} \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" \
    > gpurun_out/ncu_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_${TAG}.log
