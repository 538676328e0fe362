#!/bin/bash
# GPU-box profiling recipe (run under gpurun, one GPU):
#   tools/profile.sh <tag> [extra bench.py args]
# 1) launch list with per-launch device time (cold-cache, serialised: compare shares)
# 2) one `ncu --set full` capture of the sweep kernel (read here with ncu -i)
set -u
mkdir -p gpurun_out
TAG=$1
shift
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_(sweep|encode_members)" -s 8 -c 2 \
    -o gpurun_out/prof_${TAG} \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" \
    > gpurun_out/ncu_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_${TAG}.log
