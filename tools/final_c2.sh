#!/bin/bash
# C2 measurement refresh (run under gpurun): default bench line with the CPU
# baseline, the order study, the launch list + ncu --set full of the C2 step, and
# the per-kernel traffic pass (profiles/r2_traffic.json).   tools/final_c2.sh <tag>
TAG=$1
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -c 300 gpurun_out/bench_${TAG}.json; echo
bash tools/order_study.sh "$TAG"
bash tools/profile.sh "$TAG"
COMMIT=$(cat .commit 2>/dev/null) timeout 900 python tools/traffic.py C2 C3
cp profiles/r2_traffic.json gpurun_out/r2_traffic_${TAG}.json
