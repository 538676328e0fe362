#!/bin/bash
# ncu launch lists + one --set full capture of the 8(f) kernels: the fused
# gradient (--op grad) and the mixed step (--op step), C2.
#   tools/profile_ops.sh <tag>
TAG=$1
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}_grad.csv \
    python bench.py --op grad --steps 3 --warmup 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_r16_grad" -s 2 -c 1 \
    -o gpurun_out/prof_${TAG}_grad python bench.py --op grad --steps 2 --warmup 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}_step.csv \
    python bench.py --op step --steps 2 --warmup 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_(stress|rates)" -s 4 -c 2 \
    -o gpurun_out/prof_${TAG}_step python bench.py --op step --steps 2 --warmup 3 > /dev/null 2>&1
ls gpurun_out | grep "${TAG}_"
