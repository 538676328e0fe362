#!/bin/bash
# C5 A/B of experiment builds:   tools/exp_c5.sh 0 1 0 1
for E in "$@"; do
  if [ "$E" = 0 ]; then unset SPHX_CUDA_LIB; else export SPHX_CUDA_LIB=$PWD/exp/libsphx_cuda_e$E.so; fi
  timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('E$E C5', {k: round(v,2) for k,v in d['breakdown_ms'].items()}, d['parity']['ok'])"
done
