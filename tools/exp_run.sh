#!/bin/bash
# time experiment builds exp/libsphx_cuda_e<N>.so against the default build (E0)
for E in "$@"; do
  if [ "$E" = 0 ]; then unset SPHX_CUDA_LIB; else export SPHX_CUDA_LIB=$PWD/exp/libsphx_cuda_e$E.so; fi
  for C in C2 C3; do
    timeout 200 python bench.py --config $C --no-cpu-baseline --e2e-steps 1 --steps 20 > /tmp/b.json 2>/dev/null
    python -c "import json; d=json.load(open('/tmp/b.json')); print('E$E', '$C', {k: round(v*1e3,1) for k,v in d['breakdown_ms'].items()})"
  done
done
