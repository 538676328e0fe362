#!/bin/bash
# interleaved A/B of experiment builds (under gpurun):  tools/ab.sh <rounds> <config> E...
#   E = 0 is the default in-tree build; E = N is exp/libsphx_cuda_eN.so (tools/exp_build.sh)
#   BARGS: extra bench.py arguments (e.g. BARGS='--op grad')
R=$1; C=$2; shift 2
for k in $(seq 1 $R); do
  for E in "$@"; do
    if [ "$E" = 0 ]; then unset SPHX_CUDA_LIB; else export SPHX_CUDA_LIB=$PWD/exp/libsphx_cuda_e$E.so; fi
    timeout 200 python bench.py --config $C $BARGS --no-cpu-baseline --e2e-steps 1 --steps 30 > /tmp/b.json 2>/tmp/b.err
    python -c "import json; d=json.load(open('/tmp/b.json')); print('E$E', '$C', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in (d.get('breakdown_ms') or {}).items()}, d['parity'])" 2>/dev/null || tail -3 /tmp/b.err
  done
done
