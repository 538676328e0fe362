#!/bin/bash
# SURVEY 8(d) locality study: C2 in lattice / shuffled / cell-sorted particle order,
# bench line + ncu DRAM bytes of the sweep and encode kernels for each.
#   tools/order_study.sh <tag>
TAG=$1
mkdir -p gpurun_out
for O in lattice shuffled sorted; do
  timeout 600 python bench.py --order $O --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${TAG}_$O.json 2> gpurun_out/bench_${TAG}_$O.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$O.json')); print('$O', d['value'], {k: round(v*1e3,1) for k,v in d['breakdown_ms'].items()}, d['parity'])"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"k_(w2|rcll16|encode_rows)" -s 6 -c 2 --csv --log-file gpurun_out/ncu_${TAG}_$O.csv \
      python bench.py --order $O --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
