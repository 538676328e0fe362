#!/bin/bash
# shared-memory wavefronts / bank conflicts of k_w2 per experiment build (under gpurun)
#   tools/lsu_ab.sh E...
mkdir -p gpurun_out
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum
for E in "$@"; do
  if [ "$E" = 0 ]; then unset SPHX_CUDA_LIB; else export SPHX_CUDA_LIB=$PWD/exp/libsphx_cuda_e$E.so; fi
  timeout 300 ncu --metrics $M --clock-control none -k regex:k_w2 -s 4 -c 2 --csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/lsu_e$E.csv 2>/dev/null
  python - "$E" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/lsu_e{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    if "k_w2<" in d.get("Kernel Name", ""):
        print("E" + sys.argv[1], d["Metric Name"], d["Metric Value"])
PY
done
