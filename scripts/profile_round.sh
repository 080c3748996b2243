#!/bin/bash
# Collect: ncu launch list (per-kernel device time) + full captures of the top kernels.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 2 --profile-phases 0 --skip-cpu --no-graph > gpurun_out/launches_bench.log 2>&1
for k in dec_kernel att_bwd_kernel lstm_bwd_kernel sim_kernel dec_wgrad_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k \
      python bench.py --steps 1 --warmup 2 --profile-phases 0 --skip-cpu --no-graph > gpurun_out/prof_$k.log 2>&1
done
ls -la gpurun_out
