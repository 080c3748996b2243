#!/bin/bash
# full ncu captures (one launch each) of the named kernels: prof_<name>.ncu-rep
mkdir -p gpurun_out
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k -f \
      python bench.py --steps 1 --warmup 2 --profile-phases 0 --skip-cpu --no-graph > gpurun_out/prof_$k.log 2>&1
done
