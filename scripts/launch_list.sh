#!/bin/bash
# ncu per-launch device times for one eager bench step (shares, not absolutes).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c ${1:-80} --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --profile-phases 0 --skip-cpu --no-graph ${2:-} > gpurun_out/launches_bench.log 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv seq
