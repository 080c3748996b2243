#!/bin/bash
# Round evidence: bench line, launch list (ncu), full capture of the top kernels.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.json
bash scripts/launch_list.sh 200 > gpurun_out/launch_summary.txt 2>&1
cat gpurun_out/launch_summary.txt | head -25
bash scripts/prof_kernels.sh dec_kernel att_bwd_kernel lstm_bwd_kernel sim_kernel
python scripts/dec_phases.py C3 256 > gpurun_out/dec_phases.txt 2>&1
