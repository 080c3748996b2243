#!/bin/bash
# Re-measure the round's committed evidence on one B200 (run under gpurun):
# per-kernel ncu --set full captures -> profiles/<tag>_ncu_summary.{json,md},
# the C3 launch list, phase clocks, and the bench lines (C3 / C4 / C5 /
# reference arm).  Outputs land in gpurun_out/ (merged back by gpurun).
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT profiles
reps=()
for k in dec_kernel att_bwd_kernel lstm_bwd_kernel sim_warp_kernel enc_rec_kernel dec_wgrad_tc_kernel adv_grads_kernel; do
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $OUT/prof_$k \
        python bench.py --steps 1 --warmup 3 --skip-cpu > $OUT/ncu_$k.log 2>&1
    reps+=($OUT/prof_$k.ncu-rep)
done
python scripts/ncu_summary.py $TAG "${reps[@]}" > $OUT/ncu_summary.log 2>&1
cp profiles/${TAG}_ncu_summary.json profiles/${TAG}_ncu_summary.md $OUT/
# C5 decoder (DM streaming path) and score-recompute attention backward at their
# bench size, one launch each (reports named by kernel: bench.py reads the decoder's traffic)
mkdir -p $OUT/c5
for k in dec_kernel att_bwd_kernel; do
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $OUT/c5/prof_$k \
        python bench.py --config C5 --steps 1 --warmup 3 --skip-cpu > $OUT/ncu_c5_$k.log 2>&1
done
NCU_WORKLOAD="C5 K=4096" python scripts/ncu_summary.py ${TAG}_C5 $OUT/c5/prof_dec_kernel.ncu-rep $OUT/c5/prof_att_bwd_kernel.ncu-rep > $OUT/ncu_summary_c5.log 2>&1
cp profiles/${TAG}_C5_ncu_summary.json profiles/${TAG}_C5_ncu_summary.md $OUT/ 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${TAG}_launches_C3.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu > /dev/null 2>&1
python scripts/launch_summary.py $OUT/${TAG}_launches_C3.csv seq > $OUT/${TAG}_launch_summary.txt
python scripts/dec_phases.py C3 256 > $OUT/${TAG}_decoder_phase_clocks.txt
python scripts/dec_phases.py C5 4096 > $OUT/${TAG}_C5_decoder_phase_clocks.txt
python scripts/lstm_phases.py C3 256 > $OUT/${TAG}_lstm_bwd_phase_clocks.txt
python scripts/enc_phases.py C3 > $OUT/${TAG}_encoder_phase_clocks.txt
timeout 900 python bench.py > $OUT/${TAG}_bench_C3_1gpu.json 2> $OUT/bench_C3.err
bash scripts/launch_list.sh 150 "--config C5" > /dev/null 2>&1; python scripts/launch_summary.py $OUT/launches.csv seq > $OUT/${TAG}_launch_summary_C5.txt
timeout 900 python bench.py --config C4 > $OUT/${TAG}_bench_C4_1gpu.json 2> $OUT/bench_C4.err
timeout 900 python bench.py --config C5 > $OUT/${TAG}_bench_C5_1gpu.json 2> $OUT/bench_C5.err
timeout 900 python bench.py --impl reference > $OUT/${TAG}_bench_reference_C3.json 2> $OUT/bench_ref.err
timeout 900 python bench.py --mode sim > $OUT/${TAG}_bench_sim_C3.json 2> $OUT/bench_sim_C3.err
timeout 900 python bench.py --mode sim --config C5 > $OUT/${TAG}_bench_sim_C5.json 2> $OUT/bench_sim_C5.err
# tensor-core vs DMMA decoder weight gradient (per-launch device time)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:dec_wgrad --csv \
    python scripts/wgrad_ab.py C3 256 0,1 > $OUT/${TAG}_wgrad_ab_ncu.csv 2>&1
python scripts/sass_evidence.py > $OUT/${TAG}_sass_evidence.txt
rm -f $OUT/prof_*.ncu-rep $OUT/c5/prof_*.ncu-rep
echo done
