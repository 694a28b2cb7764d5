#!/bin/bash
# Round-2 final records: full GPU suite, bench lines (C4 default with both arms; C1-C3, C5), emulated
# global mode, and the ncu evidence for every kernel at C4 (launch list + full captures).
mkdir -p gpurun_out/rec2
R=gpurun_out/rec2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $R/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > $R/pytest.log 2>&1; echo "pytest rc=$?"; tail -16 $R/pytest.log
timeout 1500 python bench.py > $R/bench_c4.log 2>&1; echo "bench c4 rc=$?"; grep '^{' $R/bench_c4.log | tail -1 > $R/bench_c4.json
timeout 1500 python bench.py --impl reference > $R/ref_c4.log 2>&1; echo "ref c4 rc=$?"; grep '^{' $R/ref_c4.log | tail -1 > $R/ref_c4.json
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c > $R/bench_$c.log 2>&1; echo "bench $c rc=$?"; grep '^{' $R/bench_$c.log | tail -1 > $R/bench_$c.json
done
timeout 1500 python bench.py --config c5 --steps 5 --warmup 3 --no-passes > $R/bench_c5.log 2>&1; echo "bench c5 rc=$?"; grep '^{' $R/bench_c5.log | tail -1 > $R/bench_c5.json
timeout 1500 python bench.py --mode global --emulate-ranks 8 --steps 5 --warmup 3 > $R/global8_c4.log 2>&1; echo "global8 c4 rc=$?"; grep '^{' $R/global8_c4.log | tail -1 > $R/global8_c4.json
timeout 1500 python bench.py --mode global --emulate-ranks 4 --steps 5 --warmup 3 > $R/global4_c4.log 2>&1; echo "global4 c4 rc=$?"; grep '^{' $R/global4_c4.log | tail -1 > $R/global4_c4.json
timeout 1500 python bench.py --mode global --emulate-ranks 2 --steps 5 --warmup 3 > $R/global2_c4.log 2>&1; echo "global2 c4 rc=$?"; grep '^{' $R/global2_c4.log | tail -1 > $R/global2_c4.json
# ncu evidence at C4: every launch of one pass (graph rounds replaced by host rounds, whose kernel nodes ncu can profile)
timeout 600 python tools/profile_kernels.py --config c4 --host-rounds > $R/prof_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "profile/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $R/c4_launches.csv python tools/profile_kernels.py --config c4 --host-rounds > $R/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_isobands|k_ccl_|k_agg_|k_vote|k_scan_excl|k_move_sites|k_fill|k_state|k_site1_to_state|k_seed|k_site_voxel|k_phase2_copy" \
   -o $R/c4_other python tools/profile_kernels.py --config c4 --host-rounds > $R/ncu_other.log 2>&1; echo "ncu other rc=$?"
timeout 1500 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_eval_p1|k_commit" -s 6 -c 6 \
   -o $R/c4_p1 python tools/profile_kernels.py --config c4 --host-rounds > $R/ncu_p1.log 2>&1; echo "ncu p1 rc=$?"
timeout 1500 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_eval_p2" -c 4 \
   -o $R/c4_p2 python tools/profile_kernels.py --config c4 --host-rounds > $R/ncu_p2.log 2>&1; echo "ncu p2 rc=$?"
# summaries on the box (the .ncu-rep files are too large to bring back)
python tools/ncu_kernel_table.py $R/c4_other.ncu-rep $R/c4_ncu_other_kernels.json "C4 512^3 one pass of every non-eval kernel (tools/profile_kernels.py --host-rounds), ncu --set full --clock-control none, cold cache per replay" > $R/c4_ncu_other_kernels.txt 2>&1
python tools/ncu_kernel_table.py $R/c4_p1.ncu-rep $R/c4_ncu_p1_commit.json "C4 phase-1 eval and commit launches (6 after skipping 6), ncu --set full" > $R/c4_ncu_p1_commit.txt 2>&1
python tools/ncu_kernel_table.py $R/c4_p2.ncu-rep $R/c4_ncu_p2.json "C4 phase-2 eval launches (first 4), ncu --set full" > $R/c4_ncu_p2.txt 2>&1
python tools/ncu_src_breakdown.py $R/c4_p1.ncu-rep k_eval_p1 40 > $R/c4_src_p1.txt 2>&1
python tools/ncu_src_breakdown.py $R/c4_p1.ncu-rep k_commit 30 > $R/c4_src_commit.txt 2>&1
python tools/ncu_src_breakdown.py $R/c4_p2.ncu-rep k_eval_p2 40 > $R/c4_src_p2.txt 2>&1
python tools/ncu_src_breakdown.py $R/c4_other.ncu-rep k_vote_add 30 > $R/c4_src_vote_add.txt 2>&1; python tools/ncu_src_breakdown.py $R/c4_other.ncu-rep k_vote_walk 30 > $R/c4_src_vote_walk.txt 2>&1
cp $R/c4_p1.ncu-rep /tmp/ && python tools/eval_roof.py /tmp/c4_p1.ncu-rep c4 "phase-1 eval launches" > $R/eval_roof_p1.txt 2>&1; cp profiles/ncu_c4_k_eval.json $R/ncu_c4_k_eval_p1.json
python tools/eval_roof.py $R/c4_p2.ncu-rep c4 "phase-2 eval launches" > $R/eval_roof_p2.txt 2>&1; cp profiles/ncu_c4_k_eval.json $R/ncu_c4_k_eval_p2.json
python tools/eval_roof_merge.py $R/ncu_c4_k_eval_p1.json $R/ncu_c4_k_eval_p2.json $R/bench_c4.json c4 > $R/eval_roof_merged.txt 2>&1; cp profiles/ncu_c4_k_eval.json $R/ncu_c4_k_eval.json
timeout 900 python tools/e2e_probe2.py c4 > $R/e2e_probe_c4.txt 2>&1
rm -f $R/*.ncu-rep
ls -la $R; du -sh gpurun_out
