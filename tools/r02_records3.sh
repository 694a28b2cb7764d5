#!/bin/bash
# Round-2 closing records after the table-size change: GPU suite, bench lines, global mode, eval ncu per item
mkdir -p gpurun_out/rec3
R=gpurun_out/rec3
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $R/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $R/pytest.log
timeout 1500 python bench.py > $R/bench_c4.log 2>&1; echo "bench c4 rc=$?"; grep '^{' $R/bench_c4.log | tail -1 > $R/bench_c4.json
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c > $R/bench_$c.log 2>&1; echo "bench $c rc=$?"; grep '^{' $R/bench_$c.log | tail -1 > $R/bench_$c.json
done
timeout 1500 python bench.py --config c5 --steps 5 --warmup 3 --no-passes > $R/bench_c5.log 2>&1; echo "bench c5 rc=$?"; grep '^{' $R/bench_c5.log | tail -1 > $R/bench_c5.json
for k in 8 4 2; do
  timeout 1500 python bench.py --mode global --emulate-ranks $k --steps 5 --warmup 3 > $R/global${k}_c4.log 2>&1; echo "global$k rc=$?"; grep '^{' $R/global${k}_c4.log | tail -1 > $R/global${k}_c4.json
done
timeout 1500 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_eval_p1|k_commit" -s 6 -c 6 \
   -o $R/c4_p1 python tools/profile_kernels.py --config c4 --host-rounds > $R/ncu_p1.log 2>&1; echo "ncu p1 rc=$?"
timeout 1500 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_eval_p2" -c 4 \
   -o $R/c4_p2 python tools/profile_kernels.py --config c4 --host-rounds > $R/ncu_p2.log 2>&1; echo "ncu p2 rc=$?"
python tools/ncu_kernel_table.py $R/c4_p1.ncu-rep $R/c4_ncu_p1_commit.json "C4 phase-1 eval and commit launches (6 after skipping 6), ncu --set full" > $R/c4_ncu_p1_commit.txt 2>&1
python tools/ncu_kernel_table.py $R/c4_p2.ncu-rep $R/c4_ncu_p2.json "C4 phase-2 eval launches (first 4), ncu --set full" > $R/c4_ncu_p2.txt 2>&1
python tools/ncu_src_breakdown.py $R/c4_p1.ncu-rep k_eval_p1 40 > $R/c4_src_p1.txt 2>&1
python tools/ncu_src_breakdown.py $R/c4_p2.ncu-rep k_eval_p2 40 > $R/c4_src_p2.txt 2>&1
python tools/eval_roof.py $R/c4_p1.ncu-rep c4 "phase-1 eval launches" > $R/eval_roof_p1.txt 2>&1; cp profiles/ncu_c4_k_eval.json $R/ncu_c4_k_eval_p1.json
python tools/eval_roof.py $R/c4_p2.ncu-rep c4 "phase-2 eval launches" > $R/eval_roof_p2.txt 2>&1; cp profiles/ncu_c4_k_eval.json $R/ncu_c4_k_eval_p2.json
python tools/eval_roof_merge.py $R/ncu_c4_k_eval_p1.json $R/ncu_c4_k_eval_p2.json $R/bench_c4.json c4 > $R/eval_roof_merged.txt 2>&1; cp profiles/ncu_c4_k_eval.json $R/ncu_c4_k_eval.json
timeout 900 python tools/e2e_probe2.py c4 > $R/e2e_probe_c4.txt 2>&1
rm -f $R/*.ncu-rep
ls $R; du -sh gpurun_out
