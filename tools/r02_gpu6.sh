#!/bin/bash
# branch-free tables, precomputed reciprocals, register-staged ordered adds in the votes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_classify.py tests/test_gpu_multi.py tests/test_gpu_warp_eval.py tests/test_gpu_parity_big.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g6_quick.log 2>&1; echo "quick rc=$?"; tail -3 gpurun_out/g6_quick.log
rm -f gpurun_out/g6_ab.txt
for rep in 1 2; do
 for cfg in "X=0" "LRCVT_VOTE=sort"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g6_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g6_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')" >> gpurun_out/g6_ab.txt
 done
done
cat gpurun_out/g6_ab.txt
timeout 600 python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g6_prof_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "profile/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/r02d_c4_launches.csv python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g6_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_eval_p2|k_vote_scan|k_vote_prep|k_vote_sum" -c 6 \
   -o gpurun_out/r02d_c4_p2 python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g6_ncu_p2.log 2>&1; echo "ncu p2 rc=$?"
timeout 1200 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_eval_p1|k_commit" -s 4 -c 6 \
   -o gpurun_out/r02d_c4_p1 python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g6_ncu_p1.log 2>&1; echo "ncu p1 rc=$?"
