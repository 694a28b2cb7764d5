#!/bin/bash
# fast clearance DDA, own-site dedup, p1 batched gathers, sp reset (no comp load) in the bbox vote
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_classify.py tests/test_gpu_multi.py tests/test_gpu_warp_eval.py -q -x -p no:cacheprovider > gpurun_out/g5_quick.log 2>&1; echo "quick rc=$?"; tail -4 gpurun_out/g5_quick.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/g5_all.log 2>&1; echo "all rc=$?"; tail -14 gpurun_out/g5_all.log
rm -f gpurun_out/g5_ab.txt
for rep in 1 2; do
 for cfg in "X=0" "LRCVT_VOTE=sort" "LRCVT_COMPACT=1"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g5_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g5_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')" >> gpurun_out/g5_ab.txt
 done
done
cat gpurun_out/g5_ab.txt
timeout 1200 python bench.py --mode global --emulate-ranks 8 --steps 3 --warmup 3 > gpurun_out/g5_global8.log 2>&1; echo "global emulate 8 rc=$?"; grep '^{' gpurun_out/g5_global8.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], json.dumps(d.get("emulated_ranks")))'
timeout 600 python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g5_prof_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "profile/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/r02c_c4_launches.csv python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g5_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_eval_p|k_commit|k_vote_scan|k_vote_prep" -s 12 -c 10 \
   -o gpurun_out/r02c_c4_eval python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g5_ncu_eval.log 2>&1; echo "ncu eval rc=$?"
