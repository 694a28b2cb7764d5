#!/bin/bash
# p1 without shared rows, commit: sequential rows + unrolled append
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_classify.py tests/test_gpu_multi.py tests/test_gpu_warp_eval.py tests/test_gpu_parity_big.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g11_quick.log 2>&1; echo "quick rc=$?"; tail -2 gpurun_out/g11_quick.log
rm -f gpurun_out/g11_ab.txt
for rep in 1 2; do
 for cfg in "X=0" "LRCVT_VOTE=sort" "LRCVT_COMPACT=1"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g11_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g11_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')" >> gpurun_out/g11_ab.txt
 done
done
cat gpurun_out/g11_ab.txt
timeout 600 python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g11_prof_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "profile/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/r02g_c4_launches.csv python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g11_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_eval_p1|k_commit" -s 8 -c 4 \
   -o gpurun_out/r02g_c4_p1 python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g11_ncu.log 2>&1; echo "ncu rc=$?"
