#!/bin/bash
# no-improvement certificates (p1, p2), hybrid append + optional voxel-order rebuild (k_reorder)
mkdir -p gpurun_out
for env in "X=0" "LRCVT_COMPACT=1"; do
env $env timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_classify.py tests/test_gpu_multi.py tests/test_gpu_warp_eval.py tests/test_gpu_parity_big.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g7_quick.log 2>&1; echo "quick [$env] rc=$?"; tail -2 gpurun_out/g7_quick.log
done
rm -f gpurun_out/g7_ab.txt
for rep in 1 2; do
 for cfg in "X=0" "LRCVT_COMPACT=1"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g7_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g7_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')" >> gpurun_out/g7_ab.txt
 done
done
cat gpurun_out/g7_ab.txt
timeout 600 python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g7_prof_plain.log 2>&1 && \
timeout 1200 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_eval_p" -s 3 -c 6 \
   -o gpurun_out/r02e_c4_eval python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g7_ncu.log 2>&1; echo "ncu rc=$?"
