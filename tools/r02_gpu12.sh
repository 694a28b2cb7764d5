#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_classify.py tests/test_gpu_multi.py tests/test_gpu_warp_eval.py -q -x -p no:cacheprovider > gpurun_out/g12_quick.log 2>&1; echo "quick rc=$?"; tail -2 gpurun_out/g12_quick.log
rm -f gpurun_out/g12_ab.txt
for rep in 1 2; do
 for cfg in "X=0"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g12_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g12_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')" >> gpurun_out/g12_ab.txt
 done
done
cat gpurun_out/g12_ab.txt
