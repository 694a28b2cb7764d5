#!/bin/bash
# A/B: phase-2 eval CTA 32 threads vs 64
mkdir -p gpurun_out
LRCVT_EVAL_BS=128,32 timeout 900 python -m pytest tests/test_gpu_classify.py tests/test_gpu_edges.py -q -x -p no:cacheprovider > gpurun_out/g55_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g55_t.log
for rep in 1 2; do
for cfg in "X=0" "LRCVT_EVAL_BS=128,32"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g55_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g55_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')"
done
done
