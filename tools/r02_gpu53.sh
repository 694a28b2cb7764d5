#!/bin/bash
# A/B: voxel-ordered frontier rebuild (LRCVT_COMPACT=1) on the final kernels
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "X=0" "LRCVT_COMPACT=1"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g53_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g53_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')"
done
done
