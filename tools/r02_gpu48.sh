#!/bin/bash
# env A/B after the table / commit changes: phase-2 and phase-1 register budgets, warp-eval threshold
mkdir -p gpurun_out
unset LRCVT_LIB
for rep in 1 2; do
for cfg in "X=0" "LRCVT_P2_MINB=16" "LRCVT_P1_MINB=7" "LRCVT_EW_SMALL=1024" "LRCVT_EW_SMALL=4096"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g48_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g48_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')"
done
done
