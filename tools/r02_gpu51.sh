#!/bin/bash
# A/B: grid of the eligible-list passes (fill_list, site1_to_state, state, vote_count): 16 (default) / 64 / 256 waves of 148 CTAs
mkdir -p gpurun_out
for rep in 1 2; do
for lib in "" .ab/lib_el64.so .ab/lib_el256.so; do
  if [ -n "$lib" ]; then export LRCVT_LIB=$PWD/$lib; else unset LRCVT_LIB; fi
  timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g51_ab.log 2>&1
  echo "[$lib] $(grep '^{' gpurun_out/g51_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')"
done
done
unset LRCVT_LIB
