#!/bin/bash
# A/B: register budget of the phase-1 eval below a million-voxel frontier, 5 (default) vs 6 / 8
mkdir -p gpurun_out
for rep in 1 2; do
for lib in "" .ab/lib_p1s6.so .ab/lib_p1s8.so; do
  if [ -n "$lib" ]; then export LRCVT_LIB=$PWD/$lib; else unset LRCVT_LIB; fi
  timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g49_ab.log 2>&1
  echo "[$lib] $(grep '^{' gpurun_out/g49_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')"
done
done
unset LRCVT_LIB
for cfg in c2 c3; do
for lib in "" .ab/lib_p1s8.so; do
  if [ -n "$lib" ]; then export LRCVT_LIB=$PWD/$lib; else unset LRCVT_LIB; fi
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g49_ab.log 2>&1
  echo "[$cfg $lib] $(grep '^{' gpurun_out/g49_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.3f" % d["ms_per_step"], {k: round(v,3) for k,v in r["breakdown_ms_per_step"].items()})')"
done
done
unset LRCVT_LIB
