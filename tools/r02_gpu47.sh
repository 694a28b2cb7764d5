#!/bin/bash
# A/B: commit CTA size 256 (default) vs 512 / 1024
mkdir -p gpurun_out
for lib in .ab/lib_cm512.so .ab/lib_cm1024.so; do
  LRCVT_LIB=$PWD/$lib timeout 900 python -m pytest tests/test_gpu_classify.py tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/g47_t.log 2>&1; echo "$lib tests rc=$?"
done
for rep in 1 2 3; do
for lib in "" .ab/lib_cm512.so .ab/lib_cm1024.so; do
  if [ -n "$lib" ]; then export LRCVT_LIB=$PWD/$lib; else unset LRCVT_LIB; fi
  timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g47_ab.log 2>&1
  echo "[$lib] $(grep '^{' gpurun_out/g47_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')"
done
done
unset LRCVT_LIB
