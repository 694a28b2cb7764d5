#!/bin/bash
# A/B: p2 tables around (4, 2)
mkdir -p gpurun_out
for lib in .ab/lib_s4_n1_t3.so .ab/lib_s3_n2_t3.so .ab/lib_s2_n2_t3.so .ab/lib_s5_n2_t3.so; do
  LRCVT_LIB=$PWD/$lib timeout 900 python -m pytest tests/test_gpu_classify.py tests/test_gpu_edges.py -q -x -p no:cacheprovider > gpurun_out/g44_t.log 2>&1; echo "$lib tests rc=$?"
done
for rep in 1 2; do
for lib in "" .ab/lib_s4_n1_t3.so .ab/lib_s3_n2_t3.so .ab/lib_s2_n2_t3.so .ab/lib_s5_n2_t3.so; do
  if [ -n "$lib" ]; then export LRCVT_LIB=$PWD/$lib; else unset LRCVT_LIB; fi
  timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g44_ab.log 2>&1
  echo "[$lib] $(grep '^{' gpurun_out/g44_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')"
done
done
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "X=0" "LRCVT_P2_MINB=16" "LRCVT_P2_MINB=8" "LRCVT_P1_MINB=7" "LRCVT_P1_MINB=6"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g43_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g43_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')"
done
done
