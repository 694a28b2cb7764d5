#!/bin/bash
# A/B: phase-1 distinct-site table size 3 / 4 (default) / 5
mkdir -p gpurun_out
LRCVT_LIB=$PWD/.ab/lib_tab3.so timeout 900 python -m pytest tests/test_gpu_classify.py tests/test_gpu_edges.py -q -x -p no:cacheprovider > gpurun_out/g40_t3.log 2>&1; echo "tab3 tests rc=$?"; tail -1 gpurun_out/g40_t3.log
for rep in 1 2; do
for lib in "" ".ab/lib_tab3.so" ".ab/lib_tab5.so"; do
  if [ -n "$lib" ]; then export LRCVT_LIB=$PWD/$lib; else unset LRCVT_LIB; fi
  timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g40_ab.log 2>&1
  echo "[$lib] $(grep '^{' gpurun_out/g40_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')"
done
done
