#!/bin/bash
# commit with in-CTA slot compaction, vote scan prefetch, MG v2 (slab-owned state, halo, peer reads, partitioned vote)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_classify.py tests/test_gpu_multi.py tests/test_gpu_warp_eval.py tests/test_gpu_edges.py -q -x -p no:cacheprovider > gpurun_out/g4_quick.log 2>&1; echo "quick rc=$?"; tail -15 gpurun_out/g4_quick.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/g4_all.log 2>&1; echo "all rc=$?"; tail -25 gpurun_out/g4_all.log
rm -f gpurun_out/g4_ab.txt
for rep in 1 2; do
 for cfg in "LRCVT_LIB=ab/liblrcvt_r02a.so" "X=0" "LRCVT_COMPACT=1" "LRCVT_VOTE=sort"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g4_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g4_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')" >> gpurun_out/g4_ab.txt
 done
done
cat gpurun_out/g4_ab.txt
for k in 2 8; do
 timeout 1200 python bench.py --mode global --emulate-ranks $k --steps 3 --warmup 3 > gpurun_out/g4_global$k.log 2>&1; echo "global emulate $k rc=$?"; grep '^{' gpurun_out/g4_global$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], json.dumps(d.get("emulated_ranks")))'
done
