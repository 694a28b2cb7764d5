#!/bin/bash
# A/B: warp-uniform table skips etc. (default) vs warp-aggregated commit
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_classify.py tests/test_gpu_multi.py tests/test_gpu_warp_eval.py tests/test_gpu_parity_big.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g13_quick.log 2>&1; echo "quick rc=$?"; tail -2 gpurun_out/g13_quick.log
LRCVT_COMMIT_AGG=1 timeout 900 python -m pytest tests/test_gpu_classify.py tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/g13_agg.log 2>&1; echo "agg rc=$?"; tail -2 gpurun_out/g13_agg.log
rm -f gpurun_out/g13_ab.txt
for rep in 1 2; do
 for cfg in "X=0" "LRCVT_COMMIT_AGG=1" "LRCVT_VOTE=sort"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g13_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g13_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')" >> gpurun_out/g13_ab.txt
 done
done
cat gpurun_out/g13_ab.txt
timeout 1200 python bench.py --mode global --emulate-ranks 8 --steps 3 --warmup 3 > gpurun_out/g13_global8.log 2>&1; echo "global8 rc=$?"; grep '^{' gpurun_out/g13_global8.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], json.dumps(d.get("emulated_ranks")))'
