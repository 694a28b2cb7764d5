#!/bin/bash
# vote: largest boxes first; MG vote timed in the library
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_classify.py tests/test_gpu_multi.py tests/test_gpu_warp_eval.py tests/test_gpu_parity_big.py tests/test_capi.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g18_quick.log 2>&1; echo "quick rc=$?"; tail -3 gpurun_out/g18_quick.log
rm -f gpurun_out/g18_ab.txt
for rep in 1; do
 for cfg in "X=0"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g18_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g18_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')" >> gpurun_out/g18_ab.txt
 done
done
cat gpurun_out/g18_ab.txt
for cfg in "X=0"; do
env $cfg timeout 1200 python bench.py --mode global --emulate-ranks 8 --steps 3 --warmup 3 > gpurun_out/g18_global8.log 2>&1; echo "global8 [$cfg] rc=$?"; grep '^{' gpurun_out/g18_global8.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["emulated_ranks"]; print(d["ms_per_step"], round(e["slowest_rank_ms_per_step"],2), {k: round(v,2) for k,v in e["rank_ms_per_step"].items()}, {k: round(v,2) for k,v in e["slowest_rank_breakdown_ms_per_step"].items()})'
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_vote_scan -c 1 -o gpurun_out/g18_vote python bench.py --steps 1 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g18_ncu.log 2>&1; echo "ncu rc=$?"
grep '^{' gpurun_out/g18_global8.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d.get("counters"))'
