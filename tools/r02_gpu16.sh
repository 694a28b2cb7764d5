#!/bin/bash
# vote scan two-stage pipeline (+/- tags), padded ordered adds; MG round with fused own+halo commit, no per-round memsets
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_classify.py tests/test_gpu_multi.py tests/test_gpu_warp_eval.py tests/test_gpu_parity_big.py tests/test_capi.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g16_quick.log 2>&1; echo "quick rc=$?"; tail -3 gpurun_out/g16_quick.log
LRCVT_VOTE_TAGS=1 timeout 1200 python -m pytest tests/test_gpu_parity_big.py tests/test_gpu_multi.py tests/test_gpu_edges.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g16_tags.log 2>&1; echo "tags rc=$?"; tail -1 gpurun_out/g16_tags.log
rm -f gpurun_out/g16_ab.txt
for rep in 1 2; do
 for cfg in "X=0" "LRCVT_VOTE_TAGS=1"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g16_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g16_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')" >> gpurun_out/g16_ab.txt
 done
done
cat gpurun_out/g16_ab.txt
for cfg in "X=0" "LRCVT_VOTE_TAGS=1"; do
env $cfg timeout 1200 python bench.py --mode global --emulate-ranks 8 --steps 3 --warmup 3 > gpurun_out/g16_global8.log 2>&1; echo "global8 [$cfg] rc=$?"; grep '^{' gpurun_out/g16_global8.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["emulated_ranks"]; print(d["ms_per_step"], round(e["slowest_rank_ms_per_step"],2), {k: round(v,2) for k,v in e["rank_ms_per_step"].items()}, {k: round(v,2) for k,v in e["slowest_rank_breakdown_ms_per_step"].items()})'
done
for cfg in "X=0" "LRCVT_VOTE_TAGS=1"; do
env $cfg timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:k_vote_scan -c 2 --csv --log-file gpurun_out/g16_vote_ncu_$cfg.csv python bench.py --steps 1 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g16_ncu.log 2>&1; echo "ncu rc=$?"
done
