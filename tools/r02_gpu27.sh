#!/bin/bash
# vote: walk (count, write) / add split for all sites; rebalance
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_edges.py tests/test_gpu_classify.py tests/test_gpu_parity_big.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g27_quick.log 2>&1; echo "quick rc=$?"; tail -2 gpurun_out/g27_quick.log
timeout 1500 python tools/mg_check.py --config c4 --ranks 8 --iters 2 > gpurun_out/g27_c4.log 2>&1; echo "c4 check rc=$?"; tail -1 gpurun_out/g27_c4.log
for rep in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g27_ab.log 2>&1
echo "$(grep '^{' gpurun_out/g27_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')"
done
timeout 1200 python bench.py --mode global --emulate-ranks 8 --steps 3 --warmup 3 > gpurun_out/g27_global8.log 2>&1; echo "global8 rc=$?"; grep '^{' gpurun_out/g27_global8.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["emulated_ranks"]; print(d["ms_per_step"], round(e["slowest_rank_ms_per_step"],2), {k: round(v,2) for k,v in e["rank_ms_per_step"].items()}); print({k: round(v,3) for k,v in sorted(e["slowest_rank_breakdown_ms_per_step"].items())})'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_vote|k_scan" -c 12 --csv --log-file gpurun_out/g27_vote.csv python bench.py --steps 1 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g27_ncu.log 2>&1; echo "ncu rc=$?"
