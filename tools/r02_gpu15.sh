#!/bin/bash
# vote scan with 2-byte tag filter + predicated pair/weight loads
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_classify.py tests/test_gpu_multi.py tests/test_gpu_warp_eval.py tests/test_gpu_parity_big.py tests/test_capi.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g15_quick.log 2>&1; echo "quick rc=$?"; tail -3 gpurun_out/g15_quick.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g15_c4.log 2>&1; echo "c4 rc=$?"
grep '^{' gpurun_out/g15_c4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()}, d["gpu_launches"])'
for k in 8; do
timeout 1200 python bench.py --mode global --emulate-ranks $k --steps 3 --warmup 3 > gpurun_out/g15_global$k.log 2>&1; echo "global$k rc=$?"; grep '^{' gpurun_out/g15_global$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["emulated_ranks"]; print(d["ms_per_step"], round(e["slowest_rank_ms_per_step"],2), {k: round(v,2) for k,v in e["rank_ms_per_step"].items()}, {k: round(v,2) for k,v in e["slowest_rank_breakdown_ms_per_step"].items()})'
done
timeout 600 python tools/profile_kernels.py --help > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_vote --csv --log-file gpurun_out/g15_vote_ncu.csv python bench.py --steps 1 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g15_ncu.log 2>&1; echo "ncu rc=$?"
