#!/bin/bash
# global mode: MG phase-2 eval at the one-domain register budget; two calibration re-cuts
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_bench.py -q -x -p no:cacheprovider > gpurun_out/g46_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g46_t.log
timeout 1500 python tools/mg_check.py --config c4 --ranks 8 --iters 2 > gpurun_out/g46_c4.log 2>&1; echo "c4 check rc=$?"; tail -1 gpurun_out/g46_c4.log
for rep in 1 2; do
timeout 1500 python bench.py --mode global --emulate-ranks 8 --steps 5 --warmup 3 > gpurun_out/g46_global8.log 2>&1; echo "global8 rc=$?"; grep '^{' gpurun_out/g46_global8.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["emulated_ranks"]; print(d["ms_per_step"], round(e["slowest_rank_ms_per_step"],2), {k: round(v,2) for k,v in e["rank_ms_per_step"].items()}); print({k: round(v,3) for k,v in sorted(e["slowest_rank_breakdown_ms_per_step"].items())})'
done
