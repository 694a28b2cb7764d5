#!/bin/bash
# p1 halo emission restored: MG parity at scale + emulated 8-slab timing
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_edges.py tests/test_capi.py -q -x -p no:cacheprovider > gpurun_out/g25_multi.log 2>&1; echo "multi rc=$?"; tail -2 gpurun_out/g25_multi.log
timeout 1500 python tools/mg_check.py --config c4 --ranks 8 --iters 3 > gpurun_out/g25_c4.log 2>&1; echo "c4 check rc=$?"; grep "^iter [0-9]:" -A2 gpurun_out/g25_c4.log; tail -1 gpurun_out/g25_c4.log
timeout 1200 python bench.py --mode global --emulate-ranks 8 --steps 3 --warmup 3 > gpurun_out/g25_global8.log 2>&1; echo "global8 rc=$?"; grep '^{' gpurun_out/g25_global8.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["emulated_ranks"]; print(d["ms_per_step"], round(e["slowest_rank_ms_per_step"],2), {k: round(v,2) for k,v in e["rank_ms_per_step"].items()}); print({k: round(v,3) for k,v in sorted(e["slowest_rank_breakdown_ms_per_step"].items())}); print(e["slowest_rank_calls_per_step"]); print(d["counters"])'
