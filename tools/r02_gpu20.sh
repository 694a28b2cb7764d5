#!/bin/bash
# emulated 8-slab C4: per-category / per-size-class breakdown; warp-eval threshold sweep
mkdir -p gpurun_out
for ew in 2048 8192 32768; do
LRCVT_EW_SMALL=$ew timeout 1200 python bench.py --mode global --emulate-ranks 8 --steps 3 --warmup 3 > gpurun_out/g20_global8_$ew.log 2>&1; echo "global8 ew=$ew rc=$?"; grep '^{' gpurun_out/g20_global8_$ew.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["emulated_ranks"]; print(d["ms_per_step"], round(e["slowest_rank_ms_per_step"],2), {k: round(v,2) for k,v in e["rank_ms_per_step"].items()}); print({k: round(v,3) for k,v in sorted(e["slowest_rank_breakdown_ms_per_step"].items())}); print(e["slowest_rank_calls_per_step"])'
done
