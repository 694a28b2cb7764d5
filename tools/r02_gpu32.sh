#!/bin/bash
# validation: GPU suites (no C5), bench C4 with e2e, global8
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g32_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/g32_gpu.log
timeout 1200 python bench.py --steps 10 --warmup 3 --no-passes --no-cpu-baseline > gpurun_out/g32_c4.log 2>&1; echo "c4 rc=$?"; grep '^{' gpurun_out/g32_c4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()}, "e2e %.1f lazy %.1f" % (d["e2e"]["value"]/1e6, d["e2e"]["lazy"]["value"]/1e6))'
timeout 1200 python bench.py --mode global --emulate-ranks 8 --steps 3 --warmup 3 > gpurun_out/g32_global8.log 2>&1; echo "global8 rc=$?"; grep '^{' gpurun_out/g32_global8.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["emulated_ranks"]; print(d["ms_per_step"], round(e["slowest_rank_ms_per_step"],2), {k: round(v,2) for k,v in e["rank_ms_per_step"].items()}); print({k: round(v,3) for k,v in sorted(e["slowest_rank_breakdown_ms_per_step"].items())})'
