#!/bin/bash
# vote: segment counts from the eligible list instead of a count walk
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g39_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/g39_gpu.log
timeout 1500 python tools/mg_check.py --config c4 --ranks 8 --iters 2 > gpurun_out/g39_c4.log 2>&1; echo "c4 check rc=$?"; tail -1 gpurun_out/g39_c4.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g39_c4b.log 2>&1; grep '^{' gpurun_out/g39_c4b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_vote|k_scan" -c 12 --csv --log-file gpurun_out/g39_vote.csv python bench.py --steps 1 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g39_ncu.log 2>&1; echo "ncu rc=$?"
