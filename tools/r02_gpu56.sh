#!/bin/bash
# reuse runs start from a fresh eligible list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g56.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/g56.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g56_c4.log 2>&1; grep '^{' gpurun_out/g56_c4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("ms/step %.2f" % d["ms_per_step"])'
