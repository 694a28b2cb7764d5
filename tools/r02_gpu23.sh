#!/bin/bash
mkdir -p gpurun_out
for dbg in 8 17 31; do
LRCVT_MG_DEBUG=$dbg timeout 600 python tools/mg_check.py --config c2 --ranks 2 --iters 1 --uniform > gpurun_out/g24_$dbg.log 2>&1; echo "dbg=$dbg rc=$?"; grep "^iter [0-9]:" -A2 gpurun_out/g24_$dbg.log | head -3
done
