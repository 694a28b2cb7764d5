#!/bin/bash
# bisect the global-mode mismatch: old tree (2ead905) vs current, balanced vs uniform slabs
mkdir -p gpurun_out
(cd .bisect/old && timeout 600 python tools/mg_check.py --config c2 --ranks 4 --iters 2) > gpurun_out/g22_old_c2.log 2>&1; echo "old c2 rc=$?"; grep "^iter [0-9]:" -A2 gpurun_out/g22_old_c2.log | head -8
timeout 600 python tools/mg_check.py --config c2 --ranks 4 --iters 2 --uniform > gpurun_out/g22_uni_c2.log 2>&1; echo "new uniform c2 rc=$?"; grep "^iter [0-9]:" -A2 gpurun_out/g22_uni_c2.log | head -8
timeout 600 python tools/mg_check.py --config c2 --ranks 2 --iters 2 --uniform > gpurun_out/g22_uni2_c2.log 2>&1; echo "new uniform 2 c2 rc=$?"; grep "^iter [0-9]:" -A2 gpurun_out/g22_uni2_c2.log | head -8
