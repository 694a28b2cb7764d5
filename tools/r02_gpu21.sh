#!/bin/bash
# global mode vs single domain at C4 (8 emulated slabs), iteration by iteration
mkdir -p gpurun_out
timeout 1500 python tools/mg_check.py --config c4 --ranks 8 --iters 4 > gpurun_out/g21_c4.log 2>&1; echo "c4 rc=$?"; tail -20 gpurun_out/g21_c4.log
timeout 900 python tools/mg_check.py --config c2 --ranks 4 --iters 4 > gpurun_out/g21_c2.log 2>&1; echo "c2 rc=$?"; tail -8 gpurun_out/g21_c2.log
