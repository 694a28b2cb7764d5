#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bench.py tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/g37.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/g37.log
