#!/bin/bash
# final tree: quick GPU suites + smoke
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g52.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/g52.log
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -1
