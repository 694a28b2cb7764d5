#!/bin/bash
mkdir -p gpurun_out
./tools/micro/dadd_latency
timeout 600 python tools/region_stats.py > gpurun_out/g28_regions.log 2>&1; echo "regions rc=$?"; tail -15 gpurun_out/g28_regions.log
