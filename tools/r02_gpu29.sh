#!/bin/bash
# vote add pipeline depth A/B; ncu --set full of the walk / add kernels
mkdir -p gpurun_out
for cfg in "X=0" "LRCVT_VOTE_DEEP=1"; do
env $cfg timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_vote_(walk|add)" -c 3 --csv --log-file gpurun_out/g29_$cfg.csv python bench.py --steps 1 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g29_ncu.log 2>&1; echo "ncu $cfg rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_vote_(walk|add)" -c 3 -o gpurun_out/g29_vote python bench.py --steps 1 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g29_full.log 2>&1; echo "full rc=$?"
