#!/bin/bash
# vote: SoA site/phi planes for the walks; add kernel source-level profile
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_classify.py tests/test_gpu_parity_big.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g31_quick.log 2>&1; echo "quick rc=$?"; tail -2 gpurun_out/g31_quick.log
LRCVT_VOTE_DEEP=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_vote_(walk|add|prep)" -c 4 --csv --log-file gpurun_out/g31_vote.csv python bench.py --steps 1 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g31_ncu.log 2>&1; echo "ncu rc=$?"
LRCVT_VOTE_DEEP=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_vote_add" -c 1 -o gpurun_out/g31_add python bench.py --steps 1 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g31_full.log 2>&1; echo "full rc=$?"
