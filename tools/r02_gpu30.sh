#!/bin/bash
# vote add: software-pipelined, branch-free 32-add batches
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_classify.py tests/test_gpu_parity_big.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g30_quick.log 2>&1; echo "quick rc=$?"; tail -2 gpurun_out/g30_quick.log
for cfg in "X=0" "LRCVT_VOTE_DEEP=1"; do
env $cfg timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_vote_(walk|add)" -c 3 --csv --log-file gpurun_out/g30_$cfg.csv python bench.py --steps 1 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g30_ncu.log 2>&1; echo "ncu $cfg rc=$?"
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g30_c4.log 2>&1; grep '^{' gpurun_out/g30_c4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})'
