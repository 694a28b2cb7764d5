#!/bin/bash
# global mode: one collective per round (sizes + frontier + commits in the halo all-gather), P2P halos
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bench.py tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/g38.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/g38.log
timeout 1500 python tools/mg_check.py --config c4 --ranks 8 --iters 2 > gpurun_out/g38_c4.log 2>&1; echo "c4 check rc=$?"; tail -1 gpurun_out/g38_c4.log
timeout 1200 python bench.py --mode global --emulate-ranks 8 --steps 3 --warmup 3 > gpurun_out/g38_global8.log 2>&1; echo "global8 rc=$?"; grep '^{' gpurun_out/g38_global8.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["emulated_ranks"]; print(d["ms_per_step"], round(e["slowest_rank_ms_per_step"],2), d["counters"])'
LRCVT_BENCH_DEVICE=0 LRCVT_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --config c2 --steps 3 --warmup 3 > gpurun_out/g38_2r.log 2>&1; echo "2 ranks rc=$?"; grep '^{' gpurun_out/g38_2r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["counters"])'
