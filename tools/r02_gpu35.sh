#!/bin/bash
mkdir -p gpurun_out gpurun_out/g36
timeout 1200 python -m pytest tests/test_gpu_bench.py -q -x -p no:cacheprovider -k "two_ranks" > gpurun_out/g35.log 2>&1; echo "rc=$?"; tail -30 gpurun_out/g35.log
#!/bin/bash
mkdir -p gpurun_out/g36
LRCVT_BENCH_DEVICE=0 LRCVT_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --config c2 --steps 2 --warmup 3 > gpurun_out/g36/out.log 2>&1; echo "rc=$?"
grep -v "^\s*$" gpurun_out/g36/out.log | grep -B5 -A25 "rank0\]\|Abort\|abort\|what()" | head -80
