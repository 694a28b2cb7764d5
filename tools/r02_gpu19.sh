#!/bin/bash
# p1: warp-uniform skip of table batches without foreign sites and of warps without candidates
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_classify.py tests/test_gpu_warp_eval.py tests/test_gpu_parity_big.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g19_quick.log 2>&1; echo "quick rc=$?"; tail -2 gpurun_out/g19_quick.log
for rep in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g19_ab.log 2>&1
echo "$(grep '^{' gpurun_out/g19_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')"
done
