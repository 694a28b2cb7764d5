#!/bin/bash
# public API: cached Site-list arrays; e2e probe + bench e2e
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_classify.py tests/test_gpu_edges.py tests/test_gpu_bench.py tests/test_gpu_parity_big.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g34_quick.log 2>&1; echo "quick rc=$?"; tail -2 gpurun_out/g34_quick.log
timeout 900 python tools/e2e_probe2.py c4
timeout 1200 python bench.py --steps 10 --warmup 3 --no-passes --no-cpu-baseline > gpurun_out/g34_c4.log 2>&1; echo "c4 rc=$?"; grep '^{' gpurun_out/g34_c4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], "e2e %.1f lazy %.1f" % (d["e2e"]["value"]/1e6, d["e2e"]["lazy"]["value"]/1e6))'
