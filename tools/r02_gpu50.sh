#!/bin/bash
# public API with the C Site builder: API tests, e2e probe, bench e2e
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_classify.py tests/test_gpu_edges.py tests/test_gpu_bench.py tests/test_gpu_parity_big.py -k "not c5" -q -x -p no:cacheprovider > gpurun_out/g50.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g50.log
timeout 900 python tools/e2e_probe2.py c4
timeout 1200 python bench.py --steps 10 --warmup 3 --no-passes --no-cpu-baseline > gpurun_out/g50_c4.log 2>&1; echo "c4 rc=$?"; grep '^{' gpurun_out/g50_c4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("ms/step %.2f" % d["ms_per_step"], "e2e %.1f lazy %.1f" % (d["e2e"]["value"]/1e6, d["e2e"]["lazy"]["value"]/1e6))'
