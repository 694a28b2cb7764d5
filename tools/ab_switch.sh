set -x
timeout 600 python -m pytest tests/test_gpu_classify.py tests/test_gpu_warp_eval.py tests/test_gpu_multi.py -x -q > gpurun_out/sw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sw_tests.log
for rep in 1 2; do
for c in c1 c2 c3 c4; do
for sw in 0 1; do
  LRCVT_SWITCH=$sw timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-passes 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('sw=$sw', '$c', 'ms/step %.4f'%d['ms_per_step'], {k: round(v,4) for k,v in r['breakdown_ms_per_step'].items()})
" >> gpurun_out/sw_ab.txt
done; done; done
