# A/B of the smallest size-class cap (LRCVT_CLASS0 builds under build/c<cap>/)
LRCVT_LIB=build/c8192/liblrcvt_cuda.so timeout 600 python -m pytest tests/test_gpu_classify.py tests/test_gpu_warp_eval.py -x -q > gpurun_out/c0_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c0_tests.log
for rep in 1 2; do
for c in c1 c2 c3; do
for lib in paper_2208_06970_b200 build/c4096 build/c8192; do
  LRCVT_LIB=$lib/liblrcvt_cuda.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-passes 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('$lib', '$c', 'ms/step %.4f'%d['ms_per_step'], {k: round(v,4) for k,v in r['breakdown_ms_per_step'].items()})
" >> gpurun_out/c0_ab.txt
done; done; done
