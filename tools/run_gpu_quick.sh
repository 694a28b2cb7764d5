#!/bin/bash
# quick GPU iteration: parity tests + C2/C3 bench lines (no ncu)
timeout 700 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest.log 2>&1; tail -3 gpurun_out/pytest.log
for c in ${CONFIGS:-c2 c3}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print(d['config']['workload'][:12], 'ms/step %.3f'%d['ms_per_step'], 'Gvox/s %.3f'%(d['value']/1e9), 'eval avg us %.1f'%r['avg_launch_us'], 'eval share %.2f'%r['eval_share_of_step'], 'launches', d['gpu_launches'], {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()})
    else: print(l.rstrip()[:300])
"
done
