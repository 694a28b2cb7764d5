#!/bin/bash
# A/B: run the bench on each library build given as build/<name>/liblrcvt_cuda.so
cfgs=${CONFIGS:-c2 c3}
for d in "$@"; do
  for c in $cfgs; do
    LRCVT_LIB=$d/liblrcvt_cuda.so python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --no-passes 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('$d', d['config']['workload'][:3], 'ms/step %.3f'%d['ms_per_step'], {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()})
"
  done
done
