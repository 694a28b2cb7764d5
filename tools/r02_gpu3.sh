#!/bin/bash
# sparse proposals (no block barrier), CTA-size and compaction variants, bbox vote: parity under each, then A/B at C4
mkdir -p gpurun_out
T="tests/test_gpu_classify.py tests/test_gpu_warp_eval.py tests/test_gpu_edges.py tests/test_gpu_multi.py tests/test_gpu_seeding.py tests/test_gpu_blocks.py"
for env in "X=0" "LRCVT_COMPACT=1" "LRCVT_EVAL_BS=32,32" "LRCVT_VOTE=sort"; do
  env $env timeout 900 python -m pytest $T -q -x -p no:cacheprovider > gpurun_out/g3_t.log 2>&1; echo "tests [$env] rc=$? $(tail -1 gpurun_out/g3_t.log)"
done
env LRCVT_COMPACT=1 LRCVT_EVAL_BS=32,32 timeout 900 python -m pytest tests/test_gpu_parity_big.py -q -x -p no:cacheprovider -k c4 > gpurun_out/g3_big.log 2>&1; echo "big c4 [compact bs32] rc=$? $(tail -1 gpurun_out/g3_big.log)"
timeout 900 python -m pytest tests/test_gpu_parity_big.py -q -x -p no:cacheprovider -k c4 > gpurun_out/g3_big.log 2>&1; echo "big c4 [default] rc=$? $(tail -1 gpurun_out/g3_big.log)"
rm -f gpurun_out/g3_ab.txt
for rep in 1 2; do
 for cfg in "LRCVT_LIB=ab/liblrcvt_r02a.so" "X=0" "LRCVT_COMPACT=1" "LRCVT_EVAL_BS=32,32" "LRCVT_EVAL_BS=32,64" "LRCVT_EVAL_BS=128,32" "LRCVT_COMPACT=1 LRCVT_EVAL_BS=32,32" "LRCVT_VOTE=sort"; do
  env $cfg timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g3_ab.log 2>&1
  echo "[$cfg] $(grep '^{' gpurun_out/g3_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], {k: round(v,2) for k,v in r["breakdown_ms_per_step"].items()})')" >> gpurun_out/g3_ab.txt
 done
done
cat gpurun_out/g3_ab.txt
timeout 600 python tools/region_stats.py --config c4 > gpurun_out/g3_regions.txt 2>&1; tail -8 gpurun_out/g3_regions.txt
