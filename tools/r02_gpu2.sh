#!/bin/bash
# compaction change: quick parity, then big parity, A/B vs the previous library, ncu of the eval/commit/compact kernels
mkdir -p gpurun_out; free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
timeout 600 python -m pytest tests/test_gpu_classify.py tests/test_gpu_warp_eval.py tests/test_gpu_edges.py -q -x -p no:cacheprovider > gpurun_out/g2_quick.log 2>&1; echo "quick rc=$?"; tail -3 gpurun_out/g2_quick.log
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/g2_all.log 2>&1; echo "all rc=$?"; tail -25 gpurun_out/g2_all.log
for rep in 1 2; do
 for lib in ab/liblrcvt_r02a.so paper_2208_06970_b200/liblrcvt_cuda.so; do
  LRCVT_LIB=$lib timeout 900 python bench.py --steps 10 --warmup 3 --no-passes --no-e2e --no-cpu-baseline > gpurun_out/g2_ab.log 2>&1
  echo "$lib $(grep '^{' gpurun_out/g2_ab.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("ms/step %.2f" % d["ms_per_step"], r["breakdown_ms_per_step"], "E", d["counters"]["E_per_step"])')" >> gpurun_out/g2_ab.txt
 done
done
cat gpurun_out/g2_ab.txt
timeout 600 python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g2_prof_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "profile/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/r02b_c4_launches.csv python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g2_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_eval_p|k_commit|k_compact" -s 12 -c 9 \
   -o gpurun_out/r02b_c4_eval python tools/profile_kernels.py --config c4 --host-rounds > gpurun_out/g2_ncu_eval.log 2>&1; echo "ncu eval rc=$?"
