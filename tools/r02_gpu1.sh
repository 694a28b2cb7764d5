#!/bin/bash
# round 2, first GPU pass: GPU tests, C4 bench line (both arms), kernel launch list + ncu captures at C4
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest.log
timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench_c4.log | tail -1 > gpurun_out/bench_c4.json
timeout 1200 python bench.py --impl reference --steps 20 --warmup 3 --ref-budget 150 > gpurun_out/ref_c4.log 2>&1; echo "ref rc=$?"; tail -c 1500 gpurun_out/ref_c4.log
timeout 600 python tools/profile_kernels.py --config c4 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "profile/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/r02_c4_launches.csv python tools/profile_kernels.py --config c4 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_isobands|k_ccl_|k_agg_|k_vote|k_segments|k_move_sites|k_fill_state|k_state|k_site1_to_state|k_seed_groups|k_unpack" \
   -o gpurun_out/r02_c4_other python tools/profile_kernels.py --config c4 > gpurun_out/ncu_other.log 2>&1; echo "ncu other rc=$?"
timeout 1200 ncu --nvtx --nvtx-include "profile/" --set full --clock-control none --import-source on \
   -k regex:"k_eval_p|k_commit" -s 6 -c 8 \
   -o gpurun_out/r02_c4_eval python tools/profile_kernels.py --config c4 > gpurun_out/ncu_eval.log 2>&1; echo "ncu eval rc=$?"
ls -la gpurun_out
