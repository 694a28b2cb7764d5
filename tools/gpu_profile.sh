#!/bin/bash
# Launch list + full ncu capture of the eval/commit kernels for one config.
# usage: tools/gpu_profile.sh <config> <skip> <count>
cfg=${1:-c2}; skip=${2:-20}; count=${3:-8}
args="--config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-passes"
python bench.py $args > gpurun_out/plain_$cfg.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_$cfg.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv \
    python bench.py $args > gpurun_out/ncu_launch_$cfg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_eval_p|k_commit" -s $skip -c $count \
    -o gpurun_out/full_$cfg python bench.py $args > gpurun_out/ncu_full_$cfg.log 2>&1
tail -1 gpurun_out/ncu_full_$cfg.log
