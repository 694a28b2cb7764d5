# round-end records: GPU parity suite, bench lines C1-C5 + reference arm, C2/C3 launch lists
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f_gpu_tests.log
timeout 400 python bench.py > gpurun_out/f_bench_c2.json 2> gpurun_out/f_bench_c2.err
timeout 400 python bench.py --impl reference > gpurun_out/f_bench_reference_c2.json 2> gpurun_out/f_ref.err
for c in c1 c3; do timeout 400 python bench.py --config $c > gpurun_out/f_bench_$c.json 2> gpurun_out/f_bench_$c.err; done
timeout 600 python bench.py --config c4 --steps 3 > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
for c in c2 c3; do
  args="--config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-passes"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py $args > gpurun_out/ncu_launch_$c.log 2>&1
done
timeout 900 python bench.py --config c5 --steps 3 --no-e2e > gpurun_out/f_bench_c5.json 2> gpurun_out/f_bench_c5.err
echo finished
