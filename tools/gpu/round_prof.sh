# bench + ncu launch list + one full capture of the factor and solve kernels (bench workload)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-latency-point > gpurun_out/ncu_launch_r1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 1 \
  -o gpurun_out/factor_full_r1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-latency-point > gpurun_out/ncu_ff_r1.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 3 -c 1 \
  -o gpurun_out/solve_full_r1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-latency-point > gpurun_out/ncu_sf_r1.log 2>&1; echo ncu3=$?
