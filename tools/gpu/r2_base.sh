# round-2 checkpoint: smoke, GPU tests, default bench, ncu launch list, factor full capture
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2_gputests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/r2_gputests.log
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench_rc=$?
cat gpurun_out/r2_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-latency-point > gpurun_out/r2_ncu_launch.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 1 \
  -o gpurun_out/r2_factor_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-latency-point > gpurun_out/r2_ncu_ff.log 2>&1; echo ncu2=$?
