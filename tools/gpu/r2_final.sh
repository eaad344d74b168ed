# round-2 final evidence on HEAD: smoke, GPU tests, default bench line, ncu launch list,
# one ncu --set full capture each of the bench's factor and backward-solve kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke_rc=$?
timeout 2400 python -m pytest tests -q -m gpu -x --durations=5 > gpurun_out/f_gputests.log 2>&1; echo tests_rc=$?
tail -8 gpurun_out/f_gputests.log
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-latency-point"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv \
  $CMD > gpurun_out/f_ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 1 \
  -o gpurun_out/f_factor_full -f $CMD > gpurun_out/f_ncu_ff.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_kernel_tmem -s 3 -c 1 \
  -o gpurun_out/f_solve_full -f $CMD > gpurun_out/f_ncu_sf.log 2>&1; echo ncu3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:recover_blk -s 3 -c 1 \
  -o gpurun_out/f_recover_full -f $CMD > gpurun_out/f_ncu_rf.log 2>&1; echo ncu4=$?
python tools/gpu/ksweep.py > gpurun_out/f_ksweep.txt 2>&1; echo ksweep=$?
