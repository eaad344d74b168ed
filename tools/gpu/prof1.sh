# launch list + one full capture of the factor kernel (interpreter variant)
set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ladders 8192 > gpurun_out/prof_bench.log 2>&1; echo bench=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 2 -c 1 \
  -o gpurun_out/factor_full -f python tools/gpu/diag.py --variants 0 --reps 2 --ladders 4096 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 2 -c 1 \
  -o gpurun_out/solve_full -f python tools/gpu/diag.py --variants 0 --reps 2 --ladders 4096 > gpurun_out/ncu_full2.log 2>&1; echo ncu3=$?
