ncu --set full --clock-control none -k regex:recover -s 1 -c 1 -o gpurun_out/recover -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_r.log 2>&1; echo r=$?
