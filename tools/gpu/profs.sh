ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 1 -c 1 \
  -o gpurun_out/solve_G${PSP_G:-1} -f python tools/gpu/diag.py --groups ${PSP_G:-1} --reps 1 --ladders 4096 > gpurun_out/ncu_s.log 2>&1; echo s=$?
