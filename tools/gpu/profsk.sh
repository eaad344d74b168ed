# full ncu captures of the factor and solve at K = 8 (BASELINE configs[1], latency-bound)
ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 3 -c 1 \
  -o gpurun_out/sk_solve -f python tools/gpu/smallk.py 1:1:1:2 > gpurun_out/ncu_sk_s.log 2>&1; echo s=$?
ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 1 \
  -o gpurun_out/sk_factor -f python tools/gpu/smallk.py 1:1:1:2 > gpurun_out/ncu_sk_f.log 2>&1; echo f=$?
