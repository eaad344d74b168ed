# full ncu captures of the factor and solve kernels inside bench.py (fused path by default)
ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 1 \
  -o gpurun_out/${PSP_TAG:-b}_factor -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline $PSP_ARGS > gpurun_out/ncu_${PSP_TAG:-b}_f.log 2>&1; echo f=$?
ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 3 -c 1 \
  -o gpurun_out/${PSP_TAG:-b}_solve -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline $PSP_ARGS > gpurun_out/ncu_${PSP_TAG:-b}_s.log 2>&1; echo s=$?
