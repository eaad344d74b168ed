# one full ncu capture of the factor kernel (diag workload, variant $PSP_G)
ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 1 -c 1 \
  -o gpurun_out/factor_${PSP_TAG:-x} -f python tools/gpu/diag.py --groups ${PSP_G:-0} --reps 1 --ladders 8192 > gpurun_out/ncu_f.log 2>&1; echo f=$?
