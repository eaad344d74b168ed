# one full ncu capture of kernel $PSP_K (regex) on the diag workload, variant $PSP_G
ncu --set full --clock-control none --import-source on -k regex:${PSP_K:-factor_kernel} -s 1 -c 1 \
  -o gpurun_out/${PSP_TAG:-x} -f python tools/gpu/diag.py --groups ${PSP_G:-0} --reps 1 --ladders 8192 > gpurun_out/ncu_${PSP_TAG:-x}.log 2>&1; echo ${PSP_TAG:-x}=$?
