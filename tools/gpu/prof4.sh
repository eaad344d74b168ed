for GJ in ${PSP_G:-1:1}; do
G=${GJ%%:*}; 
ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 1 -c 1 \
  -o gpurun_out/factor_G$G -f python tools/gpu/diag.py --groups $GJ --reps 1 --ladders 4096 > gpurun_out/ncu_f$G.log 2>&1; echo f$G=$?
done
