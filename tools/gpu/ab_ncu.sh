# ncu --set full of the bench factor kernel for each library given (PSP_LIB), via tools/gpu/ab.py's workload
for L in "$@"; do
  N=$(basename $L .so)
  PSP_LIB=$PWD/$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 1 \
    -o gpurun_out/abn_$N -f python tools/gpu/ab.py $L --rounds 1 --steps 2 > gpurun_out/abn_$N.log 2>&1; echo "$N rc=$?"
done
