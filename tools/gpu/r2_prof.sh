# bench (short) then one ncu --set full capture of the factor kernel of the same command
set -x
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-latency-point"
$CMD > gpurun_out/r2_pb.json 2> gpurun_out/r2_pb.err && \
ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 1 \
    -o gpurun_out/r2_factor $CMD > gpurun_out/r2_ncu.log 2>&1
echo rc=$?
