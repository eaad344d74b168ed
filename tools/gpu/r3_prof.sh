# one ncu --set full capture (with source) of the bench's factor kernel
set -x
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-latency-point"
$CMD > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 1 \
    -o gpurun_out/p_factor -f $CMD > gpurun_out/p_ncu.log 2>&1
echo rc=$?
cp paper_2311_11833_b200/libpsp.so gpurun_out/p_libpsp.so
