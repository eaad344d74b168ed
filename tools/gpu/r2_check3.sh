set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "spill or fused or variant or tmem or full_parity or ragged" > gpurun_out/r2_t6.log 2>&1; echo tests_rc=$?
tail -2 gpurun_out/r2_t6.log
CMD="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-latency-point"
$CMD > gpurun_out/r2_pb6.json 2> gpurun_out/r2_pb6.err && \
ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 1 \
    -o gpurun_out/r2_factor6 $CMD > gpurun_out/r2_ncu6.log 2>&1
echo rc=$?
