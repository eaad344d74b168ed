set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests -x -q -m gpu -k "spill or variant or tmem or fused or default_pivot or full_parity or ragged or random_patterns" > gpurun_out/r2_t2.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/r2_t2.log
CMD="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-latency-point"
$CMD > gpurun_out/r2_pb2.json 2> gpurun_out/r2_pb2.err && \
ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 1 \
    -o gpurun_out/r2_factor2 $CMD > gpurun_out/r2_ncu2.log 2>&1
echo rc=$?
