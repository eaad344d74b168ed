set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests -x -q -m gpu -k "spill or predicted or pivoted or variant or tmem or fused or default_pivot" > gpurun_out/r2_t1.log 2>&1; echo tests_rc=$?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b1.json 2> gpurun_out/r2_b1.err; echo bench_rc=$?
tail -5 gpurun_out/r2_t1.log
