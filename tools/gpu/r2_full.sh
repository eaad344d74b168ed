# full GPU test suite + smoke + default bench (round-end style)
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke_rc=$?
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2_gputests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/r2_gputests.log
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench_rc=$?
