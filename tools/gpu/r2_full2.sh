# full GPU suite (durations), smoke, default bench, config lines (dense / large), launch list
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/r2b_smoke.log
timeout 2400 python -m pytest tests -q -m gpu --durations=40 > gpurun_out/r2b_gputests.log 2>&1; echo tests_rc=$?
grep -E "passed|failed" gpurun_out/r2b_gputests.log | tail -3
timeout 600 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo bench_rc=$?
timeout 600 python tools/gpu/cfgs.py > gpurun_out/r2b_cfgs.txt 2>&1; echo cfgs=$?
cat gpurun_out/r2b_cfgs.txt
timeout 300 python tools/gpu/dense_cmp.py > gpurun_out/r2b_dense_cmp.txt 2>&1; echo dense=$?
cat gpurun_out/r2b_dense_cmp.txt
