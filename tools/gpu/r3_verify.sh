# round-2 (resumed) verification of HEAD: smoke, GPU tests, default bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/v_smoke.log
timeout 2400 python -m pytest tests -q -m gpu -x --durations=10 > gpurun_out/v_gputests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/v_gputests.log
timeout 900 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo bench=$?
tail -c 1500 gpurun_out/v_bench.json
