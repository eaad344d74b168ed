set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo smoke_rc=$?
tail -1 gpurun_out/r2c_smoke.log
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/r2c_gputests.log 2>&1; echo tests_rc=$?
grep -E "passed|failed|^FAILED" gpurun_out/r2c_gputests.log | tail -12
timeout 300 python tools/gpu/latency.py > gpurun_out/r2c_latency.txt 2>&1; cat gpurun_out/r2c_latency.txt
timeout 600 python tools/gpu/cfgs.py 3,4 > gpurun_out/r2c_cfgs.txt 2>&1; cat gpurun_out/r2c_cfgs.txt
