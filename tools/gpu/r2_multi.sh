set -x
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x --durations=3 > gpurun_out/multi_tests.log 2>&1; echo tests=$?
tail -8 gpurun_out/multi_tests.log
timeout 300 python tools/gpu/fig1.py 6 > gpurun_out/fig1.txt 2>&1; echo fig1=$?
cat gpurun_out/fig1.txt
