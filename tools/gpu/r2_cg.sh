set -x
timeout 900 python -m pytest tests/test_gpu_coopg.py -q -x --durations=3 > gpurun_out/cg_tests.log 2>&1; echo tests=$?
tail -6 gpurun_out/cg_tests.log
timeout 600 python tools/gpu/cfgs.py 3,4 > gpurun_out/cg_cfgs.txt 2>&1; echo cfgs=$?
cat gpurun_out/cg_cfgs.txt
PSP_LIB=variants/cg16.so timeout 600 python tools/gpu/cfgs.py 3,4 2>&1 | tail -2
