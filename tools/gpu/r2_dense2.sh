set -x
timeout 900 python -m pytest tests/test_gpu_dense.py -q > gpurun_out/r2_dense_tests.log 2>&1; echo tests=$?
tail -30 gpurun_out/r2_dense_tests.log
timeout 300 python tools/gpu/dense_cmp.py > gpurun_out/r2_dense_cmp.txt 2>&1; echo cmp=$?
cat gpurun_out/r2_dense_cmp.txt
