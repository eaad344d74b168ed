# dense DMMA path: FP64 peak probe, dense GPU tests, dense vs sparse timings, ncu of the dense LU
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/probe/fp64mma.cu -o /tmp/fp64mma && /tmp/fp64mma > gpurun_out/r2_fp64mma.txt 2>&1; echo probe=$?
cat gpurun_out/r2_fp64mma.txt
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x > gpurun_out/r2_dense_tests.log 2>&1; echo tests=$?
tail -30 gpurun_out/r2_dense_tests.log
timeout 300 python tools/gpu/dense_cmp.py > gpurun_out/r2_dense_cmp.txt 2>&1; echo cmp=$?
cat gpurun_out/r2_dense_cmp.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_lu -s 3 -c 1 \
  -o gpurun_out/r2_dense_lu -f python tools/gpu/dense_cmp.py 2 > gpurun_out/r2_ncu_dense.log 2>&1; echo ncu=$?
