set -x
timeout 300 python tools/gpu/diag.py --reps 3 > gpurun_out/diag2.log 2>&1; echo diag=$?
cat gpurun_out/diag2.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu2.log
