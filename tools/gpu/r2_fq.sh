# factor experiment: spill/fused parity tests + short bench (factor ms)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "spill_factor or fused_factor_solve or bench_size or tmem_variant" --durations=10 > gpurun_out/fq_tests.log 2>&1; echo tests=$?
tail -20 gpurun_out/fq_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-latency-point > gpurun_out/fq_bench.json 2> gpurun_out/fq_bench.err; echo bench=$?
grep -o '"phases_ms": {[^}]*}' gpurun_out/fq_bench.json
