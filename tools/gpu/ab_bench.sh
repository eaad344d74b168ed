# A/B of library builds through bench.py itself (factor / solve / recover phase times of
# the bench workload): tools/gpu/ab_bench.sh OUT LIB1 LIB2 ...   (3 alternating rounds)
out=$1; shift
: > gpurun_out/$out
for r in 1 2 3; do
  for lib in "$@"; do
    PSP_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency-point 2>/dev/null \
      | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms']
        print('$lib', 'round $r', 'step %.4f factor %.4f solve %.4f recover %.4f bitwise %s' % (d['ms_per_step'], p['factor'], p['solve'], p['recover'], d.get('rel_err_vs_oracle',{}).get('bitwise')))
" >> gpurun_out/$out
  done
done
cat gpurun_out/$out
