# e2e leg of bench.py (default flags) next to tools/gpu/e2e.py on the same box
python tools/gpu/e2e.py 2>&1 | grep "async N=20"
for i in 1 2 3; do
python bench.py 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('bench e2e ms/step', d['e2e']['ms_per_step'], 'device', d['ms_per_step'], d['e2e']['matches_device_result'])"
done
