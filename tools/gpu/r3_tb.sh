# GPU tests (stop at first failure) + default bench line; TAG names the outputs
set -x
T=${TAG:-x}
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_gputests.log 2>&1; echo tests_rc=$?
tail -4 gpurun_out/${T}_gputests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench=$?
python - <<'PY'
import json,os
d=json.loads(open(f"gpurun_out/{os.environ.get('TAG','x')}_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], d["phases_ms"], "frac", d["roofline"]["frac"], "parity", d.get("rel_err_vs_oracle"))
PY
