set -x
timeout 600 python -m pytest tests/test_gpu_hybrid.py -q -x 2>&1 | tail -5
python - <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2311_11833_b200 import psp
from psp_inputs import config, ladder_eps
s = config(1).system()
A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
K = 65536
rng = np.random.default_rng(1)
eps = np.concatenate([ladder_eps([e * j for j in range(1, 5)]) for e in 10.0 ** rng.uniform(-3.3, -2.3, K // 8)])
for hyb in (2, 1, 3):
    sv = psp.Solver(0)
    sv.psp_set_option("phase_events", 1)
    sv.psp_set_option("factor_spill", 1)
    sv.psp_set_option("factor_hybrid", hyb)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx)
    sv.psp_set_perturbations(eps, s.d)
    for _ in range(3): sv.psp_factor_solve_batch(A, b, 0.0)
    sv.psp_get_phase_times()
    for _ in range(10): sv.psp_factor_solve_batch(A, b, 0.0)
    print("hybrid", hyb, "factor+fwd ms", sv.psp_get_phase_times(), flush=True)
PY
PSP_LIB=variants/wt.so python - <<'PY'
import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2311_11833_b200 import psp
from psp_inputs import config, ladder_eps
s = config(1).system()
A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
K = 65536
rng = np.random.default_rng(1)
eps = np.concatenate([ladder_eps([e * j for j in range(1, 5)]) for e in 10.0 ** rng.uniform(-3.3, -2.3, K // 8)])
sv = psp.Solver(0)
sv.psp_set_option("factor_spill", 1)
sv.psp_set_option("factor_hybrid", 3)
sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx)
sv.psp_set_perturbations(eps, s.d)
for _ in range(3): sv.psp_factor_solve_batch(A, b, 0.0)
torch.cuda.synchronize()
L = psp.lib()
out = np.zeros(16 * 4096, dtype=np.uint64)
L.psp_dbg_warp_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.psp_dbg_warp_times(out.ctypes.data, out.size)
t = out.reshape(-1, 16)
t = t[t[:, 0] > 0]
print("mix CTAs", len(t))
for w in range(10):
    v = t[:, w][t[:, w] > 0] / 1e3
    if len(v): print(f"warp {w}: mean {v.mean():.1f} us")
PY
