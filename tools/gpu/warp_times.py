"""Per-warp duration of the capacity-planned fused factor (experiment build with
-DPSP_WARP_TIMES: PSP_LIB=variants/wt.so): TMEM-slot warps (0..3) vs shared-memory-slot
warps (4..6), bench workload (K = 65536)."""
import ctypes
import os
import sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2311_11833_b200 import psp
from psp_inputs import config, ladder_eps

s = config(1).system()
A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
rng = np.random.default_rng(1)
eps = np.concatenate([ladder_eps([e * j for j in range(1, 5)]) for e in 10.0 ** rng.uniform(-3.3, -2.3, K // 8)])
sv = psp.Solver(0)
sv.psp_set_option("coop", 2)
sv.psp_set_option("factor_spill", 1)
if len(sys.argv) > 2:
    sv.psp_set_option("factor_warps", int(sys.argv[2]))
sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
sv.psp_set_perturbations(eps, s.d)
for _ in range(3):
    sv.psp_factor_solve_batch(A, b, 0.0)
torch.cuda.synchronize()
L = psp.lib()
out = np.zeros(8 * 4096, dtype=np.uint64)
L.psp_dbg_warp_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert L.psp_dbg_warp_times(out.ctypes.data, out.size) == 0
t = out.reshape(-1, 8)
t = t[t[:, 0] > 0]
print(f"K={K} CTAs={len(t)}")
for w in range(8):
    v = t[:, w][t[:, w] > 0] / 1e3
    if len(v):
        print(f"warp {w}: mean {v.mean():.1f} us  min {v.min():.1f}  max {v.max():.1f}")
