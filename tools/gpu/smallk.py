"""Small-K latency of the factor/solve variants (BASELINE configs[1], K = 8)."""
import os
import sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2311_11833_b200 import psp
from psp_inputs import config

w = config(1)
s = w.system()
eps = w.eps()
A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
B = torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda")
ref = None
for gjpt in sys.argv[1].split(","):
    G, J, P, T, C = (int(x) for x in (gjpt + ":0:0:0:0").split(":")[:5])
    sv = psp.Solver(0)
    for k, v in (("factor_groups", G), ("factor_lanes", J), ("factor_slab_warps", P), ("factor_tmem", T), ("coop", C),
                 ("phase_events", 1)):
        sv.psp_set_option(k, v)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
    info, _ = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s.d)
    for _ in range(3):
        sv.psp_factor_batch(A, 0.0)
        sv.psp_solve_batch(B)
    sv.psp_get_phase_times()
    for _ in range(10):
        sv.psp_factor_batch(A, 0.0)
        sv.psp_solve_batch(B)
    tf, ts = sv.psp_get_phase_times()
    X = sv.psp_get_solutions().cpu().numpy()
    same = None if ref is None else bool(np.array_equal(X, ref))
    ref = X if ref is None else ref
    print(f"{gjpt}: G={info['factor_groups']} J={info['factor_lanes_per_thread']} P={info['factor_slab_warps']}"
          f" pend={info['factor_pend_smem']} factor {tf * 1e3:.0f} us solve {ts * 1e3:.0f} us bitwise={same}", flush=True)
    sv.close()
