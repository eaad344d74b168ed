"""Factor/solve timings of the BASELINE configs (cfg0-4) through both paths."""
import os
import sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2311_11833_b200 import psp
from psp_inputs import config

for ci in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3,4").split(",")]:
    w = config(ci)
    s = w.system()
    eps = w.eps()
    sv = psp.Solver(0)
    sv.psp_set_option("phase_events", 1)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
    info, perm = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s.d)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    B = torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda")
    for _ in range(3):
        sv.psp_factor_batch(A, 0.0)
        sv.psp_solve_batch(B)
    sv.psp_get_phase_times()
    for _ in range(5):
        sv.psp_factor_batch(A, 0.0)
        sv.psp_solve_batch(B)
    tf, ts = sv.psp_get_phase_times()
    tff = None
    if B.shape[0] == 1:
        for _ in range(3):
            sv.psp_factor_solve_batch(A, B[0].contiguous(), 0.0)
        sv.psp_get_phase_times()
        for _ in range(5):
            sv.psp_factor_solve_batch(A, B[0].contiguous(), 0.0)
        tff = sv.psp_get_phase_times()
    print(f"cfg{ci} n={s.n} K={len(eps)} R={B.shape[0]} slots={info['max_live']} pend={info['factor_pend_smem']}"
          f" warps={info['factor_warps_per_cta']} factor {tf:.3f} ms solve {ts:.3f} ms fused {tff}", flush=True)
    sv.close()
