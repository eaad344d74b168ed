"""Per-round factor time of the capacity-planned (spill) fused factor vs resident warps
per SM: K = 148 x warps x 64 lanes (exactly one round), PSP_OPT_FACTOR_WARPS forced."""
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
for w in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4,5,6,7").split(",")]:
    for K in (148 * w * 64, 148 * 7 * 64):
        rng = np.random.default_rng(1)
        G = K // 8
        eps = np.concatenate([ladder_eps([e * j for j in range(1, 5)]) for e in 10.0 ** rng.uniform(-3.3, -2.3, G)])
        sv = psp.Solver(0)
        sv.psp_set_option("phase_events", 1)
        sv.psp_set_option("coop", 2)
        sv.psp_set_option("factor_spill", 1)
        sv.psp_set_option("factor_warps", w)
        sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
        info, _ = sv.psp_get_symbolic_info()
        sv.psp_set_perturbations(eps, s.d)
        for _ in range(3):
            sv.psp_factor_solve_batch(A, b, 0.0)
        sv.psp_get_phase_times()
        for _ in range(5):
            sv.psp_factor_solve_batch(A, b, 0.0)
        tf, ts = sv.psp_get_phase_times()
        print(f"warps={w} K={K} rounds={K / (148 * w * 64):.2f} factor {tf:.3f} ms ({K / tf / 1e3:.1f} M lanes/s) "
              f"kernels {sv.psp_get_last_kernels()} spill_warps {info['spill_warps_per_cta']}", flush=True)
        sv.close()
