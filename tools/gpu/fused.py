"""Fused factor+solve (augmented program) vs factor_batch + solve_batch: bitwise and timing."""
import os
import sys
import time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2311_11833_b200 import psp
from psp_inputs import config

s = config(1).system()
A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
b = torch.tensor(s.b[:, 0].copy() if s.b.ndim == 2 else s.b.copy(), dtype=torch.float64, device="cuda")
for K in [int(k) for k in (sys.argv[1] if len(sys.argv) > 1 else "33,1000,8192,65536").split(",")]:
    rng = np.random.default_rng(K)
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-6, -2, K)
    out = []
    for fused in (False, True):
        sv = psp.Solver(0)
        sv.psp_set_option("solve_tmem", int(os.environ.get("PSP_STM", "0")))
        sv.psp_set_option("factor_warps", int(os.environ.get("PSP_FW", "0")))
        sv.psp_set_option("factor_tmem", int(os.environ.get("PSP_FT", "0")))
        sv.psp_set_option("coop", int(os.environ.get("PSP_COOP", "0")))
        sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
        info, perm = sv.psp_get_symbolic_info()
        sv.psp_set_perturbations(eps, s.d)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ts, t1 = [], []
        for rep in range(4):
            torch.cuda.synchronize()
            ev[0].record(sv.stream)
            if fused:
                sv.psp_factor_solve_batch(A, b, 1e-300)
                ev[1].record(sv.stream)
            else:
                sv.psp_factor_batch(A, 1e-300)
                ev[1].record(sv.stream)
                sv.psp_solve_batch(b.view(1, -1))
            ev[2].record(sv.stream)
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[2]))
            t1.append(ev[0].elapsed_time(ev[1]))
        X = sv.psp_get_solutions().cpu().numpy()
        F = [sv.psp_get_factor(k, info["nnz_LU"]) for k in (0, K - 1)]
        rc, st = sv.psp_get_lane_status()
        out.append((X, F, st))
        print(f"K={K} fused={fused} {min(ts[1:]):.3f} ms (first part {min(t1[1:]):.3f}) rc={rc}"
              f" solve_live_smem={info['solve_live_smem']} aug warps={info['aug_warps_per_cta']} pend={info['aug_pend_smem']}", flush=True)
        sv.close()
    same = np.array_equal(out[0][0], out[1][0]) and all(np.array_equal(a, c) for a, c in zip(out[0][1], out[1][1])) \
        and np.array_equal(out[0][2], out[1][2])
    bad = [k for k in range(K) if not np.array_equal(out[0][0][k], out[1][0][k])]
    print(f"K={K} bitwise {'OK' if same else 'MISMATCH'} lanes {bad[:8]}", flush=True)
