"""Fig. 1 study on the GPU: 25 synthetic 300-bus Jacobians (operating
point re-drawn per trial), ladders alpha = 1..M at eps = 2e-3, all trials in ONE multi-Jacobian
batch (psp_factor_batch_multi / psp_solve_batch_multi / psp_recover); the relative residual
||J x_hat - b|| / ||b|| (psp_residual, on the device) per m, median / max over the trials,
for diagonal normal D (the library's path) and identity D."""
import os
import sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2311_11833_b200 import psp
from psp_inputs import config, ladder_eps

M = int(sys.argv[1]) if len(sys.argv) > 1 else 6
n_t = 25
mags = [2e-3 * j for j in range(1, M + 1)]
ss = [config(1).system(trial=t) for t in range(n_t)]
s0 = ss[0]
for dname in ("normal", "identity"):
    d = s0.d if dname == "normal" else np.ones(s0.n)
    eps = np.tile(ladder_eps(mags), n_t)
    sv = psp.Solver(0)
    sv.psp_symbolic_analyse(s0.n, s0.row_ptr, s0.col_idx)
    sv.psp_set_perturbations(eps, d)
    A = torch.tensor(np.stack([s.vals for s in ss]), dtype=torch.float64, device="cuda")
    B = torch.tensor(np.stack([s.b.T for s in ss]), dtype=torch.float64, device="cuda")
    sv.psp_factor_batch_multi(A, 0.0)
    sv.psp_solve_batch_multi(B)
    ptr, lane, val = [0], [], []
    for t in range(n_t):
        for m in range(1, M + 1):
            _, w = psp.psp_ladder_weights(mags[:m])
            for j, c in enumerate(w):
                lane.append(2 * M * t + j)
                val.append(c)
            ptr.append(len(lane))
    sv.psp_set_weights(np.array(ptr, np.int32), np.array(lane, np.int32), np.array(val))
    xh = sv.psp_recover()
    rc, st = sv.psp_get_lane_status()
    res = np.empty((n_t, M))
    for t in range(n_t):
        r = sv.psp_residual(A[t].contiguous(), B[t].contiguous(), xh[M * t:M * t + M].contiguous())
        res[t] = r[:, 0] / np.linalg.norm(ss[t].b[:, 0])
    print(f"D = {dname}: {n_t} trials x {2 * M} lanes in one batch (rc {rc}, kernels {sv.psp_get_last_kernels()})")
    print("  m (pairs):      " + " ".join(f"{m:9d}" for m in range(1, M + 1)))
    print("  median ||Jx-b||/||b||: " + " ".join(f"{v:9.2e}" for v in np.median(res, 0)))
    print("  max    ||Jx-b||/||b||: " + " ".join(f"{v:9.2e}" for v in res.max(0)))
    sv.close()
