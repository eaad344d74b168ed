import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from paper_2311_11833_b200 import psp
from psp_inputs import config
w = config(0); s = w.system(); eps = w.eps()
tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
F = {}
for G in (4, 8):
    sv = psp.Solver(0); sv.psp_set_option("factor_groups", G)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg_first", first_node=s.slot_p)
    info, perm = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s.d)
    sv.psp_factor_batch(torch.tensor(s.vals, dtype=torch.float64, device="cuda"), tol)
    torch.cuda.synchronize()
    F[G] = np.stack([sv.psp_get_factor(k, info["nnz_LU"]) for k in range(len(eps))])
    print(G, info)
d = np.argwhere(F[4] != F[8])
print("n diff", len(d), "nnz_L", info["nnz_L"], d[:20].tolist())
for k in range(1):
    for it in np.argwhere(F[4][k] != F[8][k]).ravel():
        print(it, F[4][k, it], F[8][k, it], (F[8][k, it] - F[4][k, it]) / abs(F[4][k, it]))
