import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from oracle import ordering
from paper_2311_11833_b200 import psp
from psp_inputs import config
for ci in (0, 1):
    w = config(ci); s = w.system(); eps = w.eps()
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    for lz in (False, True):
        first = s.slot_p if lz else -1
        operm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx, first=None if first < 0 else first)
        Xo, sto = oracle.dense_batch(s, operm, eps, tol)
        for G, J, P, T in ((1, 1, 1, 0), (1, 1, 1, 2), (1, 1, 2, 0), (2, 1, 1, 0), (2, 2, 1, 0), (4, 1, 1, 0), (4, 2, 1, 0)):
            sv = psp.Solver(0); sv.psp_set_option("factor_groups", G); sv.psp_set_option("factor_lanes", J)
            sv.psp_set_option("factor_slab_warps", P); sv.psp_set_option("factor_tmem", T)
            sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg_first" if lz else "mindeg", first_node=first)
            sv.psp_set_perturbations(eps, s.d)
            A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
            sv.psp_factor_batch(A, tol)
            sv.psp_solve_batch(torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda"))
            X = sv.psp_get_solutions().cpu().numpy()
            rc, st = sv.psp_get_lane_status()
            badl = [k for k in range(len(eps)) if not np.array_equal(X[k], Xo[k])]
            print(ci, lz, f"{G}:{J}:{P}:{T}:{sv.psp_get_symbolic_info()[0]['factor_pend_smem']}", rc, "bitwise" if not badl else f"MISMATCH lanes {badl[:8]}", flush=True)
            sv.close()
