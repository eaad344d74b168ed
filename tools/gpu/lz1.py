import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from oracle import ordering
from paper_2311_11833_b200 import psp
from psp_inputs import config
G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
w = config(0); s = w.system(); eps = w.eps()
tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
first = s.slot_p
operm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx, first=first)
Xo, sto = oracle.dense_batch(s, operm, eps, tol)
sv = psp.Solver(0); sv.psp_set_option("factor_groups", G)
sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg_first", first_node=first)
sv.psp_set_perturbations(eps, s.d)
A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
sv.psp_factor_batch(A, tol)
sv.psp_solve_batch(torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda"))
X = sv.psp_get_solutions().cpu().numpy()
print("G", G, "maxdiff", np.abs(X - Xo).max())
