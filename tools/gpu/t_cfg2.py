import time, sys, os
sys.path.insert(0, os.getcwd())
t0=time.time()
import numpy as np, torch
import oracle
from oracle import ordering
from psp_inputs import config
from paper_2311_11833_b200 import psp
def T(msg): print(f"{time.time()-t0:8.2f}s {msg}", flush=True)
w = config(2); s = w.system(); eps = w.eps(); T("inputs")
tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
sv = psp.Solver(0); T("solver")
sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg"); T("analyse")
sv.psp_set_perturbations(eps, s.d); T("set_pert")
A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
st = torch.empty(len(eps), dtype=torch.int32, device="cuda")
sv.psp_factor_batch(A, tol, st); torch.cuda.synchronize(); T(f"factor {sv.psp_get_last_kernels()}")
Bt = torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda")
sv.psp_solve_batch(Bt); torch.cuda.synchronize(); T(f"solve {sv.psp_get_last_kernels()}")
X = sv.psp_get_solutions(); torch.cuda.synchronize(); T("get")
