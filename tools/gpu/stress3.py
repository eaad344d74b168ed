"""Handle reuse stress: one handle, repeated re-analysis (random patterns), new
perturbation sets, factor/solve/recover in both paths; bitwise against the oracle."""
import os
import sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tools", "gpu"))
import numpy as np
import torch
import oracle
from paper_2311_11833_b200 import psp
from stress2 import system  # noqa: E402  (reuses the generator; stress2 runs nothing on import)

bad = 0
sv = psp.Solver(0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for t in range(N):
    rng = np.random.default_rng(90000 + t)
    s = system(rng)
    s.b = rng.normal(size=(s.n, 1))
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
    info, perm = sv.psp_get_symbolic_info()
    for rep in range(2):
        K = int(rng.integers(1, 3000))
        eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-4, -1, K)
        sv.psp_set_perturbations(eps, s.d)
        A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
        b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
        if rep == 0:
            sv.psp_factor_solve_batch(A, b, 1e-300)
        else:
            sv.psp_factor_batch(A, 1e-300)
            sv.psp_solve_batch(b.view(1, -1))
        X = sv.psp_get_solutions().cpu().numpy()
        rc, st = sv.psp_get_lane_status()
        idx = sorted(set(rng.integers(0, K, 12).tolist() + [0, K - 1]))
        Xo, sto = oracle.SparseOracle(s, perm).batch(eps[idx], 1e-300)
        ok = sto == 0
        if not (np.array_equal(st[idx] != 0, sto != 0) and np.array_equal(X[idx][ok], Xo[ok])):
            bad += 1
            print(t, rep, "FAILED n", s.n, "K", K, flush=True)
print("failures", bad, "of", 2 * N)
