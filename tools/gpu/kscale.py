import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from paper_2311_11833_b200 import psp
from psp_inputs import config
s = config(1).system()
tol = 1e-14
so = None
for GJ in (sys.argv[1] if len(sys.argv) > 1 else "1:1").split(","):
    G, J, P, T = (int(v) for v in (GJ + ":1:1:0").split(":")[:4])
    for K in (32, 33, 64, 96, 160, 1024, 8192):
        rng = np.random.default_rng(K)
        eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-4, -2, K)
        sv = psp.Solver(0); sv.psp_set_option("factor_groups", G); sv.psp_set_option("factor_lanes", J); sv.psp_set_option("factor_slab_warps", P); sv.psp_set_option("factor_tmem", T)
        sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
        info, perm = sv.psp_get_symbolic_info()
        sv.psp_set_perturbations(eps, s.d)
        sv.psp_factor_batch(torch.tensor(s.vals, dtype=torch.float64, device="cuda"), tol)
        sv.psp_solve_batch(torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda"))
        X = sv.psp_get_solutions().cpu().numpy()
        if so is None:
            so = oracle.SparseOracle(s, perm)
        idx = sorted(set([0, 1, 31, K - 1, K // 2] + list(range(0, K, max(1, K // 16)))))
        idx = [i for i in idx if i < K]
        Xo, sto = so.batch(eps[idx], tol)
        Fg = np.stack([sv.psp_get_factor(k, info["nnz_LU"]) for k in idx[:3]])
        bad = [i for j, i in enumerate(idx) if not np.array_equal(X[i], Xo[j])]
        print(f"G={G} J={J} P={P} T={info['factor_pend_smem']} K={K} warps/cta={info['factor_warps_per_cta']} lanes checked {len(idx)} mismatching {bad[:8]}", flush=True)
        sv.close()
