"""Randomized stress over options: random patterns (hubs, zero diagonals), orderings,
R, forced warp organisations (G, J, P), TMEM on/off, coop on/off, fused or not; every
configuration bitwise against the oracle."""
import os
import sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import oracle
from paper_2311_11833_b200 import psp


def system(rng):
    n = int(rng.integers(20, int(os.environ.get("PSP_NMAX", "90"))))
    M = (rng.random((n, n)) < rng.uniform(0.02, 0.08)).astype(float)
    for hub in rng.choice(n, int(rng.integers(0, 4)), replace=False):
        M[hub, :] = M[:, hub] = (rng.random(n) < 0.5)
    M = np.maximum(M, M.T)
    np.fill_diagonal(M, rng.random(n) < 0.85)
    vals = rng.normal(size=(n, n)) * M
    vals += np.diag(np.where(np.diag(M) > 0, 4.0 * np.sign(rng.normal(size=n)), 0.0))

    class S:
        pass
    s = S()
    rp, ci, v = [0], [], []
    for i in range(n):
        for j in range(n):
            if M[i, j] != 0 or i == j:
                ci.append(j)
                v.append(vals[i, j])
        rp.append(len(ci))
    s.n, s.row_ptr, s.col_idx, s.vals = n, np.array(rp, np.int32), np.array(ci, np.int32), np.array(v)
    s.d = rng.normal(size=n)
    s.d /= np.max(np.abs(s.d))
    return s


def main():
    bad = 0
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    for t in range(N):
        rng = np.random.default_rng(int(os.environ.get("PSP_SEED0", "20000")) + t)
        s = system(rng)
        R = int(rng.choice([1, 1, 3]))
        s.b = rng.normal(size=(s.n, R))
        K = int(rng.integers(1, 300))
        eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-4, -1, K)
        if rng.random() < 0.3:
            eps[rng.random(K) < 0.1] = 0.0   # unperturbed lanes: zero diagonals fail them
        tol = 0.0 if rng.random() < 0.5 else 1e-300
        order = str(rng.choice(["mindeg", "natural"]))
        G = int(rng.choice([0, 0, 1, 2, 4]))
        J = int(rng.choice([0, 1, 2])) if G in (2, 4) else 0
        T = int(rng.choice([0, 2]))
        C = int(rng.choice([0, 1, 2]))
        fused = R == 1 and bool(rng.integers(0, 2))
        try:
            sv = psp.Solver(0)
            for k, v in (("factor_groups", G), ("factor_lanes", J), ("factor_tmem", T), ("coop", C)):
                sv.psp_set_option(k, v)
            sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, order)
            info, perm = sv.psp_get_symbolic_info()
            sv.psp_set_perturbations(eps, s.d)
            A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
            B = torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda")
            if fused:
                sv.psp_factor_solve_batch(A, B[0].contiguous(), tol)
            else:
                sv.psp_factor_batch(A, tol)
                sv.psp_solve_batch(B)
            # random weights: ladder-like contiguous runs or arbitrary lane subsets
            Wn = int(rng.integers(1, 6))
            Wm = np.zeros((Wn, K))
            for w in range(Wn):
                if rng.random() < 0.5:
                    k0 = int(rng.integers(0, K)); ln = int(rng.integers(1, 9))
                    Wm[w, k0:k0 + ln] = rng.normal(size=len(range(k0, min(K, k0 + ln))))
                else:
                    Wm[w, rng.random(K) < 0.2] = 1.0
                    Wm[w] *= rng.normal(size=K)
            ptr, lane, val = [0], [], []
            for w in range(Wn):
                nz = np.nonzero(Wm[w])[0]
                lane += list(nz); val += list(Wm[w, nz]); ptr.append(len(lane))
            sv.psp_set_weights(np.array(ptr, np.int32), np.array(lane, np.int32), np.array(val))
            xh = sv.psp_recover().cpu().numpy()
            rc, st = sv.psp_get_lane_status()
            X = sv.psp_get_solutions().cpu().numpy()
            sv.close()
        except psp.PSPError as e:
            print(t, "config refused:", str(e)[:100], flush=True)
            continue
        otol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals) if tol == 0.0 else tol
        Xo, sto = oracle.SparseOracle(s, perm).batch(eps, otol)
        ok = sto == 0
        good = np.array_equal(st != 0, sto != 0) and np.array_equal(X[ok], Xo[ok])
        rows_ok = [w for w in range(Wn) if np.all(ok[np.nonzero(Wm[w])[0]])]
        if rows_ok:
            xo = oracle.combine(Wm[rows_ok], np.nan_to_num(Xo))
            good = good and np.array_equal(xh[rows_ok], xo)
        if not good:
            bad += 1
            print(t, f"FAILED n={s.n} K={K} R={R} order={order} G={G} J={J} T={T} C={C} fused={fused} "
                  f"G*={info['factor_groups']} J*={info['factor_lanes_per_thread']} pend={info['factor_pend_smem']} "
                  f"aug={info['aug_ok']}", flush=True)
    print("failures", bad, "of", N)


if __name__ == "__main__":
    main()
