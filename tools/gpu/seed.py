"""Diagnose one random-pattern seed: per-path status and solution agreement."""
import os
import sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import oracle
from paper_2311_11833_b200 import psp

seed = int(sys.argv[1])
rng = np.random.default_rng(100 + seed)
n = int(rng.integers(40, 90))
M = (rng.random((n, n)) < 0.05).astype(float)
for hub in rng.choice(n, 3, replace=False):
    M[hub, :] = M[:, hub] = (rng.random(n) < 0.6)
M = np.maximum(M, M.T)
np.fill_diagonal(M, rng.random(n) < 0.8)
vals = rng.normal(size=(n, n)) * M
vals += np.diag(np.where(np.diag(M) > 0, 4.0 * np.sign(rng.normal(size=n)), 0.0))
class _S: pass
s = _S()
rp, ci, v = [0], [], []
for i in range(n):
    for j in range(n):
        if M[i, j] != 0 or i == j:
            ci.append(j); v.append(vals[i, j])
    rp.append(len(ci))
s.n, s.row_ptr, s.col_idx, s.vals = n, np.array(rp, np.int32), np.array(ci, np.int32), np.array(v)
s.d = rng.normal(size=n); s.d /= np.max(np.abs(s.d))
s.b = rng.normal(size=(n, 1))
K = int(rng.integers(5, 150))
eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-4, -1, K)
A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
res = {}
for name, coop, fused in (("batch", 2, False), ("fused", 2, True), ("coop", 1, False)):
    sv = psp.Solver(0)
    sv.psp_set_option("coop", coop)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
    info, perm = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s.d)
    if fused:
        sv.psp_factor_solve_batch(A, b, 1e-300)
    else:
        sv.psp_factor_batch(A, 1e-300)
        sv.psp_solve_batch(b.view(1, -1))
    rc, st = sv.psp_get_lane_status()
    F = np.stack([sv.psp_get_factor(k, info["nnz_LU"]) for k in range(K)])
    res[name] = (sv.psp_get_solutions().cpu().numpy(), st, F)
print("n", n, "K", K, "nnz_LU", info["nnz_LU"], "slots", info["max_live"], "pend", info["factor_pend_smem"],
      "aug", info["aug_ok"], info["aug_pend_smem"])
so = oracle.SparseOracle(s, perm)
Xo, sto = so.batch(eps, 1e-300)
print("oracle failed lanes", np.nonzero(sto)[0][:10])
for name, (X, st, F) in res.items():
    ok = sto == 0
    badst = np.nonzero((st != 0) != (sto != 0))[0]
    badx = [k for k in range(K) if ok[k] and not np.array_equal(X[k], Xo[k])]
    print(name, "status mismatch lanes", badst[:10], "X mismatch lanes", badx[:10])
    if badx:
        k = badx[0]
        fo, sto_k = so.factor(float(eps[k]), 1e-300)
        print("  lane", k, "eps", eps[k], "max rel X diff", np.max(np.abs(X[k] - Xo[k]) / np.maximum(np.abs(Xo[k]), 1e-300)))
for a, bn in (("batch", "fused"), ("batch", "coop")):
    print(a, "vs", bn, "X equal", np.array_equal(res[a][0], res[bn][0], equal_nan=True),
          "F equal", np.array_equal(res[a][2], res[bn][2], equal_nan=True))
Fb, Ff = res["batch"][2], res["fused"][2]
d = np.nonzero(~np.isclose(Fb[0], Ff[0], rtol=0, atol=0) & ~(np.isnan(Fb[0]) & np.isnan(Ff[0])))[0]
print("nnz_L", info["nnz_L"], "first factor mismatches (lane 0):", d[:12], "count", len(d))
# pivot of each L position: columns of the filled pattern (oracle's symbolic, same perm)
fcp, fri = so.fcp, so.fri
col_of = []
for j in range(n):
    for q in range(fcp[j], fcp[j + 1]):
        if fri[q] > j:
            col_of.append(j)
cnt = [sum(1 for q in range(fcp[j], fcp[j + 1]) if fri[q] > j) for j in range(n)]
if len(d) and d[0] < info["nnz_L"]:
    p = col_of[d[0]]
    print("first bad L entry belongs to pivot", p, "c =", cnt[p], "prev pivots c:", cnt[max(0, p - 3):p])
print("c distribution (max, #>11):", max(cnt), sum(1 for c in cnt if c > 11))
print("F batch lane0[:6]", Fb[0][:6])
print("F fused lane0[:6]", Ff[0][:6])
print("fused X lane0[:4]", res["fused"][0][0][0][:4], "oracle", Xo[0][0][:4])
torch.cuda.synchronize()
print("cuda ok")
print("L[0:8] batch", Fb[0][:8])
print("L[0:8] fused", Ff[0][:8])
print("lane1 batch", Fb[1][:4], "fused", Ff[1][:4])
