import sys, json, numpy as np
sys.path.insert(0, '/root/repo')
import oracle
from bench import bench_workload
meta = json.load(open('out/meta.json'))
w = bench_workload(); s = w.system(); eps = w.eps()
n, nnzL, nnzLU = meta['n'], meta['nnzL'], meta['nnzLU']
perm = np.array(meta['perm']); lofs = meta['lofs']; dofs = meta['dofs']; lcol = meta['lcol']
A = s.dense()
for fn in sys.argv[1:]:
    V = np.fromfile(fn).reshape(2, nnzLU, 32)
    bad = 0
    for k in [0, 1, 2, 3, 40, 63]:
        Ak = A + np.diag(eps[k] * s.d)
        Ak = Ak[np.ix_(perm, perm)]
        LU, st = oracle.lu_nopivot(Ak, 0.0)
        v = V[k // 32, :, k % 32]
        for p in range(n):
            if v[nnzL + dofs[p]] != LU[p, p]: bad += 1
            for q, i in enumerate(lcol[p]):
                if v[lofs[p] + q] != LU[i, p]: bad += 1
                if v[nnzL + dofs[p] + 1 + q] != LU[p, i]: bad += 1
    print(fn, "mismatches vs oracle dense LU:", bad)
