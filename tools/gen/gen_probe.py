import sys, time, numpy as np
sys.path.insert(0,'/root/repo')
from oracle import ordering
from psp_inputs import config
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
mk = '--markstein' in sys.argv
outdir = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith('--') else '/tmp/gen'
s = config(ci).system()
n = s.n
perm = ordering.elimination_order(n, s.row_ptr, s.col_idx)
fcp, fri = ordering.filled_pattern(n, s.row_ptr, s.col_idx, perm)
inv = np.empty(n, int); inv[perm] = np.arange(n)
lcol = [[int(r) for r in fri[fcp[j]:fcp[j+1]] if r > j] for j in range(n)]
# A lookup
amap = {}
for i in range(n):
    for q in range(s.row_ptr[i], s.row_ptr[i+1]):
        amap[(int(inv[i]), int(inv[s.col_idx[q]]))] = q
lofs = np.concatenate([[0], np.cumsum([len(l) for l in lcol])])
dofs = np.concatenate([[0], np.cumsum([1 + len(l) for l in lcol])])
nnzL = int(lofs[-1])
nnzLU = nnzL + int(dofs[-1])
out = []
w = out.append
w('__device__ __forceinline__ double mdiv(double a, double b, double y) { double q = __dmul_rn(a, y); double r = __fma_rn(-b, q, a); double q1 = __fma_rn(r, y, q); double aq = fabs(q); if (!(aq > 0x1p-960 && aq < 0x1p960) || !(fabs(a) > 0x1p-960)) q1 = __ddiv_rn(a, b); return q1; }')
w('extern "C" __global__ void __launch_bounds__(128) factor_gen(const double* __restrict__ A, const double* __restrict__ eps, const double* __restrict__ dp, double tol, double* __restrict__ V, int* __restrict__ status, int K_pad) {')
w(' const int lane = blockIdx.x * blockDim.x + threadIdx.x; if (lane >= K_pad) return;')
w(' double* o = V + (size_t)(lane >> 5) * %d * 32 + (lane & 31);' % nnzLU)
w(' const double e = eps[lane]; int st = 0;')
pending = {}   # (i,j) -> var name
cnt = [0]
def val(i, j):
    if (i, j) in pending:
        return pending.pop((i, j))
    q = amap.get((i, j))
    return 'A[%d]' % q if q is not None else '0.0'
for p in range(n):
    L = lcol[p]; c = len(L)
    if (p, p) in pending:
        pv = pending.pop((p, p))
    else:
        q = amap.get((p, p))
        pv = '__dadd_rn(%s, __dmul_rn(e, dp[%d]))' % ('A[%d]' % q if q is not None else '0.0', p)
    w(' { const double pv = %s;' % pv)
    if mk: w('   const double rp = __drcp_rn(pv);')
    w('   if (st == 0 && (!(fabs(pv) > tol) || !isfinite(pv))) st = %d;' % (p + 1))
    w('   o[%d] = pv;' % ((nnzL + dofs[p]) * 32))
    for k, i in enumerate(L):
        if mk:
            w('   const double l%d = mdiv(%s, pv, rp); o[%d] = l%d;' % (k, val(i, p), (lofs[p] + k) * 32, k))
        else:
            w('   const double l%d = __ddiv_rn(%s, pv); o[%d] = l%d;' % (k, val(i, p), (lofs[p] + k) * 32, k))
    for k, j in enumerate(L):
        w('   const double u%d = %s; o[%d] = u%d;' % (k, val(p, j), (nnzL + dofs[p] + 1 + k) * 32, k))
    for a, i in enumerate(L):
        for b, j in enumerate(L):
            if (i, j) in pending:
                src = pending.pop((i, j))
                name = src
                w('   %s = __fma_rn(-l%d, u%d, %s);' % (name, a, b, name))
            else:
                if (i, j) == (i, i) or i == j:
                    q = amap.get((i, i))
                    init = '__dadd_rn(%s, __dmul_rn(e, dp[%d]))' % ('A[%d]' % q if q is not None else '0.0', i)
                else:
                    q = amap.get((i, j))
                    init = 'A[%d]' % q if q is not None else '0.0'
                name = 'v%d' % cnt[0]; cnt[0] += 1
                # declare at function scope: use outer declaration list
                decls.append(name) if False else None
                w('   %s = __fma_rn(-l%d, u%d, %s);' % (name, a, b, init))
            pending[(i, j)] = name
    w(' }')
w(' status[lane] = st;')
w('}')
body = "\n".join(out)
decl = ' double ' + ', '.join('v%d' % k for k in range(cnt[0])) + ';'
body = body.replace(' const double e = eps[lane]; int st = 0;', ' const double e = eps[lane]; int st = 0;\n' + decl, 1)
import os, json
os.makedirs(outdir, exist_ok=True)
open(os.path.join(outdir, 'factor_gen%s.cu' % ('_mk' if mk else '')), 'w').write(body)
json.dump(dict(n=n, nnzL=nnzL, nnzLU=nnzLU, lofs=[int(x) for x in lofs], dofs=[int(x) for x in dofs], perm=[int(x) for x in perm], lcol=lcol), open(os.path.join(outdir, 'meta.json'), 'w'))
print("vars", cnt[0], "lines", len(out), "nnzLU", nnzLU)
