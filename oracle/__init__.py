"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU FP64 implementation of what the hot path of
arXiv 2311.11833 computes (Alg. 1):

  1. perturb A by +/- alpha*eps*D for each lane (Eqs. (5)-(6));
  2. pivot-free ("static pivoting") LU + forward/back substitution per lane
     (oracle.c: dense OR1, and sparse OR2 for sizes where O(n^3) is infeasible);
  3-4. combine the lanes with the weights of Remark 2 / Eq. (13) (weights.py,
     exact rationals; oracle.c: oracle_combine);
  5. optional error test: residual ||A x - b|| (residual(), row by row) and the
     partial-pivot x* (oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  It shares no code with the CUDA path
(paper_2311_11833_b200/) and never imports it; it takes its inputs only from
psp_inputs/ (seeded generators, no method arithmetic).

Parity pins: see tests/test_oracle_*.py (every function here is pinned; none is
"parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import ordering, weights  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc, -O2, -ffp-contract=off, OpenMP over lanes)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fopenmp", "-fPIC", "-shared", "-o", tmp, src, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        L.oracle_lu_nopivot.argtypes = [I, P, D]
        L.oracle_lu_solve.argtypes = [I, P, P]
        L.oracle_lu_partial_pivot.argtypes = [I, P, P]
        L.oracle_lu_pp_solve.argtypes = [I, P, P, P]
        L.oracle_dense_lane.argtypes = [I, P, P, P, P, P, D, I, P, D, P]
        L.oracle_dense_batch.argtypes = [I, P, P, P, P, P, I, P, I, P, D, P, P]
        L.oracle_dense_batch.restype = None
        L.oracle_reference_solve.argtypes = [I, P, P, P, I, P, P]
        L.oracle_sparse_lu.argtypes = [I, P, P, P, P, P, P, D, D, P]
        L.oracle_sparse_solve.argtypes = [I, P, P, P, P, P, P]
        L.oracle_sparse_batch.argtypes = [I, P, P, P, P, P, P, P, I, P, I, P, D, P, P]
        L.oracle_sparse_batch.restype = None
        L.oracle_combine.argtypes = [I, I, I, I, P, P, P]
        L.oracle_combine.restype = None
        L.oracle_num_threads.restype = I
        L.oracle_set_num_threads.argtypes = [I]
        L.oracle_residual_fma.argtypes = [I, P, P, P, P, P, P]
        L.oracle_residual_fma.restype = None
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_num_threads(t: int) -> None:
    lib().oracle_set_num_threads(int(t))


def lu_nopivot(A, tol=0.0):
    """Dense pivot-free LU of a copy of A -> (LU, status)."""
    LU = _c(A, np.float64).copy()
    st = lib().oracle_lu_nopivot(LU.shape[0], _p(LU), float(tol))
    return LU, st


def lu_solve(LU, b):
    y = _c(b, np.float64).copy()
    lib().oracle_lu_solve(LU.shape[0], _p(_c(LU, np.float64)), _p(y))
    return y


def lu_partial_pivot(A):
    LU = _c(A, np.float64).copy()
    piv = np.zeros(LU.shape[0], dtype=np.int32)
    st = lib().oracle_lu_partial_pivot(LU.shape[0], _p(LU), _p(piv))
    return LU, piv, st


def lu_pp_solve(LU, piv, b):
    y = _c(b, np.float64).copy()
    lib().oracle_lu_pp_solve(LU.shape[0], _p(_c(LU, np.float64)), _p(_c(piv, np.int32)), _p(y))
    return y


def power_rho(sysm, v0, max_iter=500, rtol=1e-6):
    """rho(A^-1 D) by power iteration on v -> A^-1 (D v) with A^-1 applied through a
    partial-pivot LU (Eq. (4)): v_0 = v0 / ||v0||_2,
    rho_t = ||A^-1 D v_t||_2, v_{t+1} = A^-1 D v_t / rho_t, stop when
    |rho_t - rho_{t-1}| < rtol * rho_t.  Returns (rho, iterations, converged)."""
    n = sysm.n
    A = np.zeros((n, n))
    for i in range(n):
        for q in range(sysm.row_ptr[i], sysm.row_ptr[i + 1]):
            A[i, sysm.col_idx[q]] += sysm.vals[q]
    LU, piv, st = lu_partial_pivot(A)
    if st:
        raise ValueError("singular A")
    d = np.asarray(sysm.d, dtype=np.float64)
    v = np.asarray(v0, dtype=np.float64) / np.linalg.norm(v0)
    rho, it = 0.0, 0
    for it in range(1, max_iter + 1):
        u = lu_pp_solve(LU, piv, d * v)
        prev, rho = rho, float(np.linalg.norm(u))
        if rho == 0.0:
            return rho, it, False
        v = u / rho
        if it > 1 and abs(rho - prev) < rtol * rho:
            return rho, it, True
    return rho, max_iter, False


def default_tol(n, row_ptr, col_idx, vals):
    """zero_tol = n * u * ||A||_1 of the unperturbed A (reading R10)."""
    cs = np.zeros(n)
    np.add.at(cs, np.asarray(col_idx), np.abs(np.asarray(vals)))
    return n * np.finfo(np.float64).eps * float(cs.max())


def dense_batch(sysm, perm, eps, tol, B=None):
    """OR1 over all lanes: returns X [K, R, n] (original ordering) and status [K]."""
    n = sysm.n
    eps = _c(eps, np.float64)
    B = sysm.b if B is None else B
    R = B.shape[1]
    Bc = _c(B.T, np.float64)  # R x n contiguous == n x R column-major
    X = np.empty((len(eps), R, n))
    st = np.zeros(len(eps), dtype=np.int32)
    lib().oracle_dense_batch(n, _p(_c(sysm.row_ptr, np.int32)), _p(_c(sysm.col_idx, np.int32)),
                             _p(_c(sysm.vals, np.float64)), _p(_c(perm, np.int32)),
                             _p(_c(sysm.d, np.float64)), len(eps), _p(eps), R, _p(Bc),
                             float(tol), _p(X), _p(st))
    return X, st


def dense_D_batch(A, Dm, perm, eps, tol, B):
    """OR1 with a general (dense, non-diagonal) perturbation matrix D (
    the footnote at P:L72 and P:L314 "all entries of the perturbation matrix ... normally
    distributed"): per lane k, A_k = P (A + eps_k D) P^T entry by entry (one product, one
    sum: a_ij + (eps_k * D_ij)), then the same pivot-free elimination and substitutions as
    dense_batch (lu_nopivot, lu_solve).  A, Dm: n x n dense (original ordering); B: n x R.
    Returns X [K, R, n] (original ordering) and status [K] (0, or 1 + first failing
    pivot position; a failed lane's X is NaN)."""
    A = np.asarray(A, dtype=np.float64)
    Dm = np.asarray(Dm, dtype=np.float64)
    perm = np.asarray(perm, dtype=np.int64)
    B = np.asarray(B, dtype=np.float64).reshape(A.shape[0], -1)
    n, R = A.shape[0], B.shape[1]
    eps = np.asarray(eps, dtype=np.float64)
    X = np.full((len(eps), R, n), np.nan)
    st = np.zeros(len(eps), dtype=np.int32)
    for k, e in enumerate(eps):
        Ak = A + e * Dm                        # elementwise: a_ij + (e * D_ij), two roundings
        LU, st[k] = lu_nopivot(Ak[np.ix_(perm, perm)], tol)
        if st[k]:
            continue
        for r in range(R):
            y = lu_solve(LU, B[perm, r])
            X[k, r, perm] = y
    return X, st


class SparseOracle:
    """OR2: the oracle's own symbolic (ordering.filled_pattern) + sparse numeric."""

    def __init__(self, sysm, perm):
        n = sysm.n
        self.n, self.perm = n, _c(perm, np.int32)
        self.fcp, self.fri = ordering.filled_pattern(n, sysm.row_ptr, sysm.col_idx, perm)
        self.acp, self.ari, self.av = ordering.permuted_csc(n, sysm.row_ptr, sysm.col_idx,
                                                            sysm.vals, perm)
        self.dp = _c(np.asarray(sysm.d)[self.perm], np.float64)
        self.b = sysm.b

    @property
    def nnz_lu(self):
        return int(self.fcp[-1])

    def batch(self, eps, tol, B=None):
        eps = _c(eps, np.float64)
        B = self.b if B is None else B
        R = B.shape[1]
        Bc = _c(B.T, np.float64)
        X = np.empty((len(eps), R, self.n))
        st = np.zeros(len(eps), dtype=np.int32)
        lib().oracle_sparse_batch(self.n, _p(self.acp), _p(self.ari), _p(self.av), _p(self.fcp),
                                  _p(self.fri), _p(self.dp), _p(self.perm), len(eps), _p(eps), R,
                                  _p(Bc), float(tol), _p(X), _p(st))
        return X, st

    def growth(self, eps, tol):
        """Per-lane growth g_k = max|U_k| / max|A_k|: max over the
        lane's filled U (pivots included) over max over A_k = A + eps_k D (diagonal
        a_ii + (eps_k d_i), two roundings as in the factorisation).  NaN for a lane
        whose pivot-free factorisation fails (the oracle stops at the failing pivot)."""
        n = self.n
        eps = np.asarray(eps, dtype=np.float64)
        g = np.full(len(eps), np.nan)
        upper = np.zeros(self.nnz_lu, dtype=bool)
        for j in range(n):
            upper[self.fcp[j]:self.fcp[j + 1]] = np.asarray(self.fri[self.fcp[j]:self.fcp[j + 1]]) <= j
        for k, e in enumerate(eps):
            fv, st = self.factor(float(e), tol)
            if st:
                continue
            umax = float(np.max(np.abs(fv[: self.nnz_lu][upper])))
            amax = 0.0
            for j in range(n):
                has_diag = False
                for q in range(self.acp[j], self.acp[j + 1]):
                    v = float(self.av[q])
                    if self.ari[q] == j:
                        v = v + float(np.float64(e) * self.dp[j])
                        has_diag = True
                    amax = max(amax, abs(v))
                if not has_diag:
                    amax = max(amax, abs(float(np.float64(e) * self.dp[j])))
            g[k] = umax / amax
        return g

    def factor(self, eps, tol):
        fv = np.empty(max(self.nnz_lu, 1))
        st = lib().oracle_sparse_lu(self.n, _p(self.acp), _p(self.ari), _p(self.av), _p(self.fcp),
                                    _p(self.fri), _p(self.dp), float(eps), float(tol), _p(fv))
        return fv, st


def reference_solve(sysm, B=None):
    """x* = A^{-1} b by partial-pivot GE (the unperturbed system)."""
    B = sysm.b if B is None else B
    R = B.shape[1]
    Bc = _c(B.T, np.float64)
    X = np.empty((R, sysm.n))
    st = lib().oracle_reference_solve(sysm.n, _p(_c(sysm.row_ptr, np.int32)),
                                      _p(_c(sysm.col_idx, np.int32)), _p(_c(sysm.vals, np.float64)),
                                      R, _p(Bc), _p(X))
    return X, st


def _dense(sysm):
    """A as a dense n x n array (CSR entries summed in place)."""
    n = sysm.n
    A = np.zeros((n, n))
    for i in range(n):
        for q in range(sysm.row_ptr[i], sysm.row_ptr[i + 1]):
            A[i, sysm.col_idx[q]] += sysm.vals[q]
    return A


def pivoted_lanes(sysm, eps, B=None):
    """x_k^piv = (A + eps_k D)^{-1} b by partial-pivot GE for every lane (SURVEY §8(c)
    step 5: the floor of tolerance policy 3).  -> [K, R, n]."""
    B = sysm.b if B is None else B
    A = _dense(sysm)
    d = np.asarray(sysm.d, dtype=np.float64)
    out = np.empty((len(eps), B.shape[1], sysm.n))
    for k, e in enumerate(eps):
        LU, piv, st = lu_partial_pivot(A + float(e) * np.diag(d))
        if st:
            raise ValueError(f"lane {k}: singular perturbed matrix")
        for r in range(B.shape[1]):
            out[k, r] = lu_pp_solve(LU, piv, B[:, r])
    return out


def predicted_error(sysm, mags, B=None, Dm=None):
    """Theorem 1's truncation error with its constant, exactly: the identity (I3) of
    SURVEY §8(c) (Lagrange interpolation of t -> (I - t M^2)^{-1} x* at the nodes
    t_j = s_j^2, evaluated at t = 0; Remark 2's beta are that Lagrange basis, P:L197-203;
    Examples 1-2 are its leading terms):

        x* - x_hat* = (-1)^m  prod_j [ t_j M^2 (I - t_j M^2)^{-1} ]  x*,   M = A^{-1} D,

    for one ladder of m magnitudes s_j (lanes +-s_j, weights beta_j / 2).  Every operator
    is applied through partial-pivot factorisations (lu_partial_pivot):
      M v = A^{-1} (D v);
      (I - t M^2)^{-1} v = 1/2 [(A + s D)^{-1} + (A - s D)^{-1}] (A v)   (the pair average
        of Eq. (avg_hats), since (I + s M)^{-1} = (A + s D)^{-1} A).
    The factors commute (functions of M^2); each step applies t_j M^2 (I - t_j M^2)^{-1}
    so that neither prod t_j nor M^{2m} is formed on its own (no under/overflow for long
    ladders).  Dm: a dense n x n perturbation matrix in place of diag(sysm.d) (the
    identity holds for any D, SURVEY §8(c) "Any A, D").  Returns e_pred [R, n]
    (original ordering)."""
    B = sysm.b if B is None else B
    A = _dense(sysm)
    Dm = np.diag(np.asarray(sysm.d, dtype=np.float64)) if Dm is None else np.asarray(Dm, np.float64)
    LU, piv, st = lu_partial_pivot(A)
    if st:
        raise ValueError("singular A")

    def M(v):
        return lu_pp_solve(LU, piv, Dm @ v)

    pairs = []
    for s in mags:
        fp = lu_partial_pivot(A + float(s) * Dm)
        fm = lu_partial_pivot(A - float(s) * Dm)
        if fp[2] or fm[2]:
            raise ValueError(f"singular A +- {s} D")
        pairs.append((float(s), fp, fm))
    out = np.empty((B.shape[1], sysm.n))
    for r in range(B.shape[1]):
        v = lu_pp_solve(LU, piv, B[:, r])          # x*
        for s, fp, fm in pairs:
            Av = A @ v
            u = 0.5 * lu_pp_solve(fp[0], fp[1], Av) + 0.5 * lu_pp_solve(fm[0], fm[1], Av)
            v = (s * s) * M(M(u))
        out[r] = (-1.0) ** len(mags) * v
    return out


def residual_fma(sysm, x, b):
    """r = b - A x row by row, one fma per CSR entry in order (oracle.c) -> [n]."""
    r = np.empty(sysm.n)
    lib().oracle_residual_fma(sysm.n, _p(_c(sysm.row_ptr, np.int32)), _p(_c(sysm.col_idx, np.int32)),
                              _p(_c(sysm.vals, np.float64)), _p(_c(x, np.float64)), _p(_c(b, np.float64)),
                              _p(r))
    return r


def refine(sysm, perm, eps, tol, iters, b=None):
    """Iterative-refinement baseline: static pivoting by a
    perturbation plus fixed-precision iterative refinement against the UNPERTURBED A, per
    lane k, with F_k = P (A + eps_k D) P^T factored without pivoting (lu_nopivot):
        x^0 = F_k^{-1} b;   x^i = x^{i-1} + F_k^{-1} (b - A x^{i-1})   (i = 1..iters),
    the residual by residual_fma, the correction by lu_solve, the update one rounded add.
    In exact arithmetic e^i = x* - x^i = (I - F^{-1} A) e^{i-1} = eps_k M_k e^{i-1} and
    e^0 = eps_k M_k x*, so e^i = (eps_k M_k)^{i+1} x* with M_k = (A + eps_k D)^{-1} D.  Returns X [iters + 1, K, n] (original ordering; NaN
    for a failed lane) and status [K]."""
    b = sysm.b[:, 0] if b is None else np.asarray(b, dtype=np.float64)
    A = _dense(sysm)
    d = np.asarray(sysm.d, dtype=np.float64)
    perm = np.asarray(perm, dtype=np.int64)
    eps = np.asarray(eps, dtype=np.float64)
    X = np.full((iters + 1, len(eps), sysm.n), np.nan)
    st = np.zeros(len(eps), dtype=np.int32)
    for k, e in enumerate(eps):
        Ak = A.copy()
        Ak[np.diag_indices(sysm.n)] = np.diag(A) + e * d          # a_ii + (eps d_i)
        LU, st[k] = lu_nopivot(Ak[np.ix_(perm, perm)], tol)
        if st[k]:
            continue

        def solve(rhs):
            out = np.empty(sysm.n)
            out[perm] = lu_solve(LU, rhs[perm])
            return out

        x = solve(b)
        X[0, k] = x
        for i in range(1, iters + 1):
            x = x + solve(residual_fma(sysm, x, b))
            X[i, k] = x
    return X, st


def residual(sysm, X, B=None):
    """Alg. 1's optional error test: ||A x - b||_2 for every
    x = X[w, r] ([W, R, n], original ordering) against b = B[:, r] (default sysm.b):
    the definition written out row by row over the CSR entries.  -> [W, R]."""
    B = sysm.b if B is None else B
    X = np.asarray(X, dtype=np.float64)
    W, R, n = X.shape
    out = np.empty((W, R))
    for w in range(W):
        for r in range(R):
            t = np.empty(n)
            for i in range(n):
                q0, q1 = sysm.row_ptr[i], sysm.row_ptr[i + 1]
                t[i] = np.dot(sysm.vals[q0:q1], X[w, r, sysm.col_idx[q0:q1]]) - B[i, r]
            out[w, r] = np.linalg.norm(t)
    return out


def combine(weights_WK, X):
    """x_hat[w] = sum_k W[w,k] x_k (ascending k, fma) -> [W, R, n]."""
    Wm = _c(weights_WK, np.float64)
    X = _c(X, np.float64)
    K, R, n = X.shape
    out = np.empty((Wm.shape[0], R, n))
    lib().oracle_combine(K, R, n, Wm.shape[0], _p(Wm), _p(X), _p(out))
    return out


def ladder_weight_matrix(ladders):
    """W x K dense weights for a list of ladders laid out consecutively in lane
    order (ladder g occupies lanes [2*sum_{h<g} m_h, ...)); one recovered solution
    per ladder, weights beta_j/2 per sign (weights.lane_weights)."""
    K = 2 * sum(len(l) for l in ladders)
    Wm = np.zeros((len(ladders), K))
    k0 = 0
    for g, mags in enumerate(ladders):
        lw = weights.lane_weights(mags)
        Wm[g, k0:k0 + len(lw)] = lw
        k0 += len(lw)
    return Wm
