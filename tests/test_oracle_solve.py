"""Pins for the oracle's per-lane solves (oracle.c OR1/OR2, oracle/ordering.py).

Pinned against: SPEC worked examples, LAPACK (numpy), exact
rational brute force (Cramer's rule with Leibniz determinants, n <= 5), the
structural definition of fill, and the paper's failure mode."""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import ordering
from psp_inputs import build_system, config


def test_lu_nopivot_spec_examples():
    LU, st = oracle.lu_nopivot(np.eye(2))
    assert st == 0 and np.array_equal(LU, np.eye(2))
    _, st = oracle.lu_nopivot(np.array([[0.0, 1.0], [1.0, 0.0]]), tol=1e-300)
    assert st == 1                                    # ZeroPivot{row 0}
    LU, st = oracle.lu_nopivot(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert st == 0
    assert np.array_equal(np.triu(LU), np.array([[2.0, 1.0], [0.0, 1.5]]))
    assert LU[1, 0] == 0.5


def test_solve_spec_examples():
    for A, b, x in [(np.diag([2.0, 4.0]), [2.0, 4.0], [1.0, 1.0]),
                    (np.array([[2.0, 1.0], [1.0, 2.0]]), [3.0, 3.0], [1.0, 1.0]),
                    (np.eye(3), [1.0, 2.0, 3.0], [1.0, 2.0, 3.0])]:
        LU, st = oracle.lu_nopivot(A)
        assert st == 0
        assert np.array_equal(oracle.lu_solve(LU, np.array(b)), np.array(x))


def test_partial_pivot_vs_lapack():
    rng = np.random.default_rng(7)
    for n in [1, 2, 5, 10, 40]:
        A = rng.normal(size=(n, n))
        b = rng.normal(size=n)
        LU, piv, st = oracle.lu_partial_pivot(A)
        assert st == 0
        x = oracle.lu_pp_solve(LU, piv, b)
        ref = np.linalg.solve(A, b)
        assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref) * np.linalg.cond(A)
    LU, piv, st = oracle.lu_partial_pivot(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert st == 0 and list(piv) == [1, 1]


def _det(M):
    n = len(M)
    tot = Fraction(0)
    for p in itertools.permutations(range(n)):
        sgn = 1
        for i in range(n):
            for j in range(i + 1, n):
                if p[i] > p[j]:
                    sgn = -sgn
        prod = Fraction(sgn)
        for i in range(n):
            prod *= M[i][p[i]]
            if prod == 0:
                break
        tot += prod
    return tot


def cramer(M, b):
    """Exact solution by Cramer's rule (brute force, tiny n)."""
    n = len(M)
    d = _det(M)
    out = []
    for c in range(n):
        Mc = [[b[i] if j == c else M[i][j] for j in range(n)] for i in range(n)]
        out.append(_det(Mc) / d)
    return out


class _Tiny:
    """Minimal system object accepted by oracle.dense_batch."""

    def __init__(self, A, d, b):
        n = A.shape[0]
        rp, ci, v = [0], [], []
        for i in range(n):
            for j in range(n):
                if A[i, j] != 0:
                    ci.append(j)
                    v.append(A[i, j])
            rp.append(len(ci))
        self.n = n
        self.row_ptr = np.array(rp, np.int32)
        self.col_idx = np.array(ci, np.int32)
        self.vals = np.array(v)
        self.d = np.array(d, float)
        self.b = np.array(b, float).reshape(n, -1)


def tiny_zero_diag_system(seed, n=5):
    rng = np.random.default_rng(seed)
    while True:
        A = rng.integers(-3, 4, size=(n, n)).astype(float)
        A[0, 0] = 0.0                   # a leading zero
        A[2, 2] = 0.0
        if abs(np.linalg.det(A)) > 0.5:
            break
    d = rng.choice([-1.0, -0.75, -0.5, 0.5, 0.75, 1.0], size=n)
    b = rng.integers(-4, 5, size=n).astype(float)
    return A, d, b


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("perm_kind", ["natural", "reversed"])
def test_dense_lane_vs_exact_rational(seed, perm_kind):
    A, d, b = tiny_zero_diag_system(seed)
    n = A.shape[0]
    sysm = _Tiny(A, d, b)
    perm = np.arange(n, dtype=np.int32) if perm_kind == "natural" else np.arange(n, dtype=np.int32)[::-1].copy()
    eps = np.array([1 / 16, -1 / 16, 1 / 32, -1 / 32, 0.0])       # dyadic: exact inputs
    X, st = oracle.dense_batch(sysm, perm, eps, tol=0.0)
    for k, e in enumerate(eps):
        M = [[Fraction(A[i, j]) + (Fraction(e) * Fraction(d[i]) if i == j else 0) for j in range(n)]
             for i in range(n)]
        if _det(M) == 0:
            continue
        # leading-minor check: pivot-free elimination in this order is feasible iff all
        # leading principal minors of P M P^T are nonzero
        Mp = [[M[perm[i]][perm[j]] for j in range(n)] for i in range(n)]
        feasible = all(_det([r[:q] for r in Mp[:q]]) != 0 for q in range(1, n + 1))
        if not feasible:
            assert st[k] != 0
            continue
        assert st[k] == 0
        x = np.array([float(v) for v in cramer(M, [Fraction(v) for v in b])])
        assert np.linalg.norm(X[k, 0] - x) <= 1e-12 * np.linalg.norm(x)


def test_or2_equals_or1_bitwise():
    for ci in [0, 1]:
        w = config(ci)
        s = w.system()
        for first in [None, s.slot_p]:
            perm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx, first=first)
            tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
            eps = np.r_[w.eps(), 1e-6, -1e-8]
            X1, st1 = oracle.dense_batch(s, perm, eps, tol)
            X2, st2 = oracle.SparseOracle(s, perm).batch(eps, tol)
            assert np.array_equal(st1, st2)
            ok = st1 == 0
            assert np.array_equal(X1[ok], X2[ok])


def test_leading_zero_fails_unperturbed_and_succeeds_perturbed():
    # "A leading 0 was always encountered on a diagonal" -> pivot-free fails;
    # the perturbed lanes (Alg. 1) succeed.
    s = config(1).system()
    perm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx, first=s.slot_p)
    assert perm[0] == s.slot_p
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    X, st = oracle.SparseOracle(s, perm).batch(np.array([0.0, 2e-3, -2e-3]), tol)
    assert st[0] == 1 and st[1] == 0 and st[2] == 0


def test_listed_convention_negative_control():
    # literal variable order: ~all diagonals structurally zero; pivot-free LU of J + eps D
    # in natural order breaks down (tiny or non-finite pivots) -> status flagged.
    s = config(1).system(convention="listed")
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    perm = np.arange(s.n, dtype=np.int32)
    _, st = oracle.SparseOracle(s, perm).batch(np.array([0.0, 2e-3]), tol)
    assert st[0] != 0


def test_partial_pivot_reference_matches_lapack_on_jacobian():
    s = config(1).system()
    x, st = oracle.reference_solve(s)
    assert st == 0
    ref = np.linalg.solve(s.dense(), s.b[:, 0])
    assert np.linalg.norm(x[0] - ref) <= 1e-10 * np.linalg.norm(ref)


def test_eps_zero_lane_equals_unperturbed_solution():
    # slack convention + min-degree: nonzero leading minors, so eps -> 0 is the plain
    # pivot-free solve, equal to x* up to conditioning-sized rounding.
    s = config(1).system()
    perm = ordering.min_degree_order(s.n, s.row_ptr, s.col_idx)
    X, st = oracle.SparseOracle(s, perm).batch(np.array([0.0]), 0.0)
    xs, _ = oracle.reference_solve(s)
    assert st[0] == 0
    assert np.linalg.norm(X[0, 0] - xs[0]) <= 1e-10 * np.linalg.norm(xs[0])


# ---------------- ordering / symbolic ----------------

def _graph_degrees(adj, alive):
    return {v: len(adj[v]) for v in range(len(adj)) if alive[v]}


@pytest.mark.parametrize("first", [None, "slot"])
def test_min_degree_rule_brute_force(first):
    s = config(0).system()
    f = s.slot_p if first else None
    perm = ordering.min_degree_order(s.n, s.row_ptr, s.col_idx, first=f)
    assert sorted(perm.tolist()) == list(range(s.n))
    adj = ordering.symmetric_adjacency(s.n, s.row_ptr, s.col_idx)
    alive = [True] * s.n
    for step, v in enumerate(perm.tolist()):
        degs = _graph_degrees(adj, alive)
        if not (f is not None and step == 0):
            mn = min(degs.values())
            assert degs[v] == mn and v == min(u for u, dd in degs.items() if dd == mn)
        nb = list(adj[v])
        for a in nb:
            adj[a].discard(v)
            adj[a].update(u for u in nb if u != a)
        adj[v] = set()
        alive[v] = False


def test_min_degree_path_graph_no_fill():
    n = 9
    rp, ci = [0], []
    for i in range(n):
        for j in (i - 1, i + 1):
            if 0 <= j < n:
                ci.append(j)
        rp.append(len(ci))
    rp, ci = np.array(rp, np.int32), np.array(ci, np.int32)
    perm = ordering.min_degree_order(n, rp, ci)
    fcp, fri = ordering.filled_pattern(n, rp, ci, perm)
    assert fcp[-1] == n + 2 * (n - 1)        # tridiagonal: no fill


def test_filled_pattern_equals_numeric_structure():
    # generic values on pattern(A+A^T) (diagonally dominant): the nonzero structure of the
    # dense pivot-free L+U equals the symbolic filled pattern (no accidental cancellation).
    s = config(0).system()
    n = s.n
    rng = np.random.default_rng(3)
    A = np.zeros((n, n))
    for i in range(n):
        for q in range(s.row_ptr[i], s.row_ptr[i + 1]):
            j = s.col_idx[q]
            A[i, j] = rng.normal()
            A[j, i] = rng.normal()
    A += np.diag(np.full(n, 50.0))
    perm = ordering.min_degree_order(n, s.row_ptr, s.col_idx)
    Ap = A[np.ix_(perm, perm)]
    LU, st = oracle.lu_nopivot(Ap)
    assert st == 0
    fcp, fri = ordering.filled_pattern(n, s.row_ptr, s.col_idx, perm)
    sym = np.zeros((n, n), bool)
    for j in range(n):
        sym[fri[fcp[j]:fcp[j + 1]], j] = True
    assert np.array_equal(sym, LU != 0)


@pytest.mark.parametrize("ci", [0, 1, 3])
def test_postorder_is_topological_and_keeps_fill(ci):
    s = config(ci).system()
    p0 = ordering.min_degree_order(s.n, s.row_ptr, s.col_idx)
    p1 = ordering.postorder_big_first(s.n, s.row_ptr, s.col_idx, p0)
    assert sorted(p1.tolist()) == list(range(s.n))
    f0 = ordering.filled_pattern(s.n, s.row_ptr, s.col_idx, p0)
    f1 = ordering.filled_pattern(s.n, s.row_ptr, s.col_idx, p1)
    assert f0[0][-1] == f1[0][-1]
    # etree parent of every column comes after it (postorder is topological)
    fcp, fri = f1
    for j in range(s.n):
        rows = fri[fcp[j]:fcp[j + 1]]
        below = rows[rows > j]
        if len(below):
            assert below.min() > j


def test_growth_pins():
    """Oracle growth g_k = max|U_k| / max|A_k|: a diagonal matrix
    factors to itself (g = 1 exactly, any eps); [[delta, 1], [1, 1]] with delta = 2^-10
    has U = [[delta, 1], [0, 1 - 1/delta]], so g = 1023 exactly at eps = 0; with eps the
    perturbed pivot delta + eps enters both U and A_k."""
    A = np.diag([2.0, -3.0, 0.5, 4.0])
    so = oracle.SparseOracle(_Tiny(A, [1.0, -0.5, 0.25, 1.0], np.ones(4)), np.arange(4, dtype=np.int32))
    assert np.array_equal(so.growth([0.0, 1e-3, -0.25], 1e-300), [1.0, 1.0, 1.0])
    delta = 2.0 ** -10
    A2 = np.array([[delta, 1.0], [1.0, 1.0]])
    so2 = oracle.SparseOracle(_Tiny(A2, [1.0, 0.0], np.ones(2)), np.arange(2, dtype=np.int32))
    g = so2.growth([0.0, 2.0 ** -10], 1e-300)
    assert g[0] == 1023.0
    p = delta + 2.0 ** -10                       # = 2^-9, exact
    assert g[1] == abs(1.0 - 1.0 / p) / 1.0      # |u_22| = 511 > 1 = max|A_k|


def test_power_rho_pins():
    """Oracle rho(A^-1 D) by power iteration: the SPEC's worked values
    (diag(2,4), D = I -> 0.5; [[2,1],[1,2]], D = I -> 1), a diagonal closed form
    max|d_i / a_i|, and the largest |eigenvalue| of A^-1 D from LAPACK's eig on a
    random well-separated system."""
    r, it, conv = oracle.power_rho(_Tiny(np.diag([2.0, 4.0]), [1.0, 1.0], [1.0, 1.0]), [1.0, 1.0])
    assert conv and abs(r - 0.5) < 1e-6
    r, it, conv = oracle.power_rho(_Tiny(np.array([[2.0, 1.0], [1.0, 2.0]]), [1.0, 1.0], [1.0, 1.0]),
                                   [1.0, 0.3])
    assert conv and abs(r - 1.0) < 1e-6
    rng = np.random.default_rng(3)
    a = rng.uniform(1, 3, 40) * rng.choice([-1, 1], 40)
    d = rng.uniform(-1, 1, 40)
    d[7] = 1.0
    a[7] = 0.25   # dominant ratio 4, the next one < 1
    r, it, conv = oracle.power_rho(_Tiny(np.diag(a), d, np.ones(40)), np.ones(40), rtol=1e-12)
    assert conv and abs(r - np.max(np.abs(d / a))) <= 1e-12 * 4
    n = 12
    M = rng.normal(size=(n, n)) + 4 * np.eye(n)
    dd = rng.uniform(0.2, 1.0, n)
    lam = np.max(np.abs(np.linalg.eigvals(np.linalg.solve(M, np.diag(dd)))))
    r, it, conv = oracle.power_rho(_Tiny(M, dd, np.ones(n)), np.ones(n), max_iter=5000, rtol=1e-13)
    assert abs(r - lam) <= 1e-8 * lam


def test_residual_pins():
    """Alg. 1 optional error test: a hand-computed 2x2 case, x = 0 gives ||b||,
    the partial-pivot x* gives a rounding-level residual, and x* + delta e_j gives
    |delta| ||A e_j|| (linearity)."""
    from types import SimpleNamespace
    # A = [[2, 1], [0, 3]], x = [1, 1], b = [1, 1]: A x - b = [2, 2] -> 2 sqrt 2
    t = SimpleNamespace(n=2, row_ptr=np.array([0, 2, 3]), col_idx=np.array([0, 1, 1]),
                        vals=np.array([2.0, 1.0, 3.0]), b=np.ones((2, 1)))
    assert oracle.residual(t, np.ones((1, 1, 2)))[0, 0] == 2.0 * np.sqrt(2.0)
    s = config(1).system()
    n = s.n
    assert oracle.residual(s, np.zeros((1, 1, n)))[0, 0] == np.linalg.norm(s.b[:, 0])
    xs, st = oracle.reference_solve(s)
    assert st == 0
    r0 = oracle.residual(s, xs[None])[0, 0]
    Ad = np.zeros((n, n))
    for i in range(n):
        Ad[i, s.col_idx[s.row_ptr[i]:s.row_ptr[i + 1]]] = s.vals[s.row_ptr[i]:s.row_ptr[i + 1]]
    assert r0 <= 1e-12 * np.linalg.norm(Ad) * np.linalg.norm(xs)
    j, delta = 7, 1e-3
    xp = xs.copy()
    xp[0, j] += delta
    rp = oracle.residual(s, xp[None])[0, 0]
    assert abs(rp - delta * np.linalg.norm(Ad[:, j])) <= 1e-6 * rp
