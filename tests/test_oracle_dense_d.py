"""Pins for the oracle's general-D path (a dense, non-diagonal
perturbation matrix D, the footnote at P:L72 and P:L314's "all entries of the
perturbation matrix ... normally distributed"):

  * oracle.dense_D_batch per lane against exact rational solves (Cramer) of
    P (A + eps_k D) P^T on zero-diagonal 5x5 systems with a dense dyadic D, and its
    status against the exact leading-minor feasibility criterion;
  * with D = diag(d) it is bit-for-bit oracle.dense_batch (a special case that reduces
    to the already pinned routine);
  * oracle.predicted_error(..., Dm=D) against the exact identity (I3) built in rationals
    with M = A^{-1} D formed by Cramer's rule for a dense D, and against the rational
    recovery x* - x_hat* itself (Theorem 1, with its constant)."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import weights
from test_oracle_method import _matvec
from test_oracle_solve import _Tiny, _det, cramer, tiny_zero_diag_system


def _dense_dyadic_D(seed, n=5):
    rng = np.random.default_rng(100 + seed)
    D = rng.choice([-1.0, -0.5, -0.25, 0.0, 0.25, 0.5, 1.0], size=(n, n))
    D[0, 0] = 1.0                          # the leading zero of A gets a perturbation
    return D


def _solve_D(Af, Df, bf, s):
    n = len(Af)
    return cramer([[Af[i][j] + s * Df[i][j] for j in range(n)] for i in range(n)], bf)


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("perm_kind", ["natural", "reversed"])
def test_dense_D_lane_vs_exact_rational(seed, perm_kind):
    A, _, b = tiny_zero_diag_system(seed)
    n = A.shape[0]
    D = _dense_dyadic_D(seed)
    perm = np.arange(n) if perm_kind == "natural" else np.arange(n)[::-1].copy()
    eps = np.array([1 / 16, -1 / 16, 1 / 32, -1 / 32, 0.0])
    X, st = oracle.dense_D_batch(A, D, perm, eps, 0.0, b)
    n_ok = 0
    for k, e in enumerate(eps):
        M = [[Fraction(A[i, j]) + Fraction(e) * Fraction(D[i, j]) for j in range(n)] for i in range(n)]
        Mp = [[M[perm[i]][perm[j]] for j in range(n)] for i in range(n)]
        feasible = all(_det([r[:q] for r in Mp[:q]]) != 0 for q in range(1, n + 1))
        if not feasible:
            assert st[k] != 0
            continue
        assert st[k] == 0
        n_ok += 1
        x = np.array([float(v) for v in cramer(M, [Fraction(v) for v in b])])
        assert np.linalg.norm(X[k, 0] - x) <= 1e-12 * np.linalg.norm(x)
    assert n_ok >= 4                       # the perturbed lanes are feasible


def test_dense_D_unperturbed_zero_diag_fails_at_first_pivot():
    A, _, b = tiny_zero_diag_system(0)
    D = _dense_dyadic_D(0)
    X, st = oracle.dense_D_batch(A, D, np.arange(5), np.array([0.0]), 0.0, b)
    assert st[0] == 1 and np.isnan(X[0]).all()   # a_00 = 0: fails at pivot 0


@pytest.mark.parametrize("which", [0, 1])
def test_dense_D_with_diagonal_D_is_dense_batch(which):
    from psp_inputs import config
    s = config(0).system()
    rng = np.random.default_rng(7)
    perm = rng.permutation(s.n) if which else np.arange(s.n)
    eps = np.array([1e-2, -1e-2, 5e-3, -5e-3, 3e-7])
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    X1, st1 = oracle.dense_batch(s, perm.astype(np.int32), eps, tol)
    X2, st2 = oracle.dense_D_batch(s.dense(), np.diag(s.d), perm, eps, tol, s.b)
    assert np.array_equal(st1, st2)
    ok = st1 == 0
    assert ok.any()
    assert np.array_equal(X1[ok], X2[ok])


@pytest.mark.parametrize("m", [1, 2, 3])
def test_predicted_error_dense_D_exact_rationals(m):
    A, _, b = tiny_zero_diag_system(1)
    n = A.shape[0]
    D = _dense_dyadic_D(1)
    Af = [[Fraction(A[i, j]) for j in range(n)] for i in range(n)]
    Df = [[Fraction(D[i, j]) for j in range(n)] for i in range(n)]
    bf = [Fraction(v) for v in b]
    s0 = Fraction(1, 32)
    mags = [j * s0 for j in range(1, m + 1)]
    xs = cramer(Af, bf)
    # recovery in rationals (Remark 2 weights on the +-s_j pairs)
    beta = weights.beta_integer(m)
    xhat = [Fraction(0)] * n
    for bj, s in zip(beta, mags):
        xp, xm = _solve_D(Af, Df, bf, s), _solve_D(Af, Df, bf, -s)
        xhat = [h + bj * (p + q) / 2 for h, p, q in zip(xhat, xp, xm)]
    # (I3) with M = A^{-1} D, column j = A^{-1} D e_j by Cramer
    cols = [cramer(Af, [Df[i][j] for i in range(n)]) for j in range(n)]
    Mx = [[cols[j][i] for j in range(n)] for i in range(n)]
    M2 = [[sum(Mx[i][k] * Mx[k][j] for k in range(n)) for j in range(n)] for i in range(n)]
    v = list(xs)
    for s in mags:
        v = cramer([[(1 if i == j else 0) - s * s * M2[i][j] for j in range(n)] for i in range(n)], v)
    for _ in range(m):
        v = _matvec(M2, v)
    tprod = Fraction(1)
    for s in mags:
        tprod *= s * s
    pred = [(-1) ** m * tprod * vi for vi in v]
    assert [x - h for x, h in zip(xs, xhat)] == pred          # the identity, exactly
    e = oracle.predicted_error(_Tiny(A, np.zeros(n), b), [float(s) for s in mags], Dm=D)[0]
    pf = np.array([float(p) for p in pred])
    assert np.linalg.norm(e - pf) <= 1e-10 * np.linalg.norm(pf)
    # and the oracle's floating-point recovery with this D reproduces x_hat* to rounding
    lane_eps = np.array([v for s in mags for v in (float(s), -float(s))])
    X, st = oracle.dense_D_batch(A, D, np.arange(n), lane_eps, 0.0, b)
    assert (st == 0).all()
    Wm = oracle.ladder_weight_matrix([[float(s) for s in mags]])
    xh = oracle.combine(Wm, X)[0, 0]
    ref = np.array([float(v) for v in xhat])
    assert np.linalg.norm(xh - ref) <= 1e-12 * np.linalg.norm(ref)
