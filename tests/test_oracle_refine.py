"""Pins for the oracle's iterative-refinement baseline:

  * residual_fma (r = b - A x, one fma per CSR entry in order) against exact integer
    arithmetic on small integer systems (every product and sum exact in binary64);
  * refine's iterates against the same iteration carried out in exact rationals (Cramer)
    on zero-diagonal 5x5 systems with dyadic data, and the closed form of its error,
    x* - x^i = (eps M)^{i+1} x*, M = (A + eps D)^{-1} D, verified in rationals;
  * on the 300-bus Jacobian: geometric convergence to the partial-pivot x* (LAPACK) at the
    rate |eps| rho(M) until the rounding floor."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from psp_inputs import config
from test_oracle_solve import _Tiny, cramer, tiny_zero_diag_system


def test_residual_fma_exact_integers():
    rng = np.random.default_rng(3)
    for n in (1, 4, 9):
        A = rng.integers(-9, 10, size=(n, n)).astype(float)
        A[rng.random((n, n)) < 0.4] = 0.0
        x = rng.integers(-20, 21, size=n).astype(float)
        b = rng.integers(-50, 51, size=n).astype(float)
        s = _Tiny(A, np.ones(n), b)
        r = oracle.residual_fma(s, x, b)
        exact = [int(b[i]) - sum(int(A[i, j]) * int(x[j]) for j in range(n)) for i in range(n)]
        assert np.array_equal(r, np.array(exact, dtype=float))


@pytest.mark.parametrize("seed", [0, 1])
def test_refine_iterates_vs_exact_rationals(seed):
    A, d, b = tiny_zero_diag_system(seed)
    n = len(b)
    s = _Tiny(A, d, b)
    e = 1 / 16
    iters = 5
    X, st = oracle.refine(s, np.arange(n), np.array([e]), 0.0, iters)
    assert st[0] == 0
    Af = [[Fraction(v) for v in row] for row in A]
    bf = [Fraction(v) for v in b]
    F = [[Af[i][j] + (Fraction(e) * Fraction(d[i]) if i == j else 0) for j in range(n)] for i in range(n)]
    xs = cramer(Af, bf)
    x = cramer(F, bf)
    Mcols = [cramer(F, [Fraction(d[j]) if i == j else Fraction(0) for i in range(n)]) for j in range(n)]

    def eM(v):   # (eps M) v, M = F^{-1} D
        return [Fraction(e) * sum(Mcols[j][i] * v[j] for j in range(n)) for i in range(n)]

    err = eM(xs)                                        # e^0 = eps M x*
    for i in range(iters + 1):
        if i > 0:
            r = [bf[a] - sum(Af[a][j] * x[j] for j in range(n)) for a in range(n)]
            c = cramer(F, r)
            x = [u + v for u, v in zip(x, c)]
            err = eM(err)
        assert [p - q for p, q in zip(xs, x)] == err     # closed form, exactly
        ref = np.array([float(v) for v in x])
        assert np.linalg.norm(X[i, 0] - ref) <= 1e-12 * np.linalg.norm(ref)


def test_refine_converges_on_300bus():
    s = config(1).system()
    from oracle import ordering
    perm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx)
    xs = np.linalg.solve(s.dense(), s.b[:, 0])
    e = 2e-3
    X, st = oracle.refine(s, perm, np.array([e]), 0.0, 6)
    assert st[0] == 0
    errs = [np.linalg.norm(X[i, 0] - xs) / np.linalg.norm(xs) for i in range(7)]
    rho, _, _ = oracle.power_rho(s, np.ones(s.n))
    # geometric until the floor: each step gains at least the factor ~ 1 / (eps rho) / 10
    for i in range(6):
        if errs[i] > 1e-12:
            assert errs[i + 1] <= max(10 * e * rho * errs[i], 1e-13), errs
    assert errs[-1] < 1e-11
