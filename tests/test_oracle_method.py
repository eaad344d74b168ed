"""Method-level pins for the oracle pipeline (Alg. 1):
perturb -> pivot-free solve -> combine with Remark 2 weights.

Pinned against values and identities the paper and the mathematics fix:
  * SPEC S:L336 worked scalar value (derived from Eq. (9b));
  * (I1) the pair average is exactly (I - s^2 M^2)^{-1} x*, M = A^{-1} D (Eq. (7)
    summed in closed form) -- exact rationals on tiny systems;
  * (I3) the exact recovery error (-1)^m (prod t_j) M^{2m} prod_j (I - t_j M^2)^{-1} x*
    (Theorem 1 with its constant) -- exact rationals;
  * a nilpotent construction where x(eps) is an exact low-degree series, so m=2
    recovers x* exactly (up to rounding) and m=1 does not;
  * O(eps^{2m}) order of accuracy (Theorem 1) on diagonal systems;
  * affine invariance of the combination (sum beta = 1);
  * the residual ||A x_hat - b|| (Alg. 1 step 5) on the 300-bus Jacobian."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import ordering, weights
from golden_util import golden_rows
from psp_inputs import config, ladder_eps
from test_oracle_solve import _Tiny, cramer, tiny_zero_diag_system


def pipeline(sysm, perm, ladders, tol=0.0):
    eps = np.concatenate([ladder_eps(l) for l in ladders])
    X, st = oracle.dense_batch(sysm, perm, eps, tol)
    Wm = oracle.ladder_weight_matrix(ladders)
    return oracle.combine(Wm, X), X, st


def test_scalar_worked_example_spec():
    a, d, b, e, m, xprefix, errprefix = golden_rows("spec_scalar_m2.txt")[0]
    sysm = _Tiny(np.array([[float(a)]]), [float(d)], [float(b)])
    m = int(m)
    mags = [j * float(e) for j in range(1, m + 1)]
    xh, X, st = pipeline(sysm, np.array([0], np.int32), [mags])
    assert (st == 0).all()
    x = xh[0, 0, 0]
    assert f"{x:.15f}".startswith(xprefix)   # SPEC prints a truncated prefix
    assert abs((1.0 - x) - float(errprefix)) < 0.01 * float(errprefix)
    # exact closed form of this case: x* - x_hat* = 4 e^4 / ((1-e^2)(1-4e^2))
    E = Fraction(1, 10)
    exact = 4 * E ** 4 / ((1 - E ** 2) * (1 - 4 * E ** 2))
    assert abs((1.0 - x) - float(exact)) < 1e-15


def _exact_setup(seed, n=5):
    A, d, b = tiny_zero_diag_system(seed, n)
    Af = [[Fraction(A[i, j]) for j in range(n)] for i in range(n)]
    bf = [Fraction(v) for v in b]
    df = [Fraction(v) for v in d]
    return A, d, b, Af, bf, df


def _matvec(M, v):
    return [sum(M[i][j] * v[j] for j in range(len(v))) for i in range(len(M))]


def _solve_pert(Af, df, bf, s):
    n = len(Af)
    M = [[Af[i][j] + (s * df[i] if i == j else 0) for j in range(n)] for i in range(n)]
    return cramer(M, bf)


def _apply_Minv_D(Af, df, v):
    # M v = A^{-1} (D v)
    return cramer(Af, [df[i] * v[i] for i in range(len(v))])


@pytest.mark.parametrize("seed", [0, 1])
def test_I1_pair_average_exact(seed):
    A, d, b, Af, bf, df = _exact_setup(seed)
    n = len(b)
    s = Fraction(1, 16)
    xs = cramer(Af, bf)
    avg = [(p + q) / 2 for p, q in zip(_solve_pert(Af, df, bf, s), _solve_pert(Af, df, bf, -s))]
    # (I - s^2 M^2) avg == x*  (exact)
    M2avg = _apply_Minv_D(Af, df, _apply_Minv_D(Af, df, avg))
    assert [a - s * s * m2 for a, m2 in zip(avg, M2avg)] == xs
    # oracle float pair average agrees to rounding
    sysm = _Tiny(A, d, b)
    X, st = oracle.dense_batch(sysm, np.arange(n, dtype=np.int32)[::-1].copy(),
                               np.array([1 / 16, -1 / 16]), 0.0)
    assert (st == 0).all()
    favg = 0.5 * X[0, 0] + 0.5 * X[1, 0]
    ref = np.array([float(v) for v in avg])
    assert np.linalg.norm(favg - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("m", [1, 2, 3])
def test_I3_exact_error_identity(m):
    A, d, b, Af, bf, df = _exact_setup(1)
    n = len(b)
    s0 = Fraction(1, 32)
    mags = [j * s0 for j in range(1, m + 1)]
    beta = weights.beta_integer(m)
    xs = cramer(Af, bf)
    xhat = [Fraction(0)] * n
    for bj, s in zip(beta, mags):
        xp, xm = _solve_pert(Af, df, bf, s), _solve_pert(Af, df, bf, -s)
        xhat = [h + bj * (p + q) / 2 for h, p, q in zip(xhat, xp, xm)]
    # predicted: (-1)^m (prod t_j) M^{2m} prod_j (I - t_j M^2)^{-1} x*, with M = A^{-1} D
    # formed explicitly (column j = A^{-1} d_j e_j) and each (I - t M^2) y = v solved by Cramer
    cols = [cramer(Af, [df[j] if i == j else Fraction(0) for i in range(n)]) for j in range(n)]
    Mx = [[cols[j][i] for j in range(n)] for i in range(n)]
    M2 = [[sum(Mx[i][k] * Mx[k][j] for k in range(n)) for j in range(n)] for i in range(n)]
    v = list(xs)
    for s in mags:
        t = s * s
        v = cramer([[(1 if i == j else 0) - t * M2[i][j] for j in range(n)] for i in range(n)], v)
    for _ in range(m):
        v = _matvec(M2, v)
    tprod = Fraction(1)
    for s in mags:
        tprod *= s * s
    pred = [(-1) ** m * tprod * vi for vi in v]
    assert [x - h for x, h in zip(xs, xhat)] == pred          # exact identity
    # the oracle's floating-point recovery reproduces x_hat* to rounding
    sysm = _Tiny(A, d, b)
    xh, X, st = pipeline(sysm, np.arange(n, dtype=np.int32), [[float(s) for s in mags]])
    assert (st == 0).all()
    ref = np.array([float(v) for v in xhat])
    assert np.linalg.norm(xh[0, 0] - ref) <= 1e-12 * np.linalg.norm(ref)


def test_nilpotent_exact_recovery():
    # A = [[0,B1,0],[0,0,B2],[B3,0,0]], D = diag(I, I, 0): (A^{-1} D)^3 = 0, so x(eps) is an
    # exact quadratic in eps^2 ... and m >= 2 recovers x* exactly (Theorem 1, finite series).
    rng = np.random.default_rng(11)
    k = 2
    B1, B2, B3 = (rng.normal(size=(k, k)) + 3 * np.eye(k) for _ in range(3))
    Z = np.zeros((k, k))
    A = np.block([[Z, B1, Z], [Z, Z, B2], [B3, Z, Z]])
    d = np.r_[np.ones(2 * k), np.zeros(k)]
    b = rng.normal(size=3 * k)
    Minv = np.linalg.solve(A, np.diag(d))
    assert np.allclose(np.linalg.matrix_power(Minv, 3), 0, atol=1e-12)
    sysm = _Tiny(A, d, b)
    xs = np.linalg.solve(A, b)
    perm = np.arange(3 * k, dtype=np.int32)
    e1, _, st1 = pipeline(sysm, perm, [[0.05]])
    e2, _, st2 = pipeline(sysm, perm, [[0.05, 0.1]])
    assert (st1 == 0).all() and (st2 == 0).all()
    err1 = np.linalg.norm(e1[0, 0] - xs) / np.linalg.norm(xs)
    err2 = np.linalg.norm(e2[0, 0] - xs) / np.linalg.norm(xs)
    print(err1, err2)
    assert err1 > 1e-4           # m = 1 leaves eps^2 M^2 x*
    assert err2 < 1e-11          # m = 2 is exact up to rounding (pivots ~eps: growth ~1/eps^2)


@pytest.mark.parametrize("m", [1, 2, 3])
def test_order_of_accuracy_diagonal(m):
    # diagonal A, D: x* - x_hat* = (-1)^m prod t_j (d/a)^{2m} / prod (1 - t_j d^2/a^2) x*;
    # halving eps divides the error by 2^{2m} (Theorem 1), within a factor 2.
    n = 6
    rng = np.random.default_rng(5)
    a = rng.uniform(1, 2, n) * rng.choice([-1, 1], n)
    d = rng.uniform(0.5, 1, n)
    b = rng.normal(size=n)
    sysm = _Tiny(np.diag(a), d, b)
    xs = b / a
    perm = np.arange(n, dtype=np.int32)
    errs = []
    for e in [0.08, 0.04]:
        xh, _, st = pipeline(sysm, perm, [[j * e for j in range(1, m + 1)]])
        errs.append(np.linalg.norm(xh[0, 0] - xs))
    ratio = errs[0] / errs[1]
    assert 0.5 * 4 ** m <= ratio <= 2 * 4 ** m


def test_diagonal_closed_form_large_n():
    # componentwise closed form at n = 2000 through the sparse oracle (OR2)
    n = 2000
    rng = np.random.default_rng(9)
    a = rng.uniform(1, 3, n) * rng.choice([-1, 1], n)
    d = rng.normal(size=n)
    d /= np.abs(d).max()
    b = rng.normal(size=n)
    sysm = _Tiny(np.diag(a), d, b)
    m, e = 4, 2e-3
    mags = [j * e for j in range(1, m + 1)]
    perm = np.arange(n, dtype=np.int32)
    X, st = oracle.SparseOracle(sysm, perm).batch(np.concatenate([ladder_eps(mags)]), 0.0)
    xh = oracle.combine(oracle.ladder_weight_matrix([mags]), X)[0, 0]
    r = (d / a) ** 2
    pred = np.ones(n) * (-1) ** m
    for s in mags:
        pred *= s * s / (1 - s * s * r)
    pred *= r ** m * (b / a)
    err = (b / a) - xh
    assert np.max(np.abs(err - pred)) <= 4e-16 * np.max(np.abs(b / a)) * 4


def test_combination_affine_invariance():
    # sum beta = 1: a batch of identical lanes recombines to the same vector
    for m in range(1, 6):
        mags = [j * 1e-3 for j in range(1, m + 1)]
        Wm = oracle.ladder_weight_matrix([mags])
        X = np.tile(np.arange(1.0, 6.0), (2 * m, 1, 1))
        out = oracle.combine(Wm, X)[0, 0]
        assert np.allclose(out, np.arange(1.0, 6.0), rtol=4e-15 * sum(abs(w) for w in Wm[0]))


@pytest.mark.parametrize("first", [False, True])
def test_300bus_recovery_and_residual(first):
    w = config(1)
    s = w.system()
    perm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx, first=s.slot_p if first else None)
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    xh, X, st = pipeline(s, perm, w.ladders, tol)
    assert (st == 0).all()
    xs, _ = oracle.reference_solve(s)
    rel = np.linalg.norm(xh[0, 0] - xs[0]) / np.linalg.norm(xs[0])
    assert rel < 1e-11            # ~1e-14 (slack) / <=2.5e-13 floor (leading zero)
    lane = np.linalg.norm(X[0, 0] - xs[0]) / np.linalg.norm(xs[0])
    assert lane > 1e-5            # each perturbed lane alone is far from x*
    A = s.dense()
    bn = s.b[:, 0]
    assert np.linalg.norm(A @ xh[0, 0] - bn) <= 1e-10 * np.linalg.norm(bn)
