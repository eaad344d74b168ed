"""Pins for the oracle's tolerance and error references (SURVEY §8(c) step 5 and the
tolerance policy; round-1 verdict "oracle gaps"):

  * oracle.default_tol = n * u * ||A||_1 (reading R10) against SPEC's own
    matrix_one_norm examples and a hand 3x3 whose column sums, row sums and
    signed sums all differ (a row-sum / missing-abs slip fails it);
  * oracle.predicted_error (the exact truncation error (I3) of Theorem 1)
    against: exact rationals on a zero-diagonal 5x5 (an independent Cramer construction
    of M = A^{-1} D), SPEC's worked scalar value, a componentwise closed form
    for diagonal A, D, the index-2 nilpotent family where it is exactly zero, and the
    oracle's own pivot-free recovery on the 300-bus Jacobian where e_pred dominates
    the rounding floor;
  * oracle.pivoted_lanes against LAPACK (numpy.linalg.solve)."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import weights
from golden_util import golden_rows
from psp_inputs import config
from test_oracle_method import _exact_setup, _matvec, _solve_pert, pipeline
from test_oracle_solve import _Tiny, cramer

U = np.finfo(np.float64).eps   # 2^-52


def _csr(Ad):
    n = Ad.shape[0]
    rp, ci, v = [0], [], []
    for i in range(n):
        for j in range(n):
            if Ad[i, j] != 0.0:
                ci.append(j)
                v.append(Ad[i, j])
        rp.append(len(ci))
    return n, np.array(rp, np.int32), np.array(ci, np.int32), np.array(v)


@pytest.mark.parametrize("row", golden_rows("spec_one_norm.txt"), ids=lambda r: r[0])
def test_default_tol_one_norm_pins(row):
    n = int(row[1])
    Ad = np.array([float(x) for x in row[2:2 + n * n]]).reshape(n, n)
    norm1 = float(row[2 + n * n])
    tol = oracle.default_tol(*_csr(Ad))
    assert tol == n * U * norm1          # exact: products of powers of two and small ints
    # the SPEC example by value: diag(0.5, -2) -> n u ||A||_1 = 2 * 2^-52 * 2 = 2^-50
    if row[0] == "diag_half_m2":
        assert tol == 2.0 ** -50
    if row[0] == "hand3":                 # not the inf-norm (6) nor a signed column sum
        assert tol == 3 * 8 * 2.0 ** -52 and tol != 3 * 6 * 2.0 ** -52


def test_pivoted_lanes_vs_lapack():
    s = config(0).system()
    eps = np.array([1e-2, -1e-2, 3e-4])
    X = oracle.pivoted_lanes(s, eps)
    A = s.dense()
    for k, e in enumerate(eps):
        ref = np.linalg.solve(A + e * np.diag(s.d), s.b[:, 0])
        assert np.linalg.norm(X[k, 0] - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("m", [1, 2, 3])
def test_predicted_error_exact_rationals(m):
    # exact (I3) prediction built independently: M = A^{-1} D formed column by column by
    # Cramer's rule, (I - t M^2) y = v solved by Cramer, in Fractions
    A, d, b, Af, bf, df = _exact_setup(1)
    n = len(b)
    s0 = Fraction(1, 32)
    mags = [j * s0 for j in range(1, m + 1)]
    xs = cramer(Af, bf)
    cols = [cramer(Af, [df[j] if i == j else Fraction(0) for i in range(n)]) for j in range(n)]
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
    pred = np.array([float((-1) ** m * tprod * vi) for vi in v])
    # and it is x* - x_hat* exactly (the identity itself, in rationals)
    beta = weights.beta_integer(m)
    xhat = [Fraction(0)] * n
    for bj, s in zip(beta, mags):
        xp, xm = _solve_pert(Af, df, bf, s), _solve_pert(Af, df, bf, -s)
        xhat = [h + bj * (p + q) / 2 for h, p, q in zip(xhat, xp, xm)]
    assert np.array_equal(pred, np.array([float(x - h) for x, h in zip(xs, xhat)]))
    e = oracle.predicted_error(_Tiny(A, d, b), [float(s) for s in mags])[0]
    assert np.linalg.norm(e - pred) <= 1e-10 * np.linalg.norm(pred)


def test_predicted_error_spec_scalar():
    # a = d = b = 1, eps = 0.1, m = 2: x* - x_hat* = 4 e^4 / ((1 - e^2)(1 - 4 e^2))
    a, d, b, e, m, xprefix, errprefix = golden_rows("spec_scalar_m2.txt")[0]
    e = float(e)
    pred = oracle.predicted_error(_Tiny(np.array([[float(a)]]), [float(d)], [float(b)]),
                                  [e, 2 * e])[0, 0]
    E = Fraction(1, 10)
    exact = float(4 * E ** 4 / ((1 - E ** 2) * (1 - 4 * E ** 2)))
    assert abs(pred - exact) <= 4 * U * exact
    assert abs(pred - float(errprefix)) < 0.01 * float(errprefix)


@pytest.mark.parametrize("m", [1, 2, 4, 7])
def test_predicted_error_diagonal_closed_form(m):
    # diagonal A, D: componentwise (-1)^m prod t_j (d_i/a_i)^{2m} / prod_j (1 - t_j d_i^2/a_i^2) x*_i
    rng = np.random.default_rng(40 + m)
    n = 60
    a = rng.uniform(0.5, 2.0, n) * rng.choice([-1, 1], n)
    d = rng.normal(size=n)
    d /= np.abs(d).max()
    b = rng.normal(size=n)
    sysm = _Tiny(np.diag(a), d, b)
    mags = [0.03 * j for j in range(1, m + 1)]
    e = oracle.predicted_error(sysm, mags)[0]
    ld = np.longdouble
    ref = np.empty(n)
    for i in range(n):
        mu = (ld(d[i]) / ld(a[i])) ** 2
        val = ld(b[i]) / ld(a[i])
        for s in mags:
            t = ld(s) * ld(s)
            val *= t * mu / (1 - t * mu)
        ref[i] = float((-1) ** m * val)
    assert np.all(np.abs(e - ref) <= 1e-13 * np.abs(ref) + 1e-300)


def test_predicted_error_nilpotent_is_zero():
    # A = [[0, B], [C, 0]], D = diag(I, 0): M^2 = 0, so every pair average is x* exactly
    # and the predicted error vanishes identically (for any ladder)
    rng = np.random.default_rng(5)
    k = 3
    Bm, Cm = rng.normal(size=(k, k)) + 3 * np.eye(k), rng.normal(size=(k, k)) + 3 * np.eye(k)
    A = np.block([[np.zeros((k, k)), Bm], [Cm, np.zeros((k, k))]])
    d = np.concatenate([np.ones(k), np.zeros(k)])
    sysm = _Tiny(A, d, rng.normal(size=2 * k))
    for mags in ([0.1], [0.05, 0.1, 0.2]):
        assert np.all(oracle.predicted_error(sysm, mags) == 0.0)


@pytest.mark.parametrize("m,base", [(1, 2e-3), (2, 1e-2), (3, 2e-2)])
def test_predicted_error_matches_oracle_recovery_300bus(m, base):
    # where the truncation error dominates the rounding floor, the oracle's pivot-free
    # recovery reproduces x* - x_hat* = e_pred vector-wise (two independent routes:
    # pivot-free lanes + Remark 2 weights, vs partial-pivot operators of (I3))
    from oracle import ordering
    s = config(1).system()
    perm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx)
    mags = [base * j for j in range(1, m + 1)]
    xh, X, st = pipeline(s, perm, [mags])
    assert (st == 0).all()
    xs, _ = oracle.reference_solve(s)
    e = oracle.predicted_error(s, mags)[0]
    got = xs[0] - xh[0, 0]
    assert np.linalg.norm(e) > 1e-9 * np.linalg.norm(xs[0])
    assert np.linalg.norm(got - e) <= 1e-3 * np.linalg.norm(e)
