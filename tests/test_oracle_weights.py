"""Pins for oracle/weights.py (Remark 2 / Eq. (13))."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import weights
from golden_util import golden_rows


def test_beta_m2_paper_example3():
    # PAPER Example 3: beta = (1/3)[4, -1]
    want = [Fraction(x) for x in golden_rows("paper_example3_beta_m2.txt")[0]]
    assert weights.beta_integer(2) == want


def test_gamma3_paper_eq12():
    want = [[Fraction(x) for x in r] for r in golden_rows("paper_gamma3.txt")]
    assert weights.gamma_matrix([1, 2, 3]) == want


def test_beta_m3_derived():
    # SPEC S:L328 [DERIVED]: m=3 -> [3/2, -3/5, 1/10]
    assert weights.beta_integer(3) == [Fraction(3, 2), Fraction(-3, 5), Fraction(1, 10)]


def test_beta_m1_trivial():
    assert weights.beta_integer(1) == [Fraction(1)]


@pytest.mark.parametrize("m", range(1, 16))
def test_two_routes_agree(m):
    # Vandermonde solve (paper's definition) == Lagrange basis at 0 (closed form)
    assert weights.beta_vandermonde(list(range(1, m + 1))) == weights.beta_lagrange(list(range(1, m + 1)))


@pytest.mark.parametrize("m", range(1, 7))
def test_gamma_conditions(m):
    # Eq. (17): gamma_0 = 1, gamma_2 = ... = gamma_{2(m-1)} = 0
    beta = weights.beta_integer(m)
    for k in range(m):
        g = sum(b * Fraction(j + 1) ** (2 * k) for j, b in enumerate(beta))
        assert g == (1 if k == 0 else 0)


@pytest.mark.parametrize("m", range(1, 7))
def test_beta_vs_lapack(m):
    # library routine on the same Eq. (16) system, in floating point
    G = np.array([[float((j + 1) ** (2 * i)) for j in range(m)] for i in range(m)])  # Gamma_m^T
    e1 = np.zeros(m)
    e1[0] = 1
    ref = np.linalg.solve(G, e1)
    got = np.array([float(b) for b in weights.beta_integer(m)])
    assert np.allclose(got, ref, rtol=1e-9, atol=1e-12)


def test_error_constants_paper():
    for m, power, coef, sign_pinned in golden_rows("paper_error_constants.txt"):
        m, power, coef, sign_pinned = int(m), int(power), int(coef), int(sign_pinned)
        beta = weights.beta_integer(m)
        # x_hat* = sum_k (sum_j beta_j j^{2k}) (A^{-1} eps D)^{2k} A^{-1} b  (Eq. (avg_hats))
        got = sum(b * Fraction(j + 1) ** power for j, b in enumerate(beta))
        if sign_pinned:
            assert got == coef
        else:
            assert abs(got) == abs(coef)


def test_geometric_ladder_weights_depend_on_ratios_only():
    # beta depends only on node ratios: s = {1e-2, 5e-3} (ratio 1/2, cfg0) must give the
    # integer-ladder m=2 weights with the order reversed (largest magnitude first).
    got = weights.beta_lagrange([Fraction(2), Fraction(1)])
    assert got == [Fraction(-1, 3), Fraction(4, 3)]


def test_lane_weights_layout():
    lw = weights.lane_weights([1.0, 2.0])
    assert lw == [2 / 3, 2 / 3, -1 / 6, -1 / 6]
    assert abs(sum(lw) - 1.0) < 1e-15


def test_beta_invariant_under_common_scale():
    """Basis of psp_rescale_failed_rows: beta = (Gamma_m^T)^-1 e_1 (Eq. (13)) depends only
    on ratios of the squared nodes, so scaling a whole ladder leaves it unchanged —
    exactly in rationals, and to rounding in the library's host helper."""
    from fractions import Fraction
    for nodes in ([1, 2, 3], [Fraction(1, 1000), Fraction(3, 1000)], [2, 5, 7, 11]):
        for c in (Fraction(20), Fraction(1, 7), Fraction(-3)):
            assert weights.beta_vandermonde(nodes) == weights.beta_vandermonde([c * x for x in nodes])
    from paper_2311_11833_b200 import psp
    s = np.array([1e-3, 2e-3, 3.5e-3])
    _, w1 = psp.psp_ladder_weights(s)
    _, w2 = psp.psp_ladder_weights(20.0 * s)
    assert np.allclose(w1, w2, rtol=1e-14, atol=0)


def test_two_routes_agree_geometric_ladder():
    # the lane weights' Lagrange route against the paper's Vandermonde solve (Eq. (13)) on a
    # non-integer geometric ladder of binary64 magnitudes (exact rationals, 24 nodes)
    import numpy as np
    mags = [Fraction(float(s)) for s in np.geomspace(1e-1, 1e-8, 24)]
    assert weights.beta_lagrange(mags) == weights.beta_vandermonde(mags)
    lw = weights.lane_weights([float(s) for s in mags])
    assert lw == [float(b / 2) for b in weights.beta_vandermonde(mags) for _ in (0, 1)]
