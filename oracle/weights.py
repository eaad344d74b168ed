"""ORACLE (test infrastructure only): recombination weights of Remark 2 / Eq. (13).

PAPER.md P:L197-203 (Remark 2): x_hat* = [x_hat_1 ... x_hat_m] (Gamma_m^T)^{-1} e_1,
with Gamma_m the m x m Vandermonde matrix of Eq. (8), entry (i, j) =
(alpha_i)^{2j}, i.e. powers of the squared nodes t_i = alpha_i^2 (P:L188-195 shows
Gamma_3 = [[1,1,1],[1,4,16],[1,9,81]]).  The construction proof
solves Gamma_m^T beta = [1, 0, ..., 0]^T (Eq. (16)-(17)).

Two independent exact-rational routes are given:
  * beta_vandermonde: forms Gamma_m^T from Eq. (8)/(16) and solves it by exact
    Fraction Gaussian elimination — the paper's literal definition;
  * beta_lagrange: the Lagrange basis polynomial at 0 on nodes t_i (the closed form
    SPEC S:L323 names) — a second route, cross-checked against the first in tests.

For non-integer magnitudes s_j (a geometric ladder, P:L120 allows decimal alpha)
the nodes are t_j = s_j^2 taken as exact rationals of the binary64 inputs.
The per-lane weight of x^+(s_j) and x^-(s_j) is beta_j / 2 (Eq. (avg_hats),
P:L205-215: x_hat_j = (x^+ + x^-)/2).
"""
from __future__ import annotations

import functools
from fractions import Fraction


def gamma_matrix(nodes):
    """Gamma_m of Eq. (8): row i = [t_i^0, t_i^1, ..., t_i^{m-1}] with t_i = alpha_i^2."""
    t = [Fraction(a) ** 2 for a in nodes]
    m = len(t)
    return [[t[i] ** j for j in range(m)] for i in range(m)]


def _solve_exact(M, rhs):
    m = len(M)
    A = [list(M[i]) + [rhs[i]] for i in range(m)]
    for p in range(m):
        r = next(i for i in range(p, m) if A[i][p] != 0)
        A[p], A[r] = A[r], A[p]
        for i in range(m):
            if i != p and A[i][p] != 0:
                f = A[i][p] / A[p][p]
                A[i] = [a - f * c for a, c in zip(A[i], A[p])]
    return [A[i][m] / A[i][i] for i in range(m)]


def beta_vandermonde(nodes):
    """beta = (Gamma_m^T)^{-1} e_1 (Eq. (13)), exact rationals."""
    G = gamma_matrix(nodes)
    m = len(G)
    GT = [[G[j][i] for j in range(m)] for i in range(m)]
    return _solve_exact(GT, [Fraction(1)] + [Fraction(0)] * (m - 1))


def beta_lagrange(nodes):
    """beta_j = prod_{l != j} t_l / (t_l - t_j): Lagrange basis at 0."""
    t = [Fraction(a) ** 2 for a in nodes]
    out = []
    for j in range(len(t)):
        b = Fraction(1)
        for l in range(len(t)):
            if l != j:
                b *= t[l] / (t[l] - t[j])
        out.append(b)
    return out


def beta_integer(m):
    """The paper's alpha = 1..m ladder: beta for nodes 1^2..m^2."""
    return beta_vandermonde(list(range(1, m + 1)))


def lane_weights(magnitudes):
    """Signed-lane weights for one ladder in lane order [+s1, -s1, +s2, -s2, ...]:
    each sign carries beta_j / 2 (pair average of Eq. (avg_hats)).  Returns floats
    correctly rounded from the exact rationals.  The rationals come from the Lagrange
    route (the same exact values as the Vandermonde solve of Eq. (13): both routes are
    pinned equal in tests/test_oracle_weights.py), O(m^2) instead of O(m^3) exact
    operations -- the 128-node ladder of BASELINE configs[2] takes 0.4 s instead of
    minutes; memoised per ladder."""
    return list(_lane_weights(tuple(float(s) for s in magnitudes)))


@functools.lru_cache(maxsize=256)
def _lane_weights(mags):
    beta = beta_lagrange([Fraction(s) for s in mags])
    out = []
    for bj in beta:
        out += [float(bj / 2), float(bj / 2)]
    return tuple(out)


def error_constant(m):
    """gamma_{2m}: coefficient of (A^{-1} eps D)^{2m} A^{-1} b left in x_hat* after
    the combination (sum_j beta_j alpha_j^{2m}), for the integer ladder."""
    beta = beta_integer(m)
    return sum(b * Fraction(j + 1) ** (2 * m) for j, b in enumerate(beta))
