"""Generator checks (psp_inputs): the synthetic distributed-slack Jacobian is the
derivative of the power-flow mismatch it claims to be, and has the structure the
paper's workload has (J in R^{531x531}, a zero on the diagonal)."""
import numpy as np
import pytest

from psp_inputs import build_system, config, power_injections


def _mismatch(aux, x, n_bus):
    """F = [P_i(V,th) - alpha_i*lam for all buses; Q_i(V,th) for PQ buses] in the
    row order of J, as a function of the unknown vector x in J's column order."""
    th = aux["th"].copy()
    V = aux["V"].copy()
    for bus, c in aux["th_col"].items():
        th[bus] = x[c]
    for bus, c in aux["V_col"].items():
        V[bus] = x[c]
    lam = x[aux["lam_col"]]
    P, Q = power_injections(aux["Y"], V, th)
    F = np.zeros(len(x))
    F[:n_bus] = P - aux["alpha"] * lam
    for bus, r in aux["rows_q"].items():
        F[r] = Q[bus]
    return F


@pytest.mark.parametrize("convention", ["slack", "listed"])
def test_jacobian_matches_finite_differences(convention):
    s = build_system(14, 20, 4, seed=0, convention=convention)
    aux = s.aux
    x0 = np.zeros(s.n)
    for bus, c in aux["th_col"].items():
        x0[c] = aux["th"][bus]
    for bus, c in aux["V_col"].items():
        x0[c] = aux["V"][bus]
    J = s.dense()
    h = 1e-6
    Jfd = np.zeros_like(J)
    for c in range(s.n):
        e = np.zeros(s.n)
        e[c] = h
        Jfd[:, c] = (_mismatch(aux, x0 + e, s.n_bus) - _mismatch(aux, x0 - e, s.n_bus)) / (2 * h)
    assert np.max(np.abs(J - Jfd)) < 1e-7 * max(1.0, np.max(np.abs(J)))


def test_shapes_and_structure():
    s0 = config(0).system()
    assert s0.n == 24            # 13 theta + 10 V + lambda (reading R14: BASELINE says 27)
    assert s0.n_struct_zero_diag == 1
    s1 = config(1).system()
    assert s1.n == 531           # P:L302 "J in R^{531x531}"
    assert s1.n_struct_zero_diag == 1
    assert 3000 < s1.nnz < 5000
    l1 = config(1).system(convention="listed")
    assert l1.n_struct_zero_diag > 500
    # d normalisation: ||D||_1 = max|d| = 1
    assert np.max(np.abs(s1.d)) == 1.0


def test_deterministic():
    a = config(1).system()
    b = config(1).system()
    assert np.array_equal(a.vals, b.vals) and np.array_equal(a.b, b.b) and np.array_equal(a.d, b.d)
