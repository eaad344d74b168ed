"""GPU parity of the structural transversal pre-pass (PSP_OPT_TRANSVERSAL; SURVEY §8(f) 4,
P:L304: Hopcroft-Karp "permutes a matrix by moving non-zeros onto the diagonal").

The library analyses A_hat = A[q, :] and takes A's values and b in the caller's order.
The oracle computes its own matching q (oracle/transversal.py, bit-exact with the
product's, pinned in the CPU tests), forms A_hat and b[q] itself and runs its pivot-free
solve: per-lane solutions and statuses BITWISE equal, recovered x within 1e-10, and the
recovered x against the partial-pivot x* of the ORIGINAL system within the predicted
truncation error (the row permutation does not change x)."""
import dataclasses

import numpy as np
import pytest

import oracle
from oracle import ordering, transversal
from psp_inputs import config, ladder_eps

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2311_11833_b200 import psp  # noqa: E402


def hat_system(s):
    q = transversal.hopcroft_karp(s.n, s.row_ptr, s.col_idx)
    rp, ci, v = transversal.permuted_rows(s.n, s.row_ptr, s.col_idx, s.vals, q)
    return q, dataclasses.replace(s, row_ptr=rp, col_idx=ci, vals=v, b=s.b[np.array(q)])


@pytest.mark.parametrize("ci,conv", [(0, "listed"), (1, "listed"), (1, "slack")])
def test_transversal_lanes_and_recovery(ci, conv):
    s = config(ci).system(convention=conv)
    q, sh = hat_system(s)
    mags = [2e-3 * j for j in range(1, 5)]
    eps = np.r_[ladder_eps(mags), 0.0]          # + one unperturbed lane (the HK-only baseline)
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    sv = psp.Solver(0)
    sv.psp_set_option("transversal", 1)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx)
    info, perm = sv.psp_get_symbolic_info()
    assert np.array_equal(sv.psp_get_transversal(), np.array(q, np.int32))
    assert info["n_struct_zero_diag"] == 0
    assert np.array_equal(perm, ordering.elimination_order(sh.n, sh.row_ptr, sh.col_idx))
    sv.psp_set_perturbations(eps, s.d)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")       # the caller's order
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    sv.psp_factor_solve_batch(A, b, tol)
    X = sv.psp_get_solutions().cpu().numpy()
    rc, st = sv.psp_get_lane_status()
    Xo, sto = oracle.dense_batch(sh, perm, eps, tol)
    assert np.array_equal(st, sto)
    ok = sto == 0
    assert ok[:8].all()
    assert np.array_equal(X[ok], Xo[ok])                                 # bitwise per lane
    sv.psp_set_weights(*psp.ladder_weights_csr([mags]))
    xh = sv.psp_recover().cpu().numpy()
    xo = oracle.combine(oracle.ladder_weight_matrix([mags]), Xo[:8])
    assert np.linalg.norm(xh - xo) <= 1e-10 * np.linalg.norm(xo)
    xs = np.linalg.solve(s.dense(), s.b[:, 0])                           # x* of the original A
    e = oracle.predicted_error(sh, mags)[0]
    assert np.linalg.norm(xs - xh[0, 0]) <= 1.5 * np.linalg.norm(e) + 1e-9 * np.linalg.norm(xs)
    # the residual against the ORIGINAL A and b (the library gathers them itself)
    res = sv.psp_residual(A, torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda"),
                          torch.tensor(xh, device="cuda"))
    assert abs(res[0, 0] - oracle.residual(s, xh)[0, 0]) <= 1e-12 * (1 + np.linalg.norm(s.b))
