"""GPU parity of PSP_OPT_SKIP_ZERO_ROWS (the capacity-planned batch factor skips the rows
whose multiplier l_{i p} is a structural zero of A's own pattern inside the symmetrised
fill): factors, statuses and solutions BITWISE those of the same launch with the option
off (every row of the fill computed) and of the oracle's dense elimination; the stored
multipliers of the skipped rows are zeros; fused and separate calls; failed lanes
(pivots below the tolerance) keep their statuses."""
import numpy as np
import pytest

import oracle
from oracle import ordering
from psp_inputs import config, ladder_eps

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2311_11833_b200 import psp  # noqa: E402


def make_eps(K, seed):
    """K lanes = K / 8 ladders of the alpha = 1..4 sequence (signed pairs), base eps seeded."""
    rng = np.random.default_rng(seed)
    return np.concatenate([ladder_eps([e * j for j in range(1, 5)]) for e in 10.0 ** rng.uniform(-3.3, -2.3, K // 8)])


def run(s, eps, skip, fused, tol=0.0):
    sv = psp.Solver(0)
    sv.psp_set_option("coop", 2)
    sv.psp_set_option("coop_global", 2)
    sv.psp_set_option("factor_spill", 1)
    sv.psp_set_option("skip_zero_rows", skip)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx)
    info, perm = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s.d)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    if fused:
        sv.psp_factor_solve_batch(A, b, tol)
    else:
        sv.psp_factor_batch(A, tol)
        sv.psp_solve_batch(b.reshape(1, -1))
    assert sv.psp_get_last_kernels()[0] == "batch_spill"
    X = sv.psp_get_solutions().cpu().numpy()
    rc, st = sv.psp_get_lane_status()
    return sv, info, perm, X, st


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("K", [40, 448 + 64])
def test_skip_zero_rows_bitwise(K, fused):
    w = config(1)
    s = w.system()
    eps = make_eps(K, 17)
    on, info, perm, X1, st1 = run(s, eps, 1, fused)
    off, info0, perm0, X0, st0 = run(s, eps, 0, fused)
    assert info["struct_zero_l"] == 222 and info0["struct_zero_l"] == 0
    assert (info["aug_skipped_rows"] if fused else info["skipped_rows"]) > 100
    assert np.array_equal(perm, perm0)
    assert np.array_equal(st1, st0) and (st1 == 0).all()
    assert np.array_equal(X1, X0)
    lanes = np.array(sorted(k for k in {0, 31, 32, 63, K // 2, K - 1} if k < K))
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    Xo, sto = oracle.dense_batch(s, perm, eps[lanes], tol, B=s.b[:, :1])
    assert np.array_equal(X1[lanes], Xo)
    if not fused:   # the stored factor, entry by entry (== treats the skipped rows' +0 as the oracle's signed 0)
        rows = ordering.unsymmetric_structure(s.n, s.row_ptr, s.col_idx, perm)
        for k in (0, 33, K - 1):  # noqa
            f1, f0 = on.psp_get_factor(k, info["nnz_LU"]), off.psp_get_factor(k, info["nnz_LU"])
            assert np.array_equal(f1, f0)
            assert int(np.sum(f1[:info["nnz_L"]] == 0.0)) == 222
        assert sum(1 for i in range(s.n) for j in rows[i] if j < i) == info["nnz_L"] - 222
    on.close()
    off.close()


def test_skip_zero_rows_failed_lanes_status():
    """With a pivot tolerance large enough that lanes fail part-way through the elimination
    (|pivot| < tol), the statuses (1 + first failing pivot) are bit-exact with the option on
    and off and with the oracle; lanes that pass are bitwise equal."""
    w = config(1)
    s = w.system()
    eps = make_eps(64, 3)
    for tol in (0.5, 3.0, 20.0):
        on, info, perm, X1, st1 = run(s, eps, 1, True, tol)
        off, _, _, X0, st0 = run(s, eps, 0, True, tol)
        Xo, sto = oracle.dense_batch(s, perm, eps, tol, B=s.b[:, :1])
        assert np.array_equal(st1, sto) and np.array_equal(st0, sto)
        ok = sto == 0
        assert np.array_equal(X1[ok], Xo[ok]) and np.array_equal(X0[ok], Xo[ok])
        on.close()
        off.close()
    assert (sto != 0).any()
