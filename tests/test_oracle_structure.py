"""Structural zeros of A's own pattern inside the symmetrised fill (PSP_OPT_SKIP_ZERO_ROWS).

The oracle's unsymmetric_structure() is the plain definition; it is pinned here to the
NUMBERS of the oracle's dense pivot-free elimination (the exact zeros of L + U on a
generic lane are exactly the entries outside that structure), to a hand example, and the
product's planner count is compared with it."""
import numpy as np
import pytest

import oracle
from oracle import ordering
from paper_2311_11833_b200 import psp
from psp_inputs import config


def dense_lane(s, perm, eps):
    A = np.zeros((s.n, s.n))
    for i in range(s.n):
        for q in range(s.row_ptr[i], s.row_ptr[i + 1]):
            A[i, s.col_idx[q]] += s.vals[q]
    A = A + eps * np.diag(s.d)
    return A[np.ix_(perm, perm)]


def test_hand_example_arrow():
    """A = [[x, x, 0], [0, x, x], [x, 0, x]] in natural order: the symmetrised fill is full;
    under A's own pattern (2, 0) x (0, 1) fills (2, 1), nothing fills (1, 0) or (0, 2)."""
    row_ptr, col_idx = [0, 2, 4, 6], [0, 1, 1, 2, 0, 2]
    rows = ordering.unsymmetric_structure(3, row_ptr, col_idx, [0, 1, 2])
    assert rows == [{0, 1}, {1, 2}, {0, 1, 2}]
    fcp, fri = ordering.filled_pattern(3, row_ptr, col_idx, [0, 1, 2])
    assert int(fcp[-1]) == 9


@pytest.mark.parametrize("ci", [0, 1])
def test_structure_matches_the_dense_elimination_zeros(ci):
    s = config(ci).system()
    perm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx)
    rows = ordering.unsymmetric_structure(s.n, s.row_ptr, s.col_idx, perm)
    fcp, fri = ordering.filled_pattern(s.n, s.row_ptr, s.col_idx, perm)
    LU, st = oracle.lu_nopivot(dense_lane(s, perm, 1.7e-3), 0.0)
    assert st == 0
    n_zero_l = 0
    for j in range(s.n):
        for i in fri[fcp[j]:fcp[j + 1]]:
            i = int(i)
            for (a, b) in ((i, j), (j, i)):          # the filled pattern is symmetric
                assert (LU[a, b] != 0.0) == (b in rows[a]), (a, b)
            n_zero_l += i > j and j not in rows[i]
    # outside the symmetrised fill everything is zero
    mask = np.zeros((s.n, s.n), bool)
    for j in range(s.n):
        mask[fri[fcp[j]:fcp[j + 1]], j] = True
    assert not LU[~mask].any()
    # the product's planner finds the same multipliers
    hs = psp.HostSymbolic()
    info, p2 = hs.analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
    assert np.array_equal(p2, perm)
    assert info["struct_zero_l"] == n_zero_l
    assert 0 <= info["aug_skipped_rows"] <= n_zero_l and 0 <= info["skipped_rows"] <= n_zero_l
    if ci == 1:
        assert n_zero_l == 222 and info["aug_skipped_rows"] > 0


def test_option_off_reports_no_zeros():
    s = config(1).system()
    hs = psp.HostSymbolic()
    hs.set_option("skip_zero_rows", 0)
    info, _ = hs.analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
    assert info["struct_zero_l"] == 0 and info["skipped_rows"] == 0 and info["aug_skipped_rows"] == 0
