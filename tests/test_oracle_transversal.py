"""Pins for the oracle's Hopcroft-Karp transversal: the matching
is a valid matching (distinct rows, every matched pair a structural nonzero), it is maximum
(its size equals brute force over all permutations on tiny patterns, and scipy's maximum
bipartite matching on larger ones), a structurally nonsingular pattern gets a zero-free
diagonal after the row permutation, and on the power-flow Jacobian in the 'listed'
convention (almost every diagonal structurally zero) it produces a zero-free diagonal."""
import itertools

import numpy as np
import pytest

from oracle import transversal
from psp_inputs import config


def _csr_from_mask(M):
    n = M.shape[0]
    rp, ci = [0], []
    for i in range(n):
        for j in range(n):
            if M[i, j]:
                ci.append(j)
        rp.append(len(ci))
    return np.array(rp, np.int32), np.array(ci, np.int32)


def _check_valid(n, rp, ci, q):
    rows = [r for r in q if r >= 0]
    assert len(rows) == len(set(rows))
    for j, r in enumerate(q):
        if r >= 0:
            assert j in set(ci[rp[r]:rp[r + 1]])


@pytest.mark.parametrize("seed", range(8))
def test_hk_maximum_vs_brute_force(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 7))
    M = rng.random((n, n)) < 0.35
    rp, ci = _csr_from_mask(M)
    q = transversal.hopcroft_karp(n, rp, ci)
    _check_valid(n, rp, ci, q)
    best = 0
    for k in range(n, 0, -1):   # largest k such that some k columns match distinct rows
        for cols in itertools.combinations(range(n), k):
            for rows in itertools.permutations(range(n), k):
                if all(M[r, c] for r, c in zip(rows, cols)):
                    best = k
                    break
            if best:
                break
        if best:
            break
    assert sum(r >= 0 for r in q) == best


@pytest.mark.parametrize("seed", range(4))
def test_hk_maximum_vs_scipy(seed):
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import maximum_bipartite_matching
    rng = np.random.default_rng(100 + seed)
    n = 60
    M = rng.random((n, n)) < 0.05
    rp, ci = _csr_from_mask(M)
    q = transversal.hopcroft_karp(n, rp, ci)
    _check_valid(n, rp, ci, q)
    m = maximum_bipartite_matching(csr_matrix(M.astype(np.int8)), perm_type="row")
    assert sum(r >= 0 for r in q) == int((m >= 0).sum())


def test_hk_zero_free_diagonal_on_listed_jacobian():
    s = config(0).system(convention="listed")
    n = s.n
    diag0 = sum(1 for i in range(n) if i in set(s.col_idx[s.row_ptr[i]:s.row_ptr[i + 1]]))
    assert diag0 < n                               # the listed order has zero diagonals
    q = transversal.hopcroft_karp(n, s.row_ptr, s.col_idx)
    assert sorted(q) == list(range(n))             # perfect matching: a permutation
    rp, ci, v = transversal.permuted_rows(n, s.row_ptr, s.col_idx, s.vals, q)
    for j in range(n):
        assert j in set(ci[rp[j]:rp[j + 1]])       # zero-free diagonal
