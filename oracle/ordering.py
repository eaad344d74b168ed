"""ORACLE (test infrastructure only): elimination order and filled pattern.

The paper eliminates in the natural order of a dense matrix (getrf).  A
sparse solver must choose an elimination order; the result x_k of each lane is
independent of it in exact arithmetic, but its rounding is not, so for
element-by-element parity the oracle eliminates in the same order as the CUDA
path.  It does NOT take that order from the product: it computes it itself, with
the textbook exact minimum-degree rule (reading R13):

  on the elimination graph of pattern(A + A^T) (self loops removed), repeatedly
  eliminate the vertex of smallest current degree, ties to the smallest original
  index; eliminating v joins its remaining neighbours into a clique and removes v.

`first` (optional) forces one vertex to be eliminated first, then the rule
continues on the rest — the 'leading-zero' stress convention ("A leading 0
was always encountered on a diagonal").  The permutation is perm[new] = old.

Parity of the permutation itself (integer, bit-exact) is checked against the
product's in the GPU-free tests.
"""
from __future__ import annotations

import heapq

import numpy as np


def symmetric_adjacency(n, row_ptr, col_idx):
    adj = [set() for _ in range(n)]
    for i in range(n):
        for q in range(int(row_ptr[i]), int(row_ptr[i + 1])):
            j = int(col_idx[q])
            if j != i:
                adj[i].add(j)
                adj[j].add(i)
    return adj


def _eliminate(adj, v):
    nb = adj[v]
    for a in nb:
        adj[a].discard(v)
    nbl = list(nb)
    for x in range(len(nbl)):
        ax = adj[nbl[x]]
        for y in range(len(nbl)):
            if x != y:
                ax.add(nbl[y])
    adj[v] = set()
    return nbl


def min_degree_order(n, row_ptr, col_idx, first=None):
    adj = symmetric_adjacency(n, row_ptr, col_idx)
    alive = [True] * n
    heap = [(len(adj[v]), v) for v in range(n)]
    heapq.heapify(heap)
    perm = []

    def elim(v):
        alive[v] = False
        perm.append(v)
        for a in _eliminate(adj, v):
            heapq.heappush(heap, (len(adj[a]), a))

    if first is not None:
        elim(int(first))
    while heap:
        deg, v = heapq.heappop(heap)
        if not alive[v] or deg != len(adj[v]):
            continue
        elim(v)
    assert len(perm) == n
    return np.array(perm, dtype=np.int32)


def filled_pattern(n, row_ptr, col_idx, perm):
    """Filled pattern of L+U for the symmetric-pattern elimination of P A P^T
    (pattern(A+A^T) plus the diagonal, plus every fill edge the elimination graph
    creates).  Returns CSC (colptr, rowind) in the permuted numbering, rows sorted."""
    inv = np.empty(n, dtype=np.int64)
    inv[np.asarray(perm)] = np.arange(n)
    adj0 = symmetric_adjacency(n, row_ptr, col_idx)
    adj = [set(int(inv[j]) for j in adj0[int(perm[i])]) for i in range(n)]
    cols = [set([j]) for j in range(n)]
    for p in range(n):
        higher = sorted(a for a in adj[p] if a > p)
        for i in higher:          # (i, p) in L and (p, i) in U
            cols[p].add(i)
            cols[i].add(p)
        for x in higher:
            for y in higher:
                if x != y:
                    adj[x].add(y)
    colptr = np.zeros(n + 1, dtype=np.int32)
    rows = []
    for j in range(n):
        r = sorted(cols[j])
        rows += r
        colptr[j + 1] = colptr[j] + len(r)
    return colptr, np.array(rows, dtype=np.int32)


def unsymmetric_structure(n, row_ptr, col_idx, perm):
    """Structure of L + U for the pivot-free elimination of P A P^T under A's OWN pattern
    (no symmetrisation): the plain definition -- entry (i, j) is structurally non-zero if
    it is on the diagonal (a_ii + eps d_i), in pattern(A), or receives an update
    l_{i p} u_{p j} with both factors structurally non-zero, pivots p ascending.  Returns
    the list of row sets (permuted numbering).  Every entry of filled_pattern() that is not
    in this structure is exactly 0 in every lane of the dense pivot-free factorisation
    (pinned numerically in tests/test_oracle_structure.py)."""
    inv = np.empty(n, dtype=np.int64)
    inv[np.asarray(perm)] = np.arange(n)
    rows = [set([i]) for i in range(n)]
    for i in range(n):
        for q in range(row_ptr[i], row_ptr[i + 1]):
            rows[int(inv[i])].add(int(inv[col_idx[q]]))
    cols = [set() for _ in range(n)]
    for i in range(n):
        for j in rows[i]:
            cols[j].add(i)
    for p in range(n):
        lp = [i for i in cols[p] if i > p]
        up = [j for j in rows[p] if j > p]
        for i in lp:
            for j in up:
                if j not in rows[i]:
                    rows[i].add(j)
                    cols[j].add(i)
    return rows


def permuted_csc(n, row_ptr, col_idx, vals, perm):
    """CSC of P A P^T (values copied, no arithmetic)."""
    inv = np.empty(n, dtype=np.int64)
    inv[np.asarray(perm)] = np.arange(n)
    cols = [[] for _ in range(n)]
    for i in range(n):
        for q in range(int(row_ptr[i]), int(row_ptr[i + 1])):
            cols[int(inv[col_idx[q]])].append((int(inv[i]), float(vals[q])))
    colptr = np.zeros(n + 1, dtype=np.int32)
    rows, vs = [], []
    for j in range(n):
        c = sorted(cols[j])
        rows += [r for r, _ in c]
        vs += [v for _, v in c]
        colptr[j + 1] = colptr[j] + len(c)
    return colptr, np.array(rows, dtype=np.int32), np.array(vs, dtype=np.float64)


def postorder_big_first(n, row_ptr, col_idx, perm0, first=None):
    """Relabel an elimination order into a postorder of its elimination tree
    (R13): the etree parent of column j is the smallest row index of
    L(:, j) below the diagonal; each subtree gets the weight sum_{k in subtree}
    |L(:, k)|^2; roots and the children of every node are visited by descending
    weight, ties by ascending index; a node is emitted after its children.  If
    `first` is given (the leading-zero regime) that vertex — a leaf, since it is
    eliminated first — is moved to the front.  Returns perm[new] = old.  A
    postorder is a topological order of the etree, so the filled pattern is the
    same set of entries (relabelled)."""
    fcp, fri = filled_pattern(n, row_ptr, col_idx, perm0)
    lcount = [0] * n
    parent = [-1] * n
    for j in range(n):
        rows = [int(r) for r in fri[fcp[j]:fcp[j + 1]] if r > j]
        lcount[j] = len(rows)
        parent[j] = min(rows) if rows else -1
    weight = [lcount[j] ** 2 for j in range(n)]
    for j in range(n):                      # children have smaller index than parents
        if parent[j] >= 0:
            weight[parent[j]] += weight[j]
    children = [[] for _ in range(n)]
    roots = []
    for j in range(n):
        (children[parent[j]] if parent[j] >= 0 else roots).append(j)
    key = lambda v: (-weight[v], v)          # noqa: E731
    order = []
    stack = [(r, False) for r in sorted(roots, key=key, reverse=True)]
    while stack:
        v, done = stack.pop()
        if done:
            order.append(v)
            continue
        stack.append((v, True))
        for c in sorted(children[v], key=key, reverse=True):
            stack.append((c, False))
    perm0 = np.asarray(perm0)
    perm = [int(perm0[v]) for v in order]
    if first is not None:
        perm.remove(int(first))
        perm.insert(0, int(first))
    return np.array(perm, dtype=np.int32)


def elimination_order(n, row_ptr, col_idx, first=None):
    """The oracle's elimination order: exact minimum degree, then the big-first
    postorder of its elimination tree (R13)."""
    perm0 = min_degree_order(n, row_ptr, col_idx, first=first)
    return postorder_big_first(n, row_ptr, col_idx, perm0, first=first)
