"""ORACLE (test infrastructure only): the structural transversal pre-pass (
PAPER P:L304: "we additionally applied the Hopcroft-Karp algorithm (which permutes a matrix
by moving non-zeros onto the diagonal)").

A maximum matching of the bipartite graph columns j -- rows i (edge where A[i][j] is
structurally nonzero) by Hopcroft-Karp, written out in the textbook form (phases of a BFS
from every free column building the layer distances, with NIL standing for "a free row",
then a DFS from each free column along layered edges), with every choice made in a fixed
order so that the result is a function of the pattern alone (reading R20):

  BFS: free columns j ascending enter the queue with dist 0, others dist = INF; NIL = INF.
       Pop j; if dist[j] < dist[NIL]: for rows i of column j ascending: j2 = row_match[i];
       if j2 is NIL and dist[NIL] = INF: dist[NIL] = dist[j] + 1; if j2 is a column with
       dist[j2] = INF: dist[j2] = dist[j] + 1, push j2.
  DFS(j): for rows i of column j ascending: j2 = row_match[i]; if (j2 is NIL and
       dist[NIL] = dist[j] + 1) or (j2 is a column, dist[j2] = dist[j] + 1 and DFS(j2)):
       match (i, j), return true.  Otherwise dist[j] = INF, return false.
  Phase: BFS; stop when dist[NIL] = INF; else DFS(j) for every free column j ascending.

Returns q with q[j] = the row matched to column j (-1 if unmatched): the row-permuted matrix
A_hat = A[q, :] has a structurally nonzero diagonal iff the matching is perfect.  This
module shares nothing with the product and takes only the pattern."""
from __future__ import annotations

import sys

INF = float("inf")


def columns_of(n, row_ptr, col_idx):
    """rows of each column, ascending (CSR rows are scanned in order)."""
    cols = [[] for _ in range(n)]
    for i in range(n):
        for q in range(int(row_ptr[i]), int(row_ptr[i + 1])):
            cols[int(col_idx[q])].append(i)
    return cols


def hopcroft_karp(n, row_ptr, col_idx):
    cols = columns_of(n, row_ptr, col_idx)
    col_match = [-1] * n
    row_match = [-1] * n
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 4 * n + 100))
    try:
        while True:
            dist = [INF] * n
            queue = []
            for j in range(n):
                if col_match[j] < 0:
                    dist[j] = 0
                    queue.append(j)
            dnil = INF
            h = 0
            while h < len(queue):
                j = queue[h]
                h += 1
                if dist[j] < dnil:
                    for i in cols[j]:
                        j2 = row_match[i]
                        if j2 < 0:
                            if dnil == INF:
                                dnil = dist[j] + 1
                        elif dist[j2] == INF:
                            dist[j2] = dist[j] + 1
                            queue.append(j2)
            if dnil == INF:
                break

            def dfs(j):
                for i in cols[j]:
                    j2 = row_match[i]
                    if (j2 < 0 and dnil == dist[j] + 1) or (j2 >= 0 and dist[j2] == dist[j] + 1 and dfs(j2)):
                        col_match[j] = i
                        row_match[i] = j
                        return True
                dist[j] = INF
                return False

            for j in range(n):
                if col_match[j] < 0:
                    dfs(j)
    finally:
        sys.setrecursionlimit(old)
    return col_match


def permuted_rows(n, row_ptr, col_idx, vals, q):
    """CSR of A_hat = A[q, :] (row j of A_hat = row q[j] of A) -> (row_ptr, col_idx, vals)."""
    import numpy as np
    rp, ci, v = [0], [], []
    for j in range(n):
        r = q[j]
        for t in range(int(row_ptr[r]), int(row_ptr[r + 1])):
            ci.append(int(col_idx[t]))
            v.append(float(vals[t]))
        rp.append(len(ci))
    return np.array(rp, np.int32), np.array(ci, np.int32), np.array(v)
