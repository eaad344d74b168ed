"""Seeded synthetic distributed-slack AC power-flow Jacobians (input tooling only).

This module is the ONE place both the CUDA path and the oracle take their inputs
from.  It holds none of the method's arithmetic (no perturbation, factorisation,
solve or recombination): it only builds the linear system the paper applies the
method to, as a stand-in for the PGLib 300-bus Newton-Raphson Jacobians of
PAPER.md §IV ("distributed slack AC power flow problem on the PGLib
300-bus test case ... J in R^{531x531}").  PGLib is not in this container, so the
recipe below (BASELINE.json configs) generates grids of the same
shape and structure; DESIGN.md §3 states the recipe.

Recipe:
  1. bus coordinates p_i ~ U([0,1]^2) from default_rng(seed);
  2. candidate edges = 8 nearest neighbours (symmetrised); random spanning tree by
     Kruskal over the candidates in random order; plus B-(N-1) extra candidate edges;
  3. r ~ U(.005,.05), x ~ U(.02,.3), b/2 ~ U(0,.05) per branch -> Ybus;
  4. generators = first n_gen of a random permutation; ref = lowest-index generator
     with a PQ neighbour; alpha_i = 1/n_gen on every generator (sum alpha = 1);
  5. V ~ U(.95,1.05), theta ~ N(0,.1), theta_ref = 0 (trial t re-draws these only);
  6. polar-form Jacobian; P rows for all buses carry -alpha_i in the lambda column;
  7. column alignment conventions: 'slack' (default, one structural zero diagonal),
     'listed' (the literal [theta_nonref; V_PQ; lambda] order, negative control);
     the 'leading-zero' stress regime is the slack matrix with the zero slot
     eliminated first (an ordering choice, made by the caller);
  8. b ~ N(0,1)^{n x R} from default_rng([seed,2]); d ~ N(0,1)^n from
     default_rng([seed,1]) normalised to max|d| = 1 ("||D||_1 = 1"; for a
     diagonal D the 1-norm is max|d_i|).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class PowerFlowSystem:
    n: int                      # matrix dimension
    row_ptr: np.ndarray         # int32 [n+1], CSR, column indices sorted per row
    col_idx: np.ndarray         # int32 [nnz]
    vals: np.ndarray            # float64 [nnz]
    d: np.ndarray               # float64 [n], diagonal of D, max|d| = 1
    b: np.ndarray               # float64 [n, R] (column j = RHS j)
    n_bus: int
    n_gen: int
    ref: int                    # reference bus
    slot_p: int                 # the structurally-zero diagonal slot (slack convention)
    convention: str
    n_struct_zero_diag: int
    aux: dict = dataclasses.field(default_factory=dict, repr=False)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def dense(self) -> np.ndarray:
        A = np.zeros((self.n, self.n))
        for i in range(self.n):
            for q in range(self.row_ptr[i], self.row_ptr[i + 1]):
                A[i, self.col_idx[q]] += self.vals[q]
        return A


def _grid(rng: np.random.Generator, N: int, n_branch: int):
    from scipy.spatial import cKDTree
    pts = rng.random((N, 2))
    tree_kd = cKDTree(pts)
    k = 8
    while True:
        kk = min(k, N - 1)
        _, nn = tree_kd.query(pts, k=kk + 1)
        cand = sorted({(min(i, int(j)), max(i, int(j))) for i in range(N) for j in nn[i, 1:] if j != i})
        order = rng.permutation(len(cand))
        parent = list(range(N))

        def find(a):
            while parent[a] != a:
                parent[a] = parent[parent[a]]
                a = parent[a]
            return a

        tree, rest = [], []
        for e in order:
            u, v = cand[e]
            ru, rv = find(u), find(v)
            if ru != rv:
                parent[ru] = rv
                tree.append(cand[e])
            else:
                rest.append(cand[e])
        if len(tree) == N - 1:
            break
        k += 2
    n_extra = n_branch - (N - 1)
    if n_extra > len(rest):
        raise ValueError("not enough candidate edges for the requested branch count")
    rest.sort()
    pick = rng.choice(len(rest), size=n_extra, replace=False) if n_extra > 0 else []
    edges = tree + [rest[i] for i in sorted(pick)]
    return sorted(edges)


def _ybus(rng, N, edges):
    """Sparse Ybus as scipy CSR (complex)."""
    import scipy.sparse as sp
    nb = len(edges)
    r = rng.uniform(0.005, 0.05, nb)
    x = rng.uniform(0.02, 0.3, nb)
    bh = rng.uniform(0.0, 0.05, nb)
    rows, cols, vals = [], [], []
    for e, (f, t) in enumerate(edges):
        y = 1.0 / complex(r[e], x[e])
        rows += [f, t, f, t]
        cols += [f, t, t, f]
        vals += [y + 1j * bh[e], y + 1j * bh[e], -y, -y]
    Y = sp.coo_matrix((np.array(vals), (np.array(rows), np.array(cols))), shape=(N, N)).tocsr()
    Y.sum_duplicates()
    Y.sort_indices()
    return Y


def power_injections(Y, V, th):
    """P_i, Q_i of the polar power-flow equations (used by the Jacobian and by the
    finite-difference test of the Jacobian)."""
    Vc = V * np.exp(1j * th)
    S = Vc * np.conj(Y @ Vc)
    return S.real, S.imag


def build_system(N: int, n_branch: int, n_gen: int, seed: int = 0, R: int = 1,
                 trial: int = 0, convention: str = "slack") -> PowerFlowSystem:
    """Generate one synthetic distributed-slack Jacobian J (and d, b)."""
    rng = np.random.default_rng(seed)
    edges = _grid(rng, N, n_branch)
    Y = _ybus(rng, N, edges)
    perm = rng.permutation(N)
    gens = np.sort(perm[:n_gen])
    is_gen = np.zeros(N, bool)
    is_gen[gens] = True
    adj = [set() for _ in range(N)]
    for f, t in edges:
        adj[f].add(t)
        adj[t].add(f)
    ref = next(g for g in gens if any(not is_gen[q] for q in adj[g]))
    pq = [i for i in range(N) if not is_gen[i]]
    slot_p = min(q for q in adj[ref] if not is_gen[q])
    alpha = np.where(is_gen, 1.0 / n_gen, 0.0)

    rng_op = np.random.default_rng([seed, 3, trial])
    V = rng_op.uniform(0.95, 1.05, N)
    th = rng_op.normal(0.0, 0.1, N)
    th[ref] = 0.0

    P, Q = power_injections(Y, V, th)
    Yc = Y.tocoo()
    # polar-form Jacobian entries on the Ybus pattern (G + jB = Ybus, th_ij = th_i - th_j)
    blocks = {}
    for i, j, y in zip(Yc.row.tolist(), Yc.col.tolist(), Yc.data.tolist()):
        G, B = y.real, y.imag
        if i == j:
            blocks[(i, j)] = (-Q[i] - B * V[i] ** 2,          # dP/dth
                              P[i] / V[i] + G * V[i],         # dP/dV
                              P[i] - G * V[i] ** 2,           # dQ/dth
                              Q[i] / V[i] - B * V[i])         # dQ/dV
        else:
            t = th[i] - th[j]
            c, s = math.cos(t), math.sin(t)
            blocks[(i, j)] = (V[i] * V[j] * (G * s - B * c),
                              V[i] * (G * c + B * s),
                              -V[i] * V[j] * (G * c + B * s),
                              V[i] * (G * s - B * c))

    n_pq = len(pq)
    n = N + n_pq
    # column of each unknown
    th_col = {}
    V_col = {bus: N + t for t, bus in enumerate(pq)}
    if convention == "slack":
        for i in range(N):
            if i not in (ref, slot_p):
                th_col[i] = i
        th_col[slot_p] = ref
        lam_col = slot_p
    elif convention == "listed":
        nonref = [i for i in range(N) if i != ref]
        for t, i in enumerate(nonref):
            th_col[i] = t
        V_col = {bus: (N - 1) + t for t, bus in enumerate(pq)}
        lam_col = N - 1 + n_pq
    else:
        raise ValueError(convention)
    rows_q = {bus: N + t for t, bus in enumerate(pq)}

    ent = {}

    def put(r, cidx, v):
        if v != 0.0:
            ent[(r, cidx)] = ent.get((r, cidx), 0.0) + float(v)

    for (i, j), (dPth, dPV, dQth, dQV) in sorted(blocks.items()):
        if j in th_col:
            put(i, th_col[j], dPth)
            if i in rows_q:
                put(rows_q[i], th_col[j], dQth)
        if j in V_col:
            put(i, V_col[j], dPV)
            if i in rows_q:
                put(rows_q[i], V_col[j], dQV)
    for i in range(N):
        if alpha[i] != 0.0:
            put(i, lam_col, -alpha[i])

    keys = sorted(ent)
    rows = np.array([k[0] for k in keys], dtype=np.int64)
    cols = np.array([k[1] for k in keys], dtype=np.int32)
    vals = np.array([ent[k] for k in keys], dtype=np.float64)
    row_ptr = np.zeros(n + 1, dtype=np.int32)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.int32)

    d = perturbation_diagonal(n, seed)
    rng_b = np.random.default_rng([seed, 2])
    b = rng_b.normal(0.0, 1.0, (R, n)).T.copy()

    diag_present = np.zeros(n, bool)
    for (r, cidx) in keys:
        if r == cidx:
            diag_present[r] = True
    return PowerFlowSystem(n=n, row_ptr=row_ptr, col_idx=cols, vals=vals, d=d, b=b,
                           n_bus=N, n_gen=n_gen, ref=int(ref), slot_p=int(slot_p),
                           convention=convention,
                           n_struct_zero_diag=int((~diag_present).sum()),
                           aux=dict(Y=Y, V=V, th=th, pq=pq, alpha=alpha, th_col=th_col,
                                    V_col=V_col, lam_col=lam_col, rows_q=rows_q))


def perturbation_diagonal(n: int, seed: int) -> np.ndarray:
    """D = diag(d), d_i ~ N(0,1) ("normally distributed"), scaled so that
    ||D||_1 = max|d_i| = 1."""
    rng_d = np.random.default_rng([seed, 1])
    d = rng_d.normal(0.0, 1.0, n)
    return d / np.max(np.abs(d))


# ----------------------------------------------------------------------------
# Perturbation ladders (input data: signed eps_k, lane order [+s1,-s1,+s2,-s2,...])
# ----------------------------------------------------------------------------

def ladder_eps(magnitudes) -> np.ndarray:
    """Signed lanes for one ladder: x_alpha^+ and x_alpha^- of Eqs.(5)-(6)
     for each magnitude s_j = alpha_j * eps."""
    out = []
    for s in magnitudes:
        out += [float(s), -float(s)]
    return np.array(out, dtype=np.float64)


def integer_ladder(eps: float, m: int) -> np.ndarray:
    """The paper's alpha = 1..m sequence at base eps: magnitudes j*eps."""
    return np.array([j * eps for j in range(1, m + 1)], dtype=np.float64)


@dataclasses.dataclass
class Workload:
    name: str
    N: int
    n_branch: int
    n_gen: int
    R: int
    ladders: list          # list of magnitude arrays (one per ladder)
    seed: int = 0

    @property
    def K(self) -> int:
        return 2 * sum(len(l) for l in self.ladders)

    def eps(self) -> np.ndarray:
        return np.concatenate([ladder_eps(l) for l in self.ladders])

    def system(self, convention="slack", trial=0) -> PowerFlowSystem:
        return build_system(self.N, self.n_branch, self.n_gen, self.seed, self.R, trial, convention)


def config(idx: int, n_ladders: int | None = None) -> Workload:
    """BASELINE.json configs (readings c1/c2/c14 of DESIGN.md)."""
    if idx == 0:
        # 14-bus, 20 branches, 3 PV + ref; eps geometric from 1e-2 ratio 1/2, K=4 (m=2)
        return Workload("cfg0-14bus", 14, 20, 4, 1, [np.array([1e-2, 5e-3])])
    if idx == 1:
        # 300-bus, 411 branches, 69 generators; paper ladder alpha=1..4 at eps=2e-3
        G = 1 if n_ladders is None else n_ladders
        return Workload("cfg1-300bus", 300, 411, 69, 1, [integer_ladder(2e-3, 4)] * G)
    if idx == 2:
        mags = np.geomspace(1e-1, 1e-8, 128)
        return Workload("cfg2-300bus-geo128", 300, 411, 69, 16, [mags])
    if idx == 3:
        G = 64 if n_ladders is None else n_ladders
        rng = np.random.default_rng([0, 4])
        base = 10.0 ** rng.uniform(-4, -2, G)
        return Workload("cfg3-2000bus", 2000, 2700, 400, 1, [integer_ladder(e, 8) for e in base])
    if idx == 4:
        G = 32 if n_ladders is None else n_ladders
        rng = np.random.default_rng([0, 5])
        base = 10.0 ** rng.uniform(-4, -2, G)
        return Workload("cfg4-10000bus", 10000, 13500, 2000, 4, [integer_ladder(e, 8) for e in base])
    raise ValueError(idx)
