"""GPU parity of the dense path (PSP_OPT_PATH = dense; psp_dense.cu: the paper's dense
no-pivot getrf/trsm formulation, with DMMA trailing updates) and of the
general (dense) perturbation matrix D against the CPU oracle.

One DMMA.8x8x4 is exactly four chained fmas in its k order (measured on the B200,
tools/probe/fp64mma.cu; R19), so the blocked dense path keeps the canonical
per-entry order (R11): factors, per-lane solutions and statuses are asserted BITWISE
equal to the oracle's (the BASELINE bar is 1e-11 relative); recovered x within 1e-10."""
import numpy as np
import pytest

import oracle
from oracle import ordering
from psp_inputs import config, ladder_eps

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2311_11833_b200 import psp  # noqa: E402

U = np.finfo(np.float64).eps


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def dense_run(s, eps, ordering_kind="mindeg", first=-1, tol=0.0, B=None, ladders=None, Dm=None,
              path="dense"):
    sv = psp.Solver(0)
    sv.psp_set_option("path", path)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering=ordering_kind, first_node=first)
    info, perm = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s.d)
    if Dm is not None:
        sv.psp_set_perturbation_matrix(Dm)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    sv.psp_factor_batch(A, tol)
    Bm = s.b if B is None else B
    sv.psp_solve_batch(torch.tensor(Bm.T.copy(), dtype=torch.float64, device="cuda"))
    X = sv.psp_get_solutions().cpu().numpy()
    xh = None
    if ladders is not None:
        sv.psp_set_weights(*psp.ladder_weights_csr(ladders))
        xh = sv.psp_recover().cpu().numpy()
    rc, st = sv.psp_get_lane_status()
    return dict(perm=perm, X=X, xhat=xh, status=st, rc=rc, solver=sv,
                kernels=sv.psp_get_last_kernels())


def check_lanes(X, Xo, st):
    ok = st == 0
    assert np.array_equal(X[ok], Xo[ok])          # bitwise per lane


@pytest.mark.parametrize("ci", [0, 1])
@pytest.mark.parametrize("order", ["mindeg", "natural", "mindeg_first"])
def test_dense_path_vs_oracle(ci, order):
    w = config(ci)
    s = w.system()
    first = s.slot_p if order == "mindeg_first" else -1
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    eps = w.eps()
    g = dense_run(s, eps, order, first, tol, ladders=w.ladders)
    assert g["kernels"][0] == "dense" and g["kernels"][2] == "dense"
    operm = np.arange(s.n, dtype=np.int32) if order == "natural" else \
        ordering.elimination_order(s.n, s.row_ptr, s.col_idx, first=None if first < 0 else first)
    assert np.array_equal(g["perm"], operm)
    Xo, sto = oracle.dense_batch(s, operm, eps, tol)
    assert np.array_equal(g["status"], sto) and (sto == 0).all()
    assert np.array_equal(g["X"], Xo)
    xo = oracle.combine(oracle.ladder_weight_matrix(w.ladders), Xo)
    assert rel(g["xhat"], xo) <= 1e-10


def test_dense_factor_vs_oracle_lu():
    # the factor itself: P (A + eps D) P^T = L U entry by entry against OR1's lu_nopivot
    s = config(1).system()
    perm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx)
    eps = np.array([2e-3, -2e-3, 8e-3])
    g = dense_run(s, eps, tol=1e-300)
    A = s.dense()
    for k, e in enumerate(eps):
        Ak = A + e * np.diag(s.d)
        LUo, sto = oracle.lu_nopivot(Ak[np.ix_(perm, perm)], 1e-300)
        assert sto == 0
        LU = g["solver"].psp_get_dense_factor(k)
        assert np.array_equal(LU, LUo)          # every entry of L and U, bitwise


@pytest.mark.parametrize("K", [1, 5, 33, 70])
def test_dense_ragged_batches_and_unperturbed_failure(K):
    # ragged K; lane 0 unperturbed in the leading-zero order fails at pivot 0
    s = config(1).system()
    rng = np.random.default_rng(K)
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-5, -2, K)
    eps[0] = 0.0
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    g = dense_run(s, eps, "mindeg_first", s.slot_p, tol)
    operm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx, first=s.slot_p)
    Xo, sto = oracle.SparseOracle(s, operm).batch(eps, tol)
    assert sto[0] == 1 and g["status"][0] == 1
    assert np.array_equal(g["status"], sto)
    check_lanes(g["X"], Xo, g["status"])


def test_dense_vs_sparse_cfg2_multi_rhs():
    # BASELINE configs[2]: K = 256 geometric 1e-1..1e-8 magnitudes (128 +- pairs) x R = 16;
    # the dense path against the (bitwise-canonical) sparse path on every lane, and
    # sampled lanes against the oracle
    w = config(2)
    s = w.system()
    eps = w.eps()
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    gd = dense_run(s, eps, tol=tol)
    gs = dense_run(s, eps, tol=tol, path="sparse")
    assert gs["kernels"][0] != "dense"
    assert np.array_equal(gd["status"], gs["status"])
    operm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx)
    check_lanes(gd["X"], gs["X"], gd["status"])     # both paths canonical: bitwise
    sample = [0, 1, 77, 200, 254, 255]
    Xo, sto = oracle.dense_batch(s, operm, eps[sample], tol, B=s.b)
    assert np.array_equal(gd["status"][sample], sto)
    check_lanes(gd["X"][sample], Xo, sto)


def _normal_D(n, seed):
    rng = np.random.default_rng(seed)
    D = rng.normal(size=(n, n))
    return D / np.abs(D).sum(axis=0).max()          # ||D||_1 = 1


@pytest.mark.parametrize("ci", [0, 1])
def test_dense_D_vs_oracle_and_truncation_error(ci):
    # a dense normally distributed D (P:L314's reading; footnote P:L72): lanes against
    # oracle.dense_D_batch, recovered x against the oracle's, and against x* within the
    # predicted truncation error (I3) with this D (tolerance policy 3)
    w = config(ci)
    s = w.system()
    D = _normal_D(s.n, 314 + ci)
    mags = [2e-3 * j for j in range(1, 4)]
    ladders = [mags]
    eps = ladder_eps(mags)
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    g = dense_run(s, eps, tol=tol, ladders=ladders, Dm=D)
    perm = g["perm"]
    Xo, sto = oracle.dense_D_batch(s.dense(), D, perm, eps, tol, s.b)
    assert np.array_equal(g["status"], sto) and (sto == 0).all()
    assert np.array_equal(g["X"], Xo)               # bitwise per lane
    Wm = oracle.ladder_weight_matrix(ladders)
    xo = oracle.combine(Wm, Xo)
    assert rel(g["xhat"], xo) <= 1e-10
    xs, _ = oracle.reference_solve(s)
    e = oracle.predicted_error(s, mags, Dm=D)[0]
    piv = np.array([np.linalg.solve(s.dense() + e_ * D, s.b[:, 0]) for e_ in eps])
    floor = 10 * np.abs(Wm).sum() * max(np.linalg.norm(Xo[k, 0] - piv[k]) for k in range(len(eps)))
    assert np.linalg.norm(xs[0] - g["xhat"][0, 0]) <= 1.5 * np.linalg.norm(e) + floor


def test_dense_D_tiny_exact():
    # zero-diagonal 5x5, dyadic dense D: per lane against exact rational solves
    from fractions import Fraction
    from test_oracle_solve import _Tiny, cramer, tiny_zero_diag_system
    from test_oracle_dense_d import _dense_dyadic_D
    A, d, b = tiny_zero_diag_system(2)
    s = _Tiny(A, d, b)
    D = _dense_dyadic_D(2)
    eps = np.array([1 / 16, -1 / 16, 1 / 32, -1 / 32])
    g = dense_run(s, eps, "natural", tol=1e-300, Dm=D)
    for k, e in enumerate(eps):
        M = [[Fraction(A[i, j]) + Fraction(e) * Fraction(D[i, j]) for j in range(5)] for i in range(5)]
        assert g["status"][k] == 0
        x = np.array([float(v) for v in cramer(M, [Fraction(v) for v in b])])
        assert rel(g["X"][k, 0], x) <= 1e-12


def test_dense_D_rejected_on_sparse_path():
    s = config(0).system()
    sv = psp.Solver(0)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx)
    sv.psp_set_perturbations(config(0).eps(), s.d)
    sv.psp_set_perturbation_matrix(np.eye(s.n))
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    with pytest.raises(psp.PSPError):
        sv.psp_factor_batch(A, 0.0)
    sv.psp_set_perturbation_matrix(None)          # back to diag(d): the sparse path runs
    sv.psp_factor_batch(A, 0.0)
    sv.psp_set_option("path", "dense")
    sv.psp_factor_batch(A, 0.0)
    with pytest.raises(psp.PSPError):
        sv.psp_get_factor(0, 10)                  # the sparse layout does not exist


def test_dense_many_rhs_and_size_limit():
    # R = 21 right-hand sides (two 16-column passes, the second ragged) bitwise vs the
    # oracle; an n beyond the panel's shared memory (N x 33 x 8 B > 227 KB) is refused
    # with PSP_ERR_UNSUPPORTED, never computed wrongly
    s = config(0).system()
    rng = np.random.default_rng(21)
    B = rng.normal(size=(s.n, 21))
    eps = np.array([1e-2, -1e-2, 3e-3])
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    g = dense_run(s, eps, tol=tol, B=B)
    perm = g["perm"]
    Xo, sto = oracle.dense_batch(s, perm, eps, tol, B=B)
    assert (sto == 0).all() and np.array_equal(g["X"], Xo)
    big = config(3).system()               # n = 3600 -> N = 3616: 954 KB panel
    sv = psp.Solver(0)
    sv.psp_set_option("path", "dense")
    sv.psp_symbolic_analyse(big.n, big.row_ptr, big.col_idx)
    sv.psp_set_perturbations(np.array([1e-3]), big.d)
    with pytest.raises(psp.PSPError) as e:
        sv.psp_factor_batch(torch.tensor(big.vals, dtype=torch.float64, device="cuda"), 0.0)
    assert e.value.status == 8
