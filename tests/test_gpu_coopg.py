"""GPU parity of the global-memory level-scheduled kernels (psp_coopg.cu; PSP_OPT_COOP_GLOBAL):
one CTA per perturbed system with its factor image in global memory, for the large systems
of SURVEY §8(d) configs 3-4 whose image does not fit shared memory.  Same etree-level
schedule as the cooperative kernels, so every entry keeps its canonical update order (R11):
per-lane solutions, factors and statuses BITWISE equal to the oracle and to the batch
kernels; recovered x within 1e-10."""
import numpy as np
import pytest

import oracle
from oracle import ordering
from psp_inputs import build_system, config

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2311_11833_b200 import psp  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def run(s, eps, B, tol, coopg, coop=2, first=-1):
    sv = psp.Solver(0)
    sv.psp_set_option("coop", coop)
    sv.psp_set_option("coop_global", coopg)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg_first" if first >= 0 else "mindeg",
                            first_node=first)
    info, perm = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s.d)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    sv.psp_factor_batch(A, tol)
    sv.psp_solve_batch(torch.tensor(B.T.copy(), dtype=torch.float64, device="cuda"))
    X = sv.psp_get_solutions().cpu().numpy()
    rc, st = sv.psp_get_lane_status()
    return sv, info, perm, X, st


@pytest.mark.parametrize("K", [1, 37, 100])
@pytest.mark.parametrize("first", [False, True])
def test_coopg_forced_bitwise_vs_oracle_and_batch(K, first):
    # the 300-bus system (coop would fit; forced off): ragged K, multi-RHS, the leading-zero
    # order with an unperturbed lane (step-0 zero pivot)
    s = build_system(300, 411, 69, seed=0, R=3)
    rng = np.random.default_rng(K)
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-6, -2, K)
    fn = s.slot_p if first else -1
    if first:
        eps[0] = 0.0
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    sv, info, perm, X, st = run(s, eps, s.b, tol, coopg=1, first=fn)
    assert sv.psp_get_last_kernels() == ("coop_global", False, "coop_global", True)
    so = oracle.SparseOracle(s, perm)
    Xo, sto = so.batch(eps, tol)
    assert np.array_equal(st, sto)
    ok = sto == 0
    assert np.array_equal(X[ok], Xo[ok])
    if first:
        assert st[0] == 1
    svb, _, _, Xb, stb = run(s, eps, s.b, tol, coopg=2, first=fn)   # batch kernels
    assert svb.psp_get_last_kernels()[0] != "coop_global"
    assert np.array_equal(stb, st) and np.array_equal(Xb[ok], X[ok])
    for k in sorted({0, K // 2, K - 1}):   # the factor itself, entry by entry (lane-major image)
        if ok[k]:
            assert np.array_equal(sv.psp_get_factor(k, info["nnz_LU"]), svb.psp_get_factor(k, info["nnz_LU"]))


def test_cfg3_automatic_coopg_sampled():
    # BASELINE configs[3] (n = 3600, K = 1024): the automatic choice is the global-memory
    # level-scheduled path; sampled lanes and two ladders' recovered x against the oracle
    w = config(3)
    s = w.system()
    eps = w.eps()
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    sv = psp.Solver(0)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx)
    info, perm = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s.d)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    sv.psp_factor_solve_batch(A, b, tol)
    assert sv.psp_get_last_kernels()[0] == "coop_global"
    sv.psp_set_weights(*psp.ladder_weights_csr(w.ladders))
    xh = sv.psp_recover().cpu().numpy()
    X = sv.psp_get_solutions().cpu().numpy()
    rc, st = sv.psp_get_lane_status()
    assert rc == 0 and (st == 0).all()
    K = len(eps)
    sample = np.unique(np.r_[0, 1, 31, 32, K // 2, K - 1])
    so = oracle.SparseOracle(s, perm)
    Xo, _ = so.batch(eps[sample], tol)
    assert np.array_equal(X[sample], Xo)
    for gi in [0, len(w.ladders) - 1]:
        lanes = np.arange(16 * gi, 16 * gi + 16)
        Xl, _ = so.batch(eps[lanes], tol)
        xo = oracle.combine(oracle.ladder_weight_matrix([w.ladders[gi]]), Xl)
        assert rel(xh[gi], xo[0]) <= 1e-10
