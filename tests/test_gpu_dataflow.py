"""GPU parity of the fused dataflow factor + solve (psp_dataflow.cu; PSP_OPT_DATAFLOW): the
latency path of BASELINE configs[1].  Tasks keep the canonical per-value order, so the
per-lane solutions, factors and statuses are BITWISE those of the cooperative kernels and
of the oracle (configs 0-1, ragged K, the leading-zero order with an unperturbed lane
failing at pivot 0, several right-hand-side vectors in turn)."""
import numpy as np
import pytest

import oracle
from oracle import ordering
from psp_inputs import build_system, config

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2311_11833_b200 import psp  # noqa: E402


def run(s, eps, b, tol, df, first=-1):
    sv = psp.Solver(0)
    sv.psp_set_option("dataflow", 1 if df == 0 else df)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg_first" if first >= 0 else "mindeg",
                            first_node=first)
    info, perm = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s.d)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    sv.psp_factor_solve_batch(A, torch.tensor(b, dtype=torch.float64, device="cuda"), tol)
    X = sv.psp_get_solutions().cpu().numpy()
    rc, st = sv.psp_get_lane_status()
    return sv, info, perm, X, st


@pytest.mark.parametrize("ci,K,first", [(0, 4, False), (1, 8, False), (1, 8, True), (1, 37, True), (1, 300, False)])
def test_dataflow_bitwise_vs_coop_and_oracle(ci, K, first):
    s = config(ci).system()
    rng = np.random.default_rng(K + ci)
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-6, -2, K)
    fn = s.slot_p if first else -1
    if first:
        eps[0] = 0.0
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    b = s.b[:, 0].copy()
    sv, info, perm, X, st = run(s, eps, b, tol, 0, fn)
    sc, _, _, Xc, stc = run(s, eps, b, tol, 2, fn)
    if sc.psp_get_last_kernels()[0] == "coop":     # (dataflow accompanies the coop kernels)
        assert sv.psp_get_last_kernels() == ("dataflow", True, "dataflow", False)
    assert np.array_equal(st, stc)
    ok = st == 0
    assert np.array_equal(X[ok], Xc[ok])
    for k in sorted({0, K // 2, K - 1}):
        if ok[k]:
            assert np.array_equal(sv.psp_get_factor(k, info["nnz_LU"]), sc.psp_get_factor(k, info["nnz_LU"]))
    Xo, sto = oracle.SparseOracle(s, perm).batch(eps, tol)
    assert np.array_equal(st, sto)
    assert np.array_equal(X[ok], Xo[ok])
    if first:
        assert st[0] == 1
    # the same handle solves more right-hand sides with the factor the dataflow kernel wrote
    B2 = build_system(s.n_bus, 411 if ci else 20, s.n_gen, seed=0, R=3).b if ci else np.random.default_rng(1).normal(size=(s.n, 3))
    sv.psp_solve_batch(torch.tensor(B2.T.copy(), dtype=torch.float64, device="cuda"))
    X2 = sv.psp_get_solutions().cpu().numpy()
    Xo2, _ = oracle.SparseOracle(s, perm).batch(eps, tol, B=B2)
    assert np.array_equal(X2[ok], Xo2[ok])
