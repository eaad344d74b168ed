"""GPU parity of the hybrid slot store of the capacity-planned factor
(PSP_OPT_FACTOR_HYBRID = 1: every warp keeps slots 0..63 in TMEM and 64..127 in shared
memory, or all 128 in TMEM when alone on its lane quarter; = 3: mixed lanes per thread, 4 TMEM
warps x 64 lanes + shared-memory warps x 32 lanes): factors, statuses and solutions
BITWISE those of the default capacity-planned launch (4 TMEM warps + 3 shared-memory
warps) and of the oracle on sampled lanes; full rounds (7 warps per CTA: partnered and
lone warps) and partial ones (fewer warps per CTA: all alone), fused and separate."""
import numpy as np
import pytest

import oracle
from psp_inputs import config, ladder_eps

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2311_11833_b200 import psp  # noqa: E402


def run(s, eps, hybrid, fused):
    sv = psp.Solver(0)
    sv.psp_set_option("coop", 2)
    sv.psp_set_option("coop_global", 2)
    sv.psp_set_option("factor_spill", 1)
    sv.psp_set_option("factor_hybrid", hybrid)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx)
    info, perm = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s.d)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    if fused:
        sv.psp_factor_solve_batch(A, b, 0.0)
    else:
        sv.psp_factor_batch(A, 0.0)
        sv.psp_solve_batch(b.reshape(1, -1))
    assert sv.psp_get_last_kernels()[0] == "batch_spill"
    X = sv.psp_get_solutions().cpu().numpy()
    rc, st = sv.psp_get_lane_status()
    return sv, info, perm, X, st


@pytest.mark.parametrize("mode", [1, 3])
@pytest.mark.parametrize("K,fused", [(1024, True), (20480, False), (65536, True)])
def test_hybrid_bitwise(K, fused, mode):
    s = config(1).system()
    rng = np.random.default_rng(K)
    G = K // 8
    eps = np.concatenate([ladder_eps([e * j for j in range(1, 5)]) for e in 10.0 ** rng.uniform(-3.3, -2.3, G)])
    sh, info, perm, Xh, sth = run(s, eps, mode, fused)
    sd, _, _, Xd, std = run(s, eps, 2, fused)
    assert np.array_equal(sth, std) and (sth == 0).all()
    assert np.array_equal(Xh, Xd)
    for k in sorted({0, 63, 64, K // 2, K - 1}):
        assert np.array_equal(sh.psp_get_factor(k, info["nnz_LU"]), sd.psp_get_factor(k, info["nnz_LU"]))
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    sample = np.unique(np.r_[0, 1, 447, 448, K // 2, K - 1])
    Xo, sto = oracle.SparseOracle(s, perm).batch(eps[sample], tol)
    assert np.array_equal(Xh[sample], Xo)
