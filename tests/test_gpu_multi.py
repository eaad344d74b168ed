"""many Jacobians of one pattern in one launch (the 25 voltage starts of
P:L302 / Fig. 1's 25 trials) and the Fig. 1 study on the GPU from a single batch.

25 synthetic 300-bus Jacobians (the operating point re-drawn per trial, pattern shared)
x the paper's alpha = 1..4 ladder at eps = 2e-3 = 200 lanes in one
psp_factor_batch_multi + psp_solve_batch_multi; per trial four recovered solutions (m = 1..4
pairs: the first 2m lanes of the trial's ladder, Remark 2 weights) = 100 weight rows, one
psp_recover.  Per-lane solutions and statuses BITWISE equal to the oracle (each trial's own
A and tolerance), recovered x within 1e-10 of oracle.combine, and the error-vs-m curve
||J x_hat - b|| (Alg. 1's error test) decreasing with m as Fig. 1 shows."""
import numpy as np
import pytest

import oracle
from oracle import ordering, weights
from psp_inputs import config, ladder_eps

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2311_11833_b200 import psp  # noqa: E402

N_TRIALS = 25
MAGS = [2e-3 * j for j in range(1, 5)]


def trial_systems(n_t=N_TRIALS):
    ss = [config(1).system(trial=t) for t in range(n_t)]
    for s in ss[1:]:
        assert np.array_equal(s.row_ptr, ss[0].row_ptr) and np.array_equal(s.col_idx, ss[0].col_idx)
    return ss


def weights_csr(n_t):
    ptr, lane, val = [0], [], []
    for t in range(n_t):
        for m in range(1, 5):
            w = weights.lane_weights(MAGS[:m])
            for j, c in enumerate(w):
                lane.append(8 * t + j)
                val.append(float(c))
            ptr.append(len(lane))
    return np.array(ptr, np.int32), np.array(lane, np.int32), np.array(val)


@pytest.mark.parametrize("path", ["sparse", "dense"])
def test_multi_jacobian_batch_and_fig1_curve(path):
    ss = trial_systems()
    s0 = ss[0]
    n_t = len(ss)
    eps8 = ladder_eps(MAGS)
    eps = np.tile(eps8, n_t)
    sv = psp.Solver(0)
    sv.psp_set_option("path", path)
    sv.psp_symbolic_analyse(s0.n, s0.row_ptr, s0.col_idx)
    info, perm = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s0.d)
    A = torch.tensor(np.stack([s.vals for s in ss]), dtype=torch.float64, device="cuda")
    B = torch.tensor(np.stack([s.b.T for s in ss]), dtype=torch.float64, device="cuda")   # [n_t, R, n]
    sv.psp_factor_batch_multi(A, 0.0)
    sv.psp_solve_batch_multi(B)
    kernels = sv.psp_get_last_kernels()
    assert kernels[0] == ("dense" if path == "dense" else "coop")
    wp, wl, wv = weights_csr(n_t)
    sv.psp_set_weights(wp, wl, wv)
    xh = sv.psp_recover().cpu().numpy()              # [4 n_t, 1, n]
    X = sv.psp_get_solutions().cpu().numpy()
    rc, st = sv.psp_get_lane_status()
    assert rc == 0 and (st == 0).all()
    operm = ordering.elimination_order(s0.n, s0.row_ptr, s0.col_idx)
    assert np.array_equal(perm, operm)
    res = np.empty((n_t, 4))
    for t, s in enumerate(ss):
        tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
        Xo, sto = oracle.dense_batch(s, operm, eps8, tol)
        assert (sto == 0).all()
        assert np.array_equal(X[8 * t:8 * t + 8], Xo)                  # bitwise per lane
        Wm = np.zeros((4, 8))
        for m in range(1, 5):
            Wm[m - 1, :2 * m] = weights.lane_weights(MAGS[:m])
        xo = oracle.combine(Wm, Xo)
        got = xh[4 * t:4 * t + 4]
        assert np.linalg.norm(got - xo) <= 1e-10 * np.linalg.norm(xo)
        res[t] = oracle.residual(s, got)[:, 0] / np.linalg.norm(s.b[:, 0])
    med = np.median(res, axis=0)
    # Fig. 1: the error falls with every added pair until the rounding floor
    for m in range(3):
        assert med[m + 1] < med[m] or med[m + 1] < 1e-11, med


def test_multi_jacobian_rejected_on_large_batch_kernels():
    s = config(1).system()
    sv = psp.Solver(0)
    sv.psp_set_option("coop", 2)
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx)
    sv.psp_set_perturbations(np.tile(ladder_eps(MAGS), 4), s.d)
    A = torch.tensor(np.stack([s.vals] * 2), dtype=torch.float64, device="cuda")
    with pytest.raises(psp.PSPError):
        sv.psp_factor_batch_multi(A, 0.0)
    with pytest.raises(ValueError):
        sv.psp_factor_batch_multi(A[0], 0.0)
