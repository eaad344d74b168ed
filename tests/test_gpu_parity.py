"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element on the same seeded inputs.

Bar (BASELINE north_star): per-lane solutions within 1e-11 relative
— the kernels keep the canonical operation order, so they are asserted BITWISE
equal; recovered x within 1e-10 relative of the oracle's recovered x; statuses
(integers) bit-exact.  Sizes: the oracle runs every lane where it finishes in
seconds (configs 0-1, ragged K), sampled lanes at the full BASELINE sizes."""
import os

import numpy as np
import pytest

import oracle
from oracle import ordering
from psp_inputs import config, ladder_eps

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2311_11833_b200 import psp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gpu_run(s, eps, ordering_kind="mindeg", first=-1, tol=0.0, B=None, ladders=None,
            w_csr=None, lanes_out=True, coop=None):
    solver = psp.Solver(0)
    if coop is not None:
        solver.psp_set_option("coop", coop)
        if coop == 2:
            solver.psp_set_option("coop_global", 2)
    solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering=ordering_kind, first_node=first)
    info, perm = solver.psp_get_symbolic_info()
    # the oracle's own elimination order (never the product's): integer parity
    if ordering_kind == "natural":
        operm = np.arange(s.n, dtype=np.int32)
    else:
        operm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx, first=None if first < 0 else first)
    assert np.array_equal(perm, operm)
    solver.psp_set_perturbations(eps, s.d)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    st = torch.empty(len(eps), dtype=torch.int32, device="cuda")
    solver.psp_factor_batch(A, tol, st)
    Bt = torch.tensor((s.b if B is None else B).T.copy(), dtype=torch.float64, device="cuda")
    solver.psp_solve_batch(Bt)
    X = solver.psp_get_solutions() if lanes_out else None
    xh = None
    if ladders is not None or w_csr is not None:
        wp, wl, wv = w_csr if w_csr is not None else psp.ladder_weights_csr(ladders)
        solver.psp_set_weights(wp, wl, wv)
        xh = solver.psp_recover()
    torch.cuda.synchronize()
    rc, st_h = solver.psp_get_lane_status()
    out = dict(perm=perm, operm=operm, info=info, status=st.cpu().numpy(), status_h=st_h, rc=rc,
               X=None if X is None else X.cpu().numpy(),
               xhat=None if xh is None else xh.cpu().numpy(), solver=solver)
    return out


def oracle_perm(s, first):
    return ordering.elimination_order(s.n, s.row_ptr, s.col_idx, first=None if first < 0 else first)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("ci", [0, 1])
@pytest.mark.parametrize("leading_zero", [False, True])
def test_full_parity_small_configs(ci, leading_zero):
    w = config(ci)
    s = w.system()
    first = s.slot_p if leading_zero else -1
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    eps = w.eps()
    g = gpu_run(s, eps, "mindeg_first" if leading_zero else "mindeg", first, tol, ladders=w.ladders)
    perm = oracle_perm(s, first)
    assert np.array_equal(g["perm"], perm)
    Xo, sto = oracle.dense_batch(s, perm, eps, tol)
    assert np.array_equal(g["status"], sto) and np.array_equal(g["status_h"], sto)
    assert (sto == 0).all()
    assert np.array_equal(g["X"], Xo)                                   # bitwise per lane
    xo = oracle.combine(oracle.ladder_weight_matrix(w.ladders), Xo)
    assert rel(g["xhat"], xo) <= 1e-10
    xs, _ = oracle.reference_solve(s)
    assert rel(g["xhat"][0, 0], xs[0]) <= 1e-9                        # truncation + rounding


@pytest.mark.parametrize("K", [1, 5, 37, 64, 100])
def test_ragged_batches(K):
    s = config(1).system()
    rng = np.random.default_rng(K)
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-6, -1, K)
    tol = 1e-14
    g = gpu_run(s, eps, tol=tol)
    Xo, sto = oracle.dense_batch(s, g["operm"], eps, tol) if K <= 40 else \
        oracle.SparseOracle(s, g["operm"]).batch(eps, tol)
    assert np.array_equal(g["status"], sto)
    ok = sto == 0
    assert np.array_equal(g["X"][ok], Xo[ok])


def test_multi_rhs_and_leading_zero_extreme_eps():
    from psp_inputs import build_system
    s = build_system(300, 411, 69, seed=0, R=3)
    eps = np.array([1e-2, -1e-2, 1e-4, -1e-4, 1e-6, -1e-6, 1e-8, -1e-8])
    tol = 1e-300
    g = gpu_run(s, eps, "mindeg_first", s.slot_p, tol)
    Xo, sto = oracle.SparseOracle(s, g["operm"]).batch(eps, tol)
    assert np.array_equal(g["status"], sto)
    assert np.array_equal(g["X"], Xo)      # bitwise even where growth ~1/eps (DESIGN R11)


def test_failure_modes():
    w = config(1)
    s = w.system()
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    # unperturbed pivot-free solve hits a leading zero -> status 1 (step 0)
    eps = np.r_[0.0, w.eps()]
    g = gpu_run(s, eps, "mindeg_first", s.slot_p, 0.0, ladders=None)
    assert g["status"][0] == 1 and (g["status"][1:] == 0).all()
    assert g["rc"] == psp.PSP_ERR_ZERO_PIVOT
    # a non-zero weight on the failed lane -> BATCH_INFEASIBLE and NaN
    wp = np.array([0, 2, 4], np.int32)
    wl = np.array([0, 1, 1, 2], np.int32)
    wv = np.array([0.5, 0.5, 0.5, 0.5])
    g = gpu_run(s, eps, "mindeg_first", s.slot_p, 0.0, w_csr=(wp, wl, wv))
    assert g["rc"] == psp.PSP_ERR_BATCH_INFEASIBLE
    assert np.isnan(g["xhat"][0]).all() and np.isfinite(g["xhat"][1]).all()
    # literal variable order (negative control): statuses equal the oracle's
    sl = w.system(convention="listed")
    eps2 = np.array([0.0, 2e-3, -2e-3])
    g = gpu_run(sl, eps2, "natural", -1, tol)
    _, sto = oracle.SparseOracle(sl, np.arange(sl.n, dtype=np.int32)).batch(eps2, tol)
    assert np.array_equal(g["status"], sto) and g["status"][0] != 0


@pytest.mark.parametrize("L", [2, 4, 8, 16])
def test_uniform_ladder_recover_matches_general_path(L):
    """Row w = lanes [w*L, w*L+L) takes recover_uni_kernel; appending an empty row makes
    the same weights non-uniform (recover_seg_kernel).  Both bitwise equal, within 1e-10
    of the oracle's combination, NaN + BATCH_INFEASIBLE on the rows holding a failed
    lane."""
    w = config(1)
    s = w.system()
    rng = np.random.default_rng(70 + L)
    K = 6 * 32 + L  # several blocks, ragged tail
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-4, -2, K)
    eps[L + 1] = 0.0  # unperturbed lane with a leading zero pivot: fails
    W = K // L
    wv = rng.normal(size=W * L)
    wp = np.arange(W + 1, dtype=np.int32) * L
    wl = np.arange(W * L, dtype=np.int32)
    B = np.stack([s.b[:, 0], rng.normal(size=s.n)], axis=1)
    g = gpu_run(s, eps, "mindeg_first", s.slot_p, 0.0, B=B, w_csr=(wp, wl, wv))
    solver = g["solver"]
    solver.psp_set_weights(np.r_[wp, wp[-1]].astype(np.int32), wl, wv)
    xg = solver.psp_recover().cpu().numpy()
    solver.close()
    xu = g["xhat"]
    assert xu.shape == (W, 2, s.n) and xg.shape == (W + 1, 2, s.n)
    assert np.array_equal(xu, xg[:W], equal_nan=True) and (xg[W] == 0).all()
    assert g["rc"] == psp.PSP_ERR_BATCH_INFEASIBLE
    Xo, sto = oracle.SparseOracle(s, g["operm"]).batch(eps, 0.0, B)
    assert np.array_equal(g["status"], sto) and sto[L + 1] != 0
    Wm = np.zeros((W, K))
    for r in range(W):
        Wm[r, r * L:(r + 1) * L] = wv[r * L:(r + 1) * L]
    bad = 1  # row holding lane L+1
    assert np.isnan(xu[bad]).all() and np.isfinite(np.delete(xu, bad, axis=0)).all()
    xo = oracle.combine(np.delete(Wm, bad, axis=0), np.nan_to_num(Xo))
    assert rel(np.delete(xu, bad, axis=0), xo) <= 1e-10


@pytest.mark.parametrize("L", [2, 4, 8, 16])
def test_block_recover_small_system(L):
    """recover_blk_kernel on the 14-bus system (n = 24: every L fits its shared-memory
    un-permute area, L = 2 included, which the 300-bus test above leaves to the gather
    kernel), three right-hand sides, a last 32-lane block that is only partly covered by
    weight rows: bitwise equal to the general path (the same weights made non-uniform by
    an empty row), within 1e-10 of the oracle's combination (Alg. 1 steps 3-4)."""
    w = config(0)
    s = w.system()
    rng = np.random.default_rng(170 + L)
    K = 3 * 32 + L
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-4, -2, K)
    W = K // L
    wv = rng.normal(size=W * L)
    wp = np.arange(W + 1, dtype=np.int32) * L
    wl = np.arange(W * L, dtype=np.int32)
    B = np.stack([s.b[:, 0], rng.normal(size=s.n), rng.normal(size=s.n)], axis=1)
    g = gpu_run(s, eps, "mindeg", -1, 0.0, B=B, w_csr=(wp, wl, wv))
    solver = g["solver"]
    solver.psp_set_weights(np.r_[wp, wp[-1]].astype(np.int32), wl, wv)
    xg = solver.psp_recover().cpu().numpy()
    solver.close()
    xu = g["xhat"]
    assert g["rc"] == 0 and (g["status"] == 0).all()
    assert xu.shape == (W, 3, s.n) and np.array_equal(xu, xg[:W]) and (xg[W] == 0).all()
    Xo, sto = oracle.SparseOracle(s, g["operm"]).batch(eps, 0.0, B)
    assert (sto == 0).all() and np.array_equal(g["X"], Xo)
    Wm = np.zeros((W, K))
    for r in range(W):
        Wm[r, r * L:(r + 1) * L] = wv[r * L:(r + 1) * L]
    assert rel(xu, oracle.combine(Wm, Xo)) <= 1e-10


@pytest.mark.parametrize("ci", [0, 1])
def test_residual_matches_oracle(ci):
    """psp_residual (a7) on the recovered rows, a zero row (-> ||b||) and a NaN
    row, two right-hand sides: within 1e-12 (||A|| ||x|| + ||b||) of the oracle's
    row-by-row residual; the recovered solutions' residuals are small (the method's
    O(eps^2m) accuracy)."""
    w = config(ci)
    s = w.system()
    rng = np.random.default_rng(90 + ci)
    B = np.stack([s.b[:, 0], rng.normal(size=s.n)], axis=1)
    g = gpu_run(s, w.eps(), B=B, ladders=w.ladders)
    assert (g["status"] == 0).all()
    solver = g["solver"]
    xh = torch.tensor(g["xhat"], dtype=torch.float64, device="cuda")
    extra = torch.zeros((2, 2, s.n), dtype=torch.float64, device="cuda")
    extra[1, :, 3] = float("nan")
    x = torch.cat([xh, extra]).contiguous()
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    Bt = torch.tensor(B.T.copy(), dtype=torch.float64, device="cuda")
    res = solver.psp_residual(A, Bt, x)
    solver.close()
    xc = x.cpu().numpy()
    W = xh.shape[0]
    ro = oracle.residual(s, xc[:W + 1], B)
    anorm = np.abs(s.vals).sum()
    for wi in range(W + 1):
        for r in range(2):
            scale = anorm * np.linalg.norm(xc[wi, r]) + np.linalg.norm(B[:, r])
            assert abs(res[wi, r] - ro[wi, r]) <= 1e-12 * scale
    assert np.allclose(res[W], np.linalg.norm(B, axis=0), rtol=1e-14, atol=0)
    assert np.isnan(res[W + 1]).all()
    assert (res[:W, 0] <= 1e-6 * np.linalg.norm(B[:, 0])).all()


@pytest.mark.parametrize("ci", [0, 1])
def test_rescale_failed_ladders(ci):
    """SURVEY 8(f) 1 re-perturbation: with the zero-diagonal slot eliminated first its
    pivot is eps_k d exactly, so an absolute tolerance fails the small-eps lanes; every
    ladder holding a failed lane is rescaled by 20 (Remark 2 weights are scale-invariant),
    refactored, and then statuses equal the oracle's on the new eps (bit-exact) and the
    recovered x is within 1e-10 of the oracle's combination."""
    w = config(ci)
    s = w.system()
    ladders = [np.array([1e-4, 2e-4]), np.array([2e-3, 4e-3]), np.array([5e-4, 3e-3]),
               np.array([3e-3, 6e-3, 9e-3])]
    eps = np.concatenate([ladder_eps(m) for m in ladders])
    dslot = abs(s.d[s.slot_p])
    tol = 1.5e-3 * dslot
    solver = psp.Solver(0)
    solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg_first", first_node=s.slot_p)
    info, perm = solver.psp_get_symbolic_info()
    operm = oracle_perm(s, s.slot_p)
    assert np.array_equal(perm, operm)
    solver.psp_set_perturbations(eps, s.d)
    wp, wl, wv = psp.ladder_weights_csr(ladders)
    solver.psp_set_weights(wp, wl, wv)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    Bt = torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda")
    st = torch.empty(len(eps), dtype=torch.int32, device="cuda")
    solver.psp_factor_batch(A, tol, st)
    st0 = st.cpu().numpy()
    _, sto = oracle.SparseOracle(s, operm).batch(eps, tol)
    assert np.array_equal(st0, sto) and (st0 != 0).any() and (st0 == 0).any()
    # expected new eps, from the statuses and the ladder rows (lanes [wp[r], wp[r+1]))
    exp = eps.copy()
    rows = 0
    for r in range(len(wp) - 1):
        if (st0[wl[wp[r]:wp[r + 1]]] != 0).any():
            exp[wl[wp[r]:wp[r + 1]]] *= 20.0
            rows += 1
    assert solver.psp_rescale_failed_rows(20.0) == rows == 2
    eps1 = solver.psp_get_perturbations()
    assert np.array_equal(eps1, exp)
    solver.psp_factor_batch(A, tol, st)
    solver.psp_solve_batch(Bt)
    xh = solver.psp_recover().cpu().numpy()
    rc, st1 = solver.psp_get_lane_status()
    X = solver.psp_get_solutions().cpu().numpy()
    solver.close()
    Xo, sto1 = oracle.SparseOracle(s, operm).batch(eps1, tol)
    assert np.array_equal(st1, sto1) and (st1 == 0).all() and rc == psp.PSP_OK
    assert np.array_equal(X, Xo)
    xo = oracle.combine(oracle.ladder_weight_matrix(ladders), Xo)
    assert rel(xh, xo) <= 1e-10


def test_identity_vs_normal_D_study():
    """D = I against D = diag(N(0,1)) on cfg1, one ladder per
    m = 1..4 (base eps 2e-3, alpha = 1..m): the recovered x's error against the
    partial-pivot x* falls by >= 10x per extra m for both (Theorem 1's O(eps^2m)).  Run with -s for the table."""
    w = config(1)
    s = w.system()
    xs, st = oracle.reference_solve(s)
    assert st == 0
    rng = np.random.default_rng(314)
    table = {}
    for name, d in (("identity", np.ones(s.n)), ("normal", rng.normal(size=s.n))):
        ladders = [2e-3 * np.arange(1, m + 1) for m in range(1, 5)]
        eps = np.concatenate([ladder_eps(m) for m in ladders])
        solver = psp.Solver(0)
        solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
        solver.psp_set_perturbations(eps, d)
        solver.psp_set_weights(*psp.ladder_weights_csr(ladders))
        A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
        Bt = torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda")
        solver.psp_factor_batch(A, 0.0)
        solver.psp_solve_batch(Bt)
        xh = solver.psp_recover().cpu().numpy()
        rc, _ = solver.psp_get_lane_status()
        solver.close()
        assert rc == psp.PSP_OK
        errs = [rel(xh[m, 0], xs[0]) for m in range(4)]
        table[name] = errs
        assert all(errs[m + 1] < errs[m] * 0.1 for m in range(3)) and errs[3] <= 1e-7
    print("\nD study (rel err of recovered x vs x*, m = 1..4):")
    for name, errs in table.items():
        print(f"  {name:8s} " + "  ".join(f"{e:.2e}" for e in errs))


@pytest.mark.parametrize("coop", [0, 2])
def test_values_only_refactorisation_many_jacobians(coop):
    """one symbolic analysis, several Jacobians with the same pattern
    (values-only re-upload, e.g. the NR steps / V-starts of P:L302): each
    factor_solve_batch on the same handle bitwise equal to the oracle on its values."""
    w = config(1)
    s = w.system()
    ladders = [w.ladders[0] * f for f in np.linspace(0.5, 2.0, 12)]   # K = 96 lanes
    eps = np.concatenate([ladder_eps(m) for m in ladders])
    rng = np.random.default_rng(302)
    solver = psp.Solver(0)
    solver.psp_set_option("coop", coop)
    if coop == 2:
        solver.psp_set_option("coop_global", 2)
    solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
    info, perm = solver.psp_get_symbolic_info()
    solver.psp_set_perturbations(eps, s.d)
    solver.psp_set_weights(*psp.ladder_weights_csr(ladders))
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    for j in range(3):
        vals = s.vals * (1.0 + 0.1 * rng.normal(size=len(s.vals)))
        A = torch.tensor(vals, dtype=torch.float64, device="cuda")
        solver.psp_factor_solve_batch(A, b, 0.0)
        xh = solver.psp_recover().cpu().numpy()
        rc, st = solver.psp_get_lane_status()
        X = solver.psp_get_solutions().cpu().numpy()
        sj = w.system()
        sj.vals = vals
        assert len(eps) == 2 * sum(len(l) for l in ladders)
        tol = oracle.default_tol(sj.n, sj.row_ptr, sj.col_idx, sj.vals)
        Xo, sto = oracle.SparseOracle(sj, perm).batch(eps, tol, s.b[:, :1])
        assert np.array_equal(st, sto) and np.array_equal(X[sto == 0], Xo[sto == 0])
        if (sto == 0).all():
            xo = oracle.combine(oracle.ladder_weight_matrix(ladders), Xo)
            assert rel(xh, xo) <= 1e-10
    solver.close()


@pytest.mark.parametrize("coop", [0, 2])
def test_default_pivot_tol_and_lane_independence(coop):
    w = config(1)
    s = w.system()
    eps = w.eps()
    g1 = gpu_run(s, eps, coop=coop)            # pivot_tol <= 0: device-computed default
    assert g1["solver"].psp_get_last_kernels()[0] == ("coop" if coop == 0 else
                                                      g1["solver"].psp_get_last_kernels()[0])
    if coop == 2:
        assert g1["solver"].psp_get_last_kernels()[0] != "coop"
    # the same lanes at other batch positions (another slab, another warp lane)
    eps2 = np.r_[np.full(45, 3e-3), eps[::-1]]
    g2 = gpu_run(s, eps2, coop=coop)
    assert np.array_equal(g2["X"][45:][::-1], g1["X"])
    assert (g1["status"] == 0).all()
    Xo, sto = oracle.dense_batch(s, g1["operm"], eps, oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals))
    assert np.array_equal(g1["X"], Xo) and np.array_equal(g1["status"], sto)


@pytest.mark.parametrize("coop", [0, 2])
def test_default_pivot_tol_discriminating_pivot(coop):
    """The device's default tolerance (n u ||A||_1, R10) decides a pivot the same way as
    oracle.default_tol where it matters: a lane whose leading pivot eps_k d_p (the
    structurally zero diagonal of the leading-zero order) sits just below tol
    fails at step 0, one just above succeeds (tol/2 and 2 tol; both sides exact)."""
    w = config(1)
    s = w.system()
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    dp = s.d[s.slot_p]
    e_lo, e_hi = 0.5 * tol / abs(dp), 2.0 * tol / abs(dp)
    eps = np.r_[w.eps(), e_lo, -e_lo, e_hi, -e_hi]
    g = gpu_run(s, eps, "mindeg_first", s.slot_p, 0.0, coop=coop)   # 0.0: the device default
    Xo, sto = oracle.SparseOracle(s, g["operm"]).batch(eps, tol)
    assert np.array_equal(g["status"], sto)
    assert list(sto[-4:-2]) == [1, 1] and (sto[-2:] != 1).all() and (sto[:-4] == 0).all()
    ok = sto == 0
    assert np.array_equal(g["X"][ok], Xo[ok])


def test_host_api_e2e_matches_device_path():
    w = config(1, n_ladders=4)
    s = w.system()
    eps = w.eps()
    g = gpu_run(s, eps, ladders=w.ladders)
    solver = g["solver"]
    A_h = torch.tensor(s.vals, dtype=torch.float64).pin_memory()
    B_h = torch.tensor(s.b.T.copy(), dtype=torch.float64).pin_memory()
    x_h = torch.empty((len(w.ladders), 1, s.n), dtype=torch.float64).pin_memory()
    rc = solver.psp_solve_host(A_h, B_h, x_h)
    assert rc == 0
    assert np.array_equal(x_h.numpy(), g["xhat"])


def test_host_api_async_pipeline():
    """psp_solve_host_async: three back-to-back calls with different A values (the
    double-buffered copies back overlap the next call) give, after psp_synchronize,
    exactly what the synchronous psp_solve_host gives for each."""
    w = config(1, n_ladders=4)
    s = w.system()
    eps = w.eps()
    g = gpu_run(s, eps, ladders=w.ladders)
    solver = g["solver"]
    B_h = torch.tensor(s.b.T.copy(), dtype=torch.float64).pin_memory()
    As = [torch.tensor(s.vals * f, dtype=torch.float64).pin_memory() for f in (1.0, 0.5, 2.0)]
    xs = [torch.full((len(w.ladders), 1, s.n), np.nan, dtype=torch.float64).pin_memory() for _ in As]
    for A_h, x_h in zip(As, xs):
        solver.psp_solve_host_async(A_h, B_h, x_h)
    solver.psp_synchronize()
    for A_h, x_h in zip(As, xs):
        ref = torch.empty_like(x_h).pin_memory()
        assert solver.psp_solve_host(A_h, B_h, ref) == 0
        assert np.array_equal(x_h.numpy(), ref.numpy())
    assert np.array_equal(xs[0].numpy(), g["xhat"])


@pytest.mark.parametrize("ci", [2])
def test_cfg2_geometric_ladder_sampled(ci):
    w = config(ci)
    s = w.system()
    eps = w.eps()
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    g = gpu_run(s, eps, tol=tol, ladders=w.ladders)
    assert (g["status"] == 0).all()
    sample = np.array([0, 1, 2, 3, 127, 128, 254, 255])
    Xo, sto = oracle.dense_batch(s, g["operm"], eps[sample], tol)
    assert np.array_equal(g["X"][sample], Xo)
    # recovered with all 128 pairs against the oracle's combination of the GPU-independent
    # sparse oracle lanes (all 256 lanes via OR2, bitwise equal to OR1)
    Xs, _ = oracle.SparseOracle(s, g["operm"]).batch(eps, tol)
    xo = oracle.combine(oracle.ladder_weight_matrix(w.ladders), Xs)
    assert rel(g["xhat"], xo) <= 1e-10


@pytest.mark.slow
@pytest.mark.parametrize("ci", [3, 4])
def test_large_configs_sampled_lanes(ci):
    w = config(ci)
    s = w.system()
    eps = w.eps()
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    g = gpu_run(s, eps, tol=tol, ladders=w.ladders)
    assert np.array_equal(g["perm"], oracle_perm(s, -1))
    assert (g["status"] == 0).all()
    K = len(eps)
    sample = np.unique(np.r_[0, 1, 15, 16, K // 2, K // 2 + 1, K - 16, K - 1])
    so = oracle.SparseOracle(s, g["operm"])
    Xo, sto = so.batch(eps[sample], tol)
    assert np.array_equal(g["X"][sample], Xo)
    # recovered solution of the first and last ladder
    for gi in [0, len(w.ladders) - 1]:
        lo = 16 * gi
        lanes = np.arange(lo, lo + 16)
        Xl, _ = so.batch(eps[lanes], tol)
        xo = oracle.combine(oracle.ladder_weight_matrix([w.ladders[gi]]), Xl)
        assert rel(g["xhat"][gi], xo[0]) <= 1e-10


def test_bench_size_sampled():
    """The launch configuration bench.py times (300-bus, K = 65536, R = 1): the fused
    psp_factor_solve_batch (the capacity-planned factor with the forward substitution,
    then the backward solve) and the uniform-ladder recover, lanes sampled from every
    CTA-sized stretch of the batch (first, middle, last CTA, the ragged end) against the
    oracle bitwise, and recovered ladders within 1e-10."""
    from bench import bench_workload
    w = bench_workload()
    s = w.system()
    eps = w.eps()
    K = len(eps)
    solver = psp.Solver(0)
    solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
    info, perm = solver.psp_get_symbolic_info()
    assert np.array_equal(perm, oracle_perm(s, -1))
    solver.psp_set_perturbations(eps, s.d)
    wp, wl, wv = psp.ladder_weights_csr(w.ladders)
    solver.psp_set_weights(wp, wl, wv)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    solver.psp_factor_solve_batch(A, b, 0.0)
    kernels = solver.psp_get_last_kernels()
    assert kernels[:2] == ("batch_spill", True), kernels   # the bench's factor
    xh = solver.psp_recover().cpu().numpy()
    rc, st = solver.psp_get_lane_status()
    assert rc == 0 and (st == 0).all()
    X = solver.psp_get_solutions()
    lanes_per_cta = 64 * info["spill_warps_per_cta"]
    n_cta = (K + lanes_per_cta - 1) // lanes_per_cta
    sample = set()
    for cta in (0, 1, n_cta // 2, n_cta - 2, n_cta - 1):
        lo = cta * lanes_per_cta
        sample |= {lo, lo + 31, lo + 32, lo + 63, lo + 64, lo + lanes_per_cta - 1}
    sample = np.array(sorted(k for k in sample | {K - 1, K - 2} if 0 <= k < K))
    Xs = X[torch.tensor(sample, device="cuda")].cpu().numpy()
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    Xo, sto = oracle.dense_batch(s, perm, eps[sample], tol, B=s.b[:, :1])
    assert (sto == 0).all()
    assert np.array_equal(Xs, Xo)
    for gi in [0, len(w.ladders) // 2, len(w.ladders) - 1]:
        lanes = np.arange(8 * gi, 8 * gi + 8)
        Xl, _ = oracle.dense_batch(s, perm, eps[lanes], tol, B=s.b[:, :1])
        xo = oracle.combine(oracle.ladder_weight_matrix([w.ladders[gi]]), Xl)
        assert rel(xh[gi], xo[0]) <= 1e-10


def test_infeasible_then_rescale_then_feasible():
    """recover on a batch with a failed lane raises BATCH_INFEASIBLE; after
    psp_rescale_failed_rows + refactor + recover the flag is gone (PSP_OK)."""
    w = config(1)
    s = w.system()
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    dp = abs(s.d[s.slot_p])
    bad = 0.25 * tol / dp                        # the leading pivot eps * d_p falls below tol
    mags = [bad, 2 * bad]
    eps = ladder_eps(mags)
    solver = psp.Solver(0)
    solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg_first", first_node=s.slot_p)
    solver.psp_set_perturbations(eps, s.d)
    wp, wl, wv = psp.ladder_weights_csr([mags])
    solver.psp_set_weights(wp, wl, wv)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    solver.psp_factor_solve_batch(A, b, 0.0)
    solver.psp_recover()
    rc, st = solver.psp_get_lane_status()
    assert rc == psp.PSP_ERR_BATCH_INFEASIBLE and (st[:2] == 1).all()
    assert solver.psp_rescale_failed_rows(2e-3 / bad) == 1
    solver.psp_factor_solve_batch(A, b, 0.0)
    xh = solver.psp_recover().cpu().numpy()
    rc, st = solver.psp_get_lane_status()
    assert rc == 0 and (st == 0).all() and np.isfinite(xh).all()


def test_diagonal_closed_form_at_full_size():
    """n = 18000 diagonal A, D: recovered x against the componentwise closed form
    (exact error identity, holds at any size)."""
    from test_oracle_solve import _Tiny
    n = 18000
    rng = np.random.default_rng(21)
    a = rng.uniform(1, 3, n) * rng.choice([-1, 1], n)
    d = rng.normal(size=n)
    d /= np.abs(d).max()
    b = rng.normal(size=n)
    sysm = _Tiny.__new__(_Tiny)
    sysm.n = n
    sysm.row_ptr = np.arange(n + 1, dtype=np.int32)
    sysm.col_idx = np.arange(n, dtype=np.int32)
    sysm.vals = a.copy()
    sysm.d = d
    sysm.b = b.reshape(n, 1)
    m, e = 4, 2e-3
    mags = [j * e for j in range(1, m + 1)]
    g = gpu_run(sysm, ladder_eps(mags), "natural", ladders=[mags])
    r = (d / a) ** 2
    pred = np.ones(n) * (-1) ** m
    for sm in mags:
        pred *= sm * sm / (1 - sm * sm * r)
    pred *= r ** m * (b / a)
    err = (b / a) - g["xhat"][0, 0]
    assert np.max(np.abs(err - pred)) <= 16 * np.finfo(float).eps * np.max(np.abs(b / a))


@pytest.mark.parametrize("gjp", [(1, 1, 1), (1, 1, 2), (2, 1, 1), (2, 2, 1), (4, 1, 1), (4, 2, 1),
                                 (1, 1, 1, 0)])
def test_factor_kernel_variants_bitwise(gjp):
    """Every warp/lane organisation of the factor kernel (G groups per warp, J lanes per
    thread, P warps per slab) keeps the canonical order: lanes bitwise equal to the
    oracle (leading-zero regime, growth ~1/eps, several slabs and a ragged tail)."""
    G, J, P = gjp[:3]
    pairs = gjp[3] if len(gjp) > 3 else 1
    gjp = gjp[:3]
    s = config(1).system()
    rng = np.random.default_rng(7)
    K = 100
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-6, -2, K)
    solver = psp.Solver(0)
    solver.psp_set_option("coop", 2)          # K = 100 would otherwise take the coop kernels
    solver.psp_set_option("coop_global", 2)   # (nor the global level-scheduled ones)
    solver.psp_set_option("factor_groups", G)
    solver.psp_set_option("factor_lanes", J)
    solver.psp_set_option("factor_slab_warps", P)
    solver.psp_set_option("factor_pairs", pairs)
    solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg_first", first_node=s.slot_p)
    info, perm = solver.psp_get_symbolic_info()
    assert (info["factor_groups"], info["factor_lanes_per_thread"], info["factor_slab_warps"]) == gjp
    solver.psp_set_perturbations(eps, s.d)
    solver.psp_factor_batch(torch.tensor(s.vals, dtype=torch.float64, device="cuda"), 1e-300)
    assert solver.psp_get_last_kernels()[0] in ("batch", "batch_tmem")
    solver.psp_solve_batch(torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda"))
    assert solver.psp_get_last_kernels()[2] in ("batch", "batch_tmem")
    X = solver.psp_get_solutions().cpu().numpy()
    Xo, sto = oracle.SparseOracle(s, perm).batch(eps, 1e-300)
    assert np.array_equal(X, Xo)
    # the factor itself, entry by entry, against a G=J=P=1 run
    ref = psp.Solver(0)
    ref.psp_set_option("coop", 2)
    ref.psp_set_option("coop_global", 2)   # (nor the global level-scheduled ones)
    ref.psp_set_option("factor_groups", 1)
    ref.psp_set_option("factor_pairs", 1 - pairs if gjp == (1, 1, 1) else 1)
    ref.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg_first", first_node=s.slot_p)
    ref.psp_set_perturbations(eps, s.d)
    ref.psp_factor_batch(torch.tensor(s.vals, dtype=torch.float64, device="cuda"), 1e-300)
    for k in (0, 31, 32, 99):
        assert np.array_equal(solver.psp_get_factor(k, info["nnz_LU"]), ref.psp_get_factor(k, info["nnz_LU"]))


@pytest.mark.parametrize("K", [33, 300, 1000])
def test_factor_tmem_variant_bitwise(K):
    """The factor variant whose warps 0..3 keep their pending slots in tensor memory
    (PSP_OPT_FACTOR_TMEM) and the solve variant with its live slots in tensor memory
    (PSP_OPT_SOLVE_TMEM) against the oracle and, factor entry by entry, against the
    shared-memory variants; K = 33 / 300 / 1000 leave partial last CTAs (TMEM warps only,
    or some shared-memory warps inactive) and a ragged last slab."""
    s = config(1).system()
    rng = np.random.default_rng(K)
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-6, -2, K)
    out = {}
    for tm in (1, 2):
        solver = psp.Solver(0)
        solver.psp_set_option("coop", 2)      # (K <= 8 x SMs would take the coop kernels)
        solver.psp_set_option("coop_global", 2)   # (nor the global level-scheduled ones)
        solver.psp_set_option("factor_tmem", tm)
        solver.psp_set_option("solve_tmem", tm)
        solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
        info, perm = solver.psp_get_symbolic_info()
        assert info["factor_pend_smem"] == (2 if tm == 1 else 1)
        assert info["solve_live_smem"] == (2 if tm == 1 else 1)
        solver.psp_set_perturbations(eps, s.d)
        solver.psp_factor_batch(torch.tensor(s.vals, dtype=torch.float64, device="cuda"), 1e-300)
        solver.psp_solve_batch(torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda"))
        want = "batch_tmem" if tm == 1 else "batch"
        assert solver.psp_get_last_kernels() == (want, False, want, True)
        out[tm] = (solver, info, perm, solver.psp_get_solutions().cpu().numpy())
    solver, info, perm, X = out[1]
    Xo, sto = oracle.SparseOracle(s, perm).batch(eps, 1e-300)
    assert np.array_equal(X, Xo)
    assert np.array_equal(X, out[2][3])
    for k in sorted(k for k in {0, 31, 32, 127, 128, K // 2, K - 1} if k < K):
        assert np.array_equal(solver.psp_get_factor(k, info["nnz_LU"]),
                              out[2][0].psp_get_factor(k, info["nnz_LU"]))


@pytest.mark.parametrize("ci,K", [(0, 37), (1, 33), (1, 1000), (2, 300)])
def test_fused_factor_solve_bitwise(ci, K):
    """psp_factor_solve_batch (forward substitution fused into the factorisation of
    [A | b]) against the oracle, and against factor_batch + solve_batch: solutions,
    lane statuses and the factor itself bitwise equal (ragged K, several CTAs)."""
    s = config(ci).system()
    rng = np.random.default_rng(K + 17 * ci)
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-6, -2, K)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    outs = []
    for fused in (True, False):
        solver = psp.Solver(0)
        solver.psp_set_option("coop", 2)      # (K <= 8 x SMs would take the coop kernels)
        solver.psp_set_option("coop_global", 2)   # (nor the global level-scheduled ones)
        solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
        info, perm = solver.psp_get_symbolic_info()
        solver.psp_set_perturbations(eps, s.d)
        if fused:
            solver.psp_factor_solve_batch(A, b, 0.0)
            kf, aug, ks, fwd = solver.psp_get_last_kernels()
            assert kf in ("batch", "batch_tmem", "batch_spill") and ks in ("batch", "batch_tmem")
            assert (aug, fwd) == ((True, False) if info["aug_ok"] == 2 else (False, True))
        else:
            solver.psp_factor_batch(A, 0.0)
            solver.psp_solve_batch(b.view(1, -1))
        X = solver.psp_get_solutions().cpu().numpy()
        rc, st = solver.psp_get_lane_status()
        F = [solver.psp_get_factor(k, info["nnz_LU"]) for k in sorted({0, K // 2, K - 1})]
        outs.append((X, st, F))
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    Xo, sto = oracle.SparseOracle(s, perm).batch(eps, tol, B=s.b[:, :1])
    X, st, F = outs[0]
    ok = sto == 0
    assert np.array_equal(st != 0, sto != 0)
    assert np.array_equal(X[ok], Xo[ok])
    assert np.array_equal(X[ok], outs[1][0][ok]) and np.array_equal(st, outs[1][1])
    assert all(np.array_equal(f1, f2) for f1, f2 in zip(F, outs[1][2]))


@pytest.mark.parametrize("fused", [False, True])
def test_lane_growth_matches_oracle(fused):
    """PSP_OPT_GROWTH: per-lane g_k = max|U_k| / max|A_k| computed on the device after
    the factorisation (a pass over the DU region of the factor) equals the oracle's
    exactly (max and one division), in both
    the plain and the fused factorisation; the option leaves the solutions unchanged."""
    s = config(1).system()
    rng = np.random.default_rng(5)
    K = 70
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-6, -2, K)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    Xs = []
    for grow in (1, 0):
        solver = psp.Solver(0)
        solver.psp_set_option("growth", grow)
        solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
        info, perm = solver.psp_get_symbolic_info()
        solver.psp_set_perturbations(eps, s.d)
        if fused:
            solver.psp_factor_solve_batch(A, b, 1e-300)
        else:
            solver.psp_factor_batch(A, 1e-300)
            solver.psp_solve_batch(b.view(1, -1))
        Xs.append(solver.psp_get_solutions().cpu().numpy())
        if grow:
            g = solver.psp_get_lane_growth()
            go = oracle.SparseOracle(s, perm).growth(eps[:12], 1e-300)
            assert np.array_equal(g[:12], go)
            assert np.all(np.isfinite(g)) and np.all(g > 0)
    assert np.array_equal(Xs[0], Xs[1])


def test_estimate_rho_matches_oracle_power_iteration():
    """psp_estimate_rho: power iteration for rho(A^-1 D) through the method's own
    recovered solutions (one alpha = 1..4 ladder at eps = 2e-3; eps_c * rho ~ 0.01, so
    the truncation error is ~1e-16) against the oracle's power iteration with a
    partial-pivot A^-1, same start vector and stopping rule; and a diagonal system's
    closed form max|d_i / a_i|."""
    w = config(1, n_ladders=1)
    s = w.system()
    eps = w.eps()
    g = gpu_run(s, eps, ladders=w.ladders)
    rho, it, conv = g["solver"].psp_estimate_rho(0, 500, 1e-6)
    ro, ito, convo = oracle.power_rho(s, np.ones(s.n), 500, 1e-6)
    assert conv and convo
    assert abs(rho - ro) <= 1e-5 * ro
    assert np.max(np.abs(eps)) * rho < 1.0   # Theorem 1's premise eps_c * rho < 1
    # diagonal: A^-1 D is diagonal, rho = max |d_i / a_i|
    rng = np.random.default_rng(11)
    n = 40
    a = rng.uniform(1, 3, n) * rng.choice([-1, 1], n)
    d = rng.uniform(-1, 1, n)
    a[5], d[5] = 0.25, 1.0
    class _Diag:
        pass
    sd = _Diag()
    sd.n, sd.row_ptr, sd.col_idx, sd.vals = n, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), a
    sd.d, sd.b = d, np.ones((n, 1))
    ladder = [np.array([1e-5, 2e-5])]
    eps_d = psp.psp_ladder_weights(ladder[0])[0]
    gd = gpu_run(sd, eps_d, ordering_kind="natural", ladders=ladder)
    rho_d, _, conv_d = gd["solver"].psp_estimate_rho(0, 500, 1e-12)
    assert conv_d and abs(rho_d - np.max(np.abs(d / a))) <= 1e-9 * 4


@pytest.mark.parametrize("n", [1, 2, 40])
def test_degenerate_patterns_fused_and_separate(n):
    """Degenerate shapes through both paths: n = 1 (one pivot, empty L), a 2 x 2 with a
    zero diagonal entry (the method's leading-zero regime in miniature), and a diagonal
    n = 40 (every pivot with c = 0: births and pivots only); K = 33 (ragged)."""
    rng = np.random.default_rng(n)
    if n == 2:
        Ad = np.array([[0.0, 1.5], [2.0, 1.0]])
    else:
        Ad = np.diag(rng.uniform(1, 3, n) * rng.choice([-1, 1], n))

    class _S:
        pass
    s = _S()
    rp, ci, v = [0], [], []
    for i in range(n):
        for j in range(n):
            if Ad[i, j] != 0 or i == j:
                ci.append(j)
                v.append(Ad[i, j])
        rp.append(len(ci))
    s.n, s.row_ptr, s.col_idx, s.vals = n, np.array(rp, np.int32), np.array(ci, np.int32), np.array(v)
    s.d = np.where(np.arange(n) % 2 == 0, 1.0, -0.5)
    s.b = rng.normal(size=(n, 1))
    K = 33
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-4, -1, K)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    outs = []
    for fused in (True, False):
        solver = psp.Solver(0)
        solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="natural")
        info, perm = solver.psp_get_symbolic_info()
        solver.psp_set_perturbations(eps, s.d)
        if fused:
            solver.psp_factor_solve_batch(A, b, 1e-300)
        else:
            solver.psp_factor_batch(A, 1e-300)
            solver.psp_solve_batch(b.view(1, -1))
        outs.append(solver.psp_get_solutions().cpu().numpy())
    Xo, sto = oracle.SparseOracle(s, np.arange(n, dtype=np.int32)).batch(eps, 1e-300)
    assert np.all(sto == 0)
    assert np.array_equal(outs[0], Xo) and np.array_equal(outs[1], Xo)


@pytest.mark.parametrize("ci,order,K", [(0, "mindeg", 37), (1, "mindeg", 8), (1, "mindeg_first", 40),
                                        (2, "mindeg", 64)])
def test_coop_kernels_bitwise_vs_batch_kernels(ci, order, K):
    """PSP_OPT_COOP: the cooperative small-batch kernels (one CTA per system, etree-level
    steps) against the batch kernels and the oracle: factor entries, statuses and
    solutions bitwise (slack-slot and leading-zero orderings, multi-RHS on cfg2, a
    failing lane: eps = 0 in the leading-zero regime)."""
    s = config(ci).system()
    rng = np.random.default_rng(K + ci)
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-6, -2, K)
    first = s.slot_p if order == "mindeg_first" else -1
    if order == "mindeg_first":
        eps[3] = 0.0   # unperturbed: the structural zero pivot fails this lane
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    B = torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda")
    outs = []
    for coop in (1, 2):
        solver = psp.Solver(0)
        solver.psp_set_option("coop", coop)
        if coop == 2:
            solver.psp_set_option("coop_global", 2)
        solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering=order, first_node=first)
        info, perm = solver.psp_get_symbolic_info()
        solver.psp_set_perturbations(eps, s.d)
        solver.psp_factor_batch(A, 0.0)
        solver.psp_solve_batch(B)
        rc, st = solver.psp_get_lane_status()
        F = [solver.psp_get_factor(k, info["nnz_LU"]) for k in sorted({0, K // 2, K - 1})]
        outs.append((solver.psp_get_solutions().cpu().numpy(), st, F, perm))
    (X1, st1, F1, perm), (X2, st2, F2, _) = outs
    assert np.array_equal(st1, st2)
    assert all(np.array_equal(a, b, equal_nan=True) for a, b in zip(F1, F2))
    assert np.array_equal(X1, X2, equal_nan=True)
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    Xo, sto = oracle.SparseOracle(s, perm).batch(eps, tol)
    ok = sto == 0
    assert np.array_equal(st1 != 0, sto != 0)
    assert np.array_equal(X1[ok], Xo[ok])
    if order == "mindeg_first":
        assert st1[3] != 0


def test_phase_times_cover_the_launches():
    """PSP_OPT_PHASE_EVENTS / psp_get_phase_times: mean device time of the factor and the
    solve launches since the last read (positive, and reset by the read)."""
    s = config(1).system()
    eps = np.tile([1e-3, -1e-3], 64)
    solver = psp.Solver(0)
    solver.psp_set_option("phase_events", 1)
    solver.psp_set_option("coop", 2)
    solver.psp_set_option("coop_global", 2)   # (nor the global level-scheduled ones)
    solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
    solver.psp_set_perturbations(eps, s.d)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    for _ in range(3):
        solver.psp_factor_solve_batch(A, b, 0.0)
    tf, ts = solver.psp_get_phase_times()
    assert tf > 0 and ts > 0
    assert solver.psp_get_phase_times() == (0.0, 0.0)


@pytest.mark.parametrize("seed", [1, 2, 3, 1009, 5120, 5141])
def test_random_patterns_all_paths(seed, hubs=3, density=0.05):
    """Random structurally symmetric patterns with a few dense rows/columns (pivots with
    c > kFusedMax: scratch rows and UPDATE records; supernode pairs; zero diagonals),
    random K: the batch kernels (plain and fused) and the cooperative kernels, all
    bitwise against the oracle."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(40, 90))
    M = (rng.random((n, n)) < density).astype(float)
    for hub in rng.choice(n, hubs, replace=False):   # dense hubs -> large fronts
        M[hub, :] = M[:, hub] = (rng.random(n) < 0.6)
    M = np.maximum(M, M.T)
    np.fill_diagonal(M, rng.random(n) < 0.8)      # some structurally zero diagonals
    vals = rng.normal(size=(n, n)) * M
    vals += np.diag(np.where(np.diag(M) > 0, 4.0 * np.sign(rng.normal(size=n)), 0.0))

    class _S:
        pass
    s = _S()
    rp, ci, v = [0], [], []
    for i in range(n):
        for j in range(n):
            if M[i, j] != 0 or i == j:
                ci.append(j)
                v.append(vals[i, j])
        rp.append(len(ci))
    s.n, s.row_ptr, s.col_idx, s.vals = n, np.array(rp, np.int32), np.array(ci, np.int32), np.array(v)
    s.d = rng.normal(size=n)
    s.d /= np.max(np.abs(s.d))
    s.b = rng.normal(size=(n, 1))
    K = int(rng.integers(5, 150))
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-4, -1, K)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    res = []
    for coop, fused in ((2, False), (2, True), (1, False)):
        solver = psp.Solver(0)
        solver.psp_set_option("coop", coop)
        if coop == 2:
            solver.psp_set_option("coop_global", 2)
        solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
        info, perm = solver.psp_get_symbolic_info()
        solver.psp_set_perturbations(eps, s.d)
        if fused:
            solver.psp_factor_solve_batch(A, b, 1e-300)
        else:
            solver.psp_factor_batch(A, 1e-300)
            solver.psp_solve_batch(b.view(1, -1))
        rc, st = solver.psp_get_lane_status()
        res.append((solver.psp_get_solutions().cpu().numpy(), st, info))
    Xo, sto = oracle.SparseOracle(s, perm).batch(eps, 1e-300)
    ok = sto == 0
    for X, st, info in res:
        assert np.array_equal(st != 0, sto != 0)
        assert np.array_equal(X[ok], Xo[ok])
    assert res[0][2]["max_live"] > 0


@pytest.mark.parametrize("seed", [7001, 7002, 7003])
def test_random_sparse_patterns_tmem_fused(seed):
    """Random sparse patterns whose slots fit TMEM (the fused augmented program runs on
    the TMEM factor kernel): all paths bitwise against the oracle."""
    test_random_patterns_all_paths(seed, hubs=0, density=0.035)


def test_random_configurations_stress():
    """30 random configurations of tools/gpu/stress2.py (patterns with hubs and zero
    diagonals, orderings, R, forced G/J, TMEM, coop, fused, failing lanes, default
    tolerance, random weight rows): solutions, statuses and recovered rows bitwise
    against the oracle."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gpu", "stress2.py"), "30"],
                       capture_output=True, text=True, cwd=ROOT, env={**os.environ, "PSP_SEED0": "123000"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert "failures 0 of 30" in r.stdout, r.stdout[-2000:]


def test_sharded_recover_partials_sum_to_full():
    """Row a6 on one GPU through the library's sharding API: lanes split over two handles
    (psp_set_perturbations_shard; a ladder straddles the split), each with the dense
    GLOBAL weights (psp_set_weights_dense keeps its shard's columns) and its partial sums
    (psp_recover_reduce without a communicator); their sum equals the single-handle
    recovery up to the summation order (reading R16), and the oracle's within 1e-10."""
    w = config(1, n_ladders=6)
    s = w.system()
    eps = w.eps()
    K = len(eps)
    Wg = oracle.ladder_weight_matrix(w.ladders)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    B = torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda")

    def run(kb, ke):
        sv = psp.Solver(0)
        sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
        sv.psp_set_perturbations_shard(eps, s.d, kb, ke - kb)
        sv.psp_factor_batch(A, 0.0)
        sv.psp_solve_batch(B)
        sv.psp_set_weights_dense(Wg)
        out = sv.psp_recover_reduce(root=-1)
        torch.cuda.synchronize()
        return out.cpu().numpy()

    full = run(0, K)
    cut = K // 2 + 4                   # mid-ladder: lanes [0, cut) and [cut, K)
    assert cut % 8 != 0
    tot = run(0, cut) + run(cut, K)
    scale = np.abs(full).max()
    assert np.max(np.abs(tot - full)) <= 64 * np.finfo(float).eps * scale
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    Xo, _ = oracle.dense_batch(s, oracle_perm(s, -1), eps, tol)
    assert rel(full, oracle.combine(Wg, Xo)) <= 1e-10


@pytest.mark.parametrize("root", [-1, 0])
def test_nccl_recover_reduce_single_rank(root):
    """Row a6 through NCCL inside libpsp at nranks = 1 (psp_get_unique_id,
    psp_comm_init, psp_recover_reduce: ncclAllReduce / ncclReduce on the handle's stream):
    the reduced result equals the local combination bitwise (a 1-rank sum is a copy) and
    the oracle's combination within 1e-10; cfg2's single 128-pair ladder, R = 2."""
    w = config(2)
    s = w.system()
    eps = w.eps()
    Bn = s.b[:, :2].copy()
    sv = psp.Solver(0)
    sv.psp_comm_init(1, 0, psp.psp_get_unique_id())
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
    sv.psp_set_perturbations_shard(eps, s.d, 0, len(eps))
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    sv.psp_factor_batch(A, 0.0)
    sv.psp_solve_batch(torch.tensor(Bn.T.copy(), dtype=torch.float64, device="cuda"))
    Wg = oracle.ladder_weight_matrix(w.ladders)
    sv.psp_set_weights_dense(Wg)
    red = sv.psp_recover_reduce(root=root).cpu().numpy()
    loc = sv.psp_recover().cpu().numpy()
    assert np.array_equal(red, loc)
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    Xo, _ = oracle.SparseOracle(s, oracle_perm(s, -1)).batch(eps, tol, B=Bn)
    assert rel(red, oracle.combine(Wg, Xo)) <= 1e-10
    sv.close()


@pytest.mark.parametrize("K,fused", [(1000, False), (1000, True), (4133, True), (33, True)])
def test_spill_factor_bitwise(K, fused):
    """The capacity-planned factor (PSP_OPT_FACTOR_SPILL: <= 127 pending slots per lane,
    the entries with the furthest next use spilled to a global area and reloaded before
    their next use; 2 CTAs x 7 warps per SM) against the oracle and, factor entry by entry,
    against the unlimited-slot TMEM kernel: ragged K, several CTAs, the fused [A | b]
    program (its root step split into pivot and update steps) and the plain one."""
    s = config(1).system()
    rng = np.random.default_rng(K + 3)
    eps = rng.choice([-1, 1], K) * 10.0 ** rng.uniform(-6, -2, K)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    out = {}
    for sp in (1, 2):
        solver = psp.Solver(0)
        solver.psp_set_option("coop", 2)
        solver.psp_set_option("coop_global", 2)   # (nor the global level-scheduled ones)
        solver.psp_set_option("factor_spill", sp)
        solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
        info, perm = solver.psp_get_symbolic_info()
        if sp == 1:
            assert info["spill_ok"] == 3 and info["spill_ops"] > 0 and info["aug_spill_ops"] > 0
        solver.psp_set_perturbations(eps, s.d)
        if fused:
            solver.psp_factor_solve_batch(A, b, 0.0)
        else:
            solver.psp_factor_batch(A, 0.0)
            solver.psp_solve_batch(b.view(1, -1))
        kf, aug, ks, fwd = solver.psp_get_last_kernels()
        assert kf == ("batch_spill" if sp == 1 else "batch_tmem")
        assert aug == fused and fwd == (not fused)
        rc, st = solver.psp_get_lane_status()
        X = solver.psp_get_solutions().cpu().numpy()
        F = [solver.psp_get_factor(k, info["nnz_LU"]) for k in sorted({0, 31, 32, K // 2, K - 1})]
        out[sp] = (X, st, F, perm)
    X, st, F, perm = out[1]
    tol = oracle.default_tol(s.n, s.row_ptr, s.col_idx, s.vals)
    sample = np.unique(np.r_[0, 1, 31, 32, 223, 224, K // 2, K - 2, K - 1]) if K > 300 else np.arange(K)
    sample = sample[sample < K]
    Xo, sto = oracle.SparseOracle(s, perm).batch(eps[sample], tol, B=s.b[:, :1])
    assert np.array_equal(st[sample], sto)
    ok = sto == 0
    assert np.array_equal(X[sample][ok], Xo[ok])
    assert np.array_equal(X, out[2][0]) and np.array_equal(st, out[2][1])
    assert all(np.array_equal(f1, f2) for f1, f2 in zip(F, out[2][2]))


def _bound_check(xh, xs, e_pred, X, Xp, wrow):
    """Tolerance policy 3: ||x_hat - x*|| <= 1.5 ||e_pred|| + floor, floor =
    10 sum_k |w_k| ||x_k - x_k^piv||; where e_pred dominates the floor, x* - x_hat = e_pred
    vector-wise to within half its norm.  Per right-hand side."""
    for r in range(xs.shape[0]):
        floor = 10.0 * sum(abs(wk) * np.linalg.norm(X[k, r] - Xp[k, r]) for k, wk in wrow.items())
        err = xs[r] - xh[r]
        ne = np.linalg.norm(e_pred[r])
        assert np.linalg.norm(err) <= 1.5 * ne + floor, (np.linalg.norm(err), ne, floor)
        if ne > 100 * floor:
            assert np.linalg.norm(err - e_pred[r]) <= 0.5 * ne + floor


@pytest.mark.parametrize("m,base", [(1, 2e-3), (2, 2e-3), (2, 1e-2), (3, 2e-3), (4, 2e-3)])
def test_recovered_vs_pivoted_within_predicted_error(m, base):
    """The north star's third bar: the GPU's recovered x against the partial-pivot x*
    within the truncation error Theorem 1 predicts for this ladder (its exact form (I3),
    oracle.predicted_error), on the 300-bus Jacobian, the paper's alpha = 1..m ladder."""
    w = config(1)
    s = w.system()
    mags = [base * j for j in range(1, m + 1)]
    eps = ladder_eps(mags)
    g = gpu_run(s, eps, ladders=[mags])
    assert (g["status"] == 0).all()
    xs, st = oracle.reference_solve(s)
    assert st == 0
    e_pred = oracle.predicted_error(s, mags)
    Xp = oracle.pivoted_lanes(s, eps)
    wrow = dict(enumerate(oracle.ladder_weight_matrix([mags])[0]))
    _bound_check(g["xhat"][0], xs, e_pred, g["X"], Xp, wrow)


@pytest.mark.slow
def test_recovered_vs_pivoted_cfg2_geometric_ladder():
    """The same bar on BASELINE configs[2]'s ladder: 128 geometric magnitudes 1e-1..1e-8
    (K = 256), two right-hand sides."""
    w = config(2)
    s = w.system()
    B = s.b[:, :2].copy()
    eps = w.eps()
    mags = w.ladders[0]
    g = gpu_run(s, eps, B=B, ladders=w.ladders)
    assert (g["status"] == 0).all()
    xs, st = oracle.reference_solve(s, B)
    e_pred = oracle.predicted_error(s, mags, B)
    Xp = oracle.pivoted_lanes(s, eps, B)
    wrow = dict(enumerate(oracle.ladder_weight_matrix(w.ladders)[0]))
    _bound_check(g["xhat"][0], xs, e_pred, g["X"], Xp, wrow)
