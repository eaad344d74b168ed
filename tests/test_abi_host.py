"""GPU-free checks of the product library: it loads, exports every symbol the
header declares, and its host logic (ordering, symbolic analysis, weights, argument
validation) agrees with the oracle's independent implementation (integer parity is
bit-exact; weights within a few ulps of the exact rationals)."""
import os
import re

import numpy as np
import pytest

import oracle
from oracle import ordering, weights
from paper_2311_11833_b200 import psp
from psp_inputs import config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "psp.h")).read()
    return sorted(set(re.findall(r"^(?:psp_status|const char\*)\s+(psp_\w+)\s*\(", txt, re.M)))


def test_library_exports_header_symbols():
    L = psp.lib()
    syms = header_symbols()
    assert len(syms) >= 17
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(psp.EXPORTS) == syms


def test_status_strings():
    L = psp.lib()
    assert L.psp_status_string(0) == b"PSP_OK"
    assert L.psp_status_string(4) == b"PSP_ERR_ZERO_PIVOT"


@pytest.mark.parametrize("mags", [[1.0, 2.0], [1e-2, 5e-3], [2e-3 * j for j in range(1, 5)],
                                  [1e-3 * j for j in range(1, 9)],
                                  list(np.geomspace(1e-1, 1e-8, 16))])
def test_ladder_weights_vs_exact(mags):
    eps, w = psp.psp_ladder_weights(mags)
    assert np.array_equal(eps, np.array([s * sg for s in mags for sg in (1, -1)]))
    exact = weights.lane_weights(mags)
    scale = sum(abs(x) for x in exact)
    assert np.max(np.abs(w - np.array(exact))) <= 8 * np.finfo(float).eps * scale


def test_ladder_weights_errors():
    with pytest.raises(psp.PSPError):
        psp.psp_ladder_weights([1.0, 1.0])
    with pytest.raises(psp.PSPError):
        psp.psp_ladder_weights([0.0, 1.0])


@pytest.mark.parametrize("ci,first", [(0, False), (0, True), (1, False), (1, True), (3, False)])
def test_ordering_and_fill_parity_with_oracle(ci, first):
    s = config(ci).system()
    f = s.slot_p if first else None
    hs = psp.HostSymbolic()
    info, perm = hs.analyse(s.n, s.row_ptr, s.col_idx,
                            ordering="mindeg_first" if first else "mindeg",
                            first_node=-1 if f is None else f)
    operm = ordering.elimination_order(s.n, s.row_ptr, s.col_idx, first=f)
    assert np.array_equal(perm, operm)                      # integer parity, bit-exact
    fcp, fri = ordering.filled_pattern(s.n, s.row_ptr, s.col_idx, perm)
    assert info["nnz_LU"] == int(fcp[-1])
    assert info["nnz_L"] == (int(fcp[-1]) - s.n) // 2
    assert info["n"] == s.n and info["nnz_A"] == s.nnz
    assert info["n_struct_zero_diag"] == s.n_struct_zero_diag
    # factor fma count = sum over columns p of |Lcol(p)| * |Urow(p)| (symmetric: c_p^2)
    cp = np.array([np.sum(fri[fcp[j]:fcp[j + 1]] > j) for j in range(s.n)])
    assert info["factor_fma"] == int(np.sum(cp * cp))
    assert info["solve_fma"] == 2 * info["nnz_L"]


def test_natural_and_user_orderings():
    s = config(0).system()
    hs = psp.HostSymbolic()
    _, perm = hs.analyse(s.n, s.row_ptr, s.col_idx, ordering="natural")
    assert np.array_equal(perm, np.arange(s.n))
    up = np.arange(s.n)[::-1].copy()
    _, perm = hs.analyse(s.n, s.row_ptr, s.col_idx, ordering="user", user_perm=up)
    assert np.array_equal(perm, up)
    with pytest.raises(psp.PSPError):
        hs.analyse(s.n, s.row_ptr, s.col_idx, ordering="user", user_perm=np.zeros(s.n, np.int32))


def test_malformed_pattern_rejected():
    hs = psp.HostSymbolic()
    with pytest.raises(psp.PSPError):   # unsorted columns
        hs.analyse(2, [0, 2, 3], [1, 0, 1])
    with pytest.raises(psp.PSPError):   # out of range
        hs.analyse(2, [0, 1, 2], [0, 5])
    with pytest.raises(psp.PSPError):   # duplicates
        hs.analyse(2, [0, 2, 3], [0, 0, 1])


def test_host_only_handle_refuses_numeric_calls():
    import ctypes
    hs = psp.HostSymbolic()
    s = config(0).system()
    hs.analyse(s.n, s.row_ptr, s.col_idx)
    eps = np.array([1e-3, -1e-3])
    st = psp.lib().psp_set_perturbations(hs.h, 2, psp._np_ptr(eps), psp._np_ptr(np.asarray(s.d)))
    assert st == 8  # PSP_ERR_UNSUPPORTED


def test_options_validated_and_reported():
    """psp_set_option rejects out-of-range values (PSP_ERR_ARG) before any work; the
    kernel-variant options show up in the symbolic info; PSP_OPT_PHASE_EVENTS needs a
    device handle (PSP_ERR_STATE on a host-only one)."""
    hs = psp.HostSymbolic()
    for name, bad in (("factor_groups", 3), ("factor_lanes", 4), ("factor_slab_warps", 3),
                      ("factor_pairs", 2), ("factor_tmem", 4), ("solve_tmem", 3), ("growth", 2),
                      ("phase_events", 2)):
        with pytest.raises(psp.PSPError) as e:
            hs.set_option(name, bad)
        assert e.value.status == 1, name   # PSP_ERR_ARG
    with pytest.raises(psp.PSPError) as e:
        hs.set_option("phase_events", 1)
    assert e.value.status == 3   # PSP_ERR_STATE
    s = config(1).system()
    info, _ = hs.analyse(s.n, s.row_ptr, s.col_idx)
    assert info["factor_pend_smem"] == 2 and info["aug_ok"] == 2     # TMEM variant, fused path
    hs.set_option("factor_tmem", 2)
    info, _ = hs.analyse(s.n, s.row_ptr, s.col_idx)
    assert info["factor_pend_smem"] == 1 and info["factor_warps_per_cta"] == 4
    hs.set_option("factor_tmem", 1)
    info3, _ = hs.analyse(s.n, s.row_ptr, s.col_idx)
    assert info3["factor_pend_smem"] == 2 and info3["aug_max_live"] > info3["max_live"]
    hs.close()


# --- structural transversal (PSP_OPT_TRANSVERSAL) --------------------------------
def _hk_case(n, rp, ci):
    from oracle import transversal
    hs = psp.HostSymbolic()
    hs.set_option("transversal", 1)
    info, perm = hs.analyse(n, rp, ci)
    q = hs.get_transversal(n)
    qo = transversal.hopcroft_karp(n, rp, ci)
    assert np.array_equal(q, np.array(qo, np.int32))        # bit-exact integer work
    # the symmetric order is the oracle's min-degree order of A_hat = A[q, :]
    trp, tci, _ = transversal.permuted_rows(n, rp, ci, np.ones(len(ci)), qo)
    assert np.array_equal(perm, ordering.elimination_order(n, trp, tci))
    return info


@pytest.mark.parametrize("ci", [0, 1])
def test_transversal_matches_oracle_on_listed_jacobian(ci):
    s = config(ci).system(convention="listed")
    info = _hk_case(s.n, s.row_ptr, s.col_idx)
    assert info["n_struct_zero_diag"] == 0                    # zero-free diagonal after it


@pytest.mark.parametrize("seed", range(6))
def test_transversal_matches_oracle_random(seed):
    rng = np.random.default_rng(seed)
    n = 40
    M = rng.random((n, n)) < 0.08
    M[np.arange(n), np.arange(n)] &= rng.random(n) < 0.3        # few diagonal entries
    M[np.arange(n), rng.permutation(n)] = True                  # structurally nonsingular
    rp, ci = [0], []
    for i in range(n):
        ci.extend(np.flatnonzero(M[i]).tolist())
        rp.append(len(ci))
    _hk_case(n, np.array(rp, np.int32), np.array(ci, np.int32))


def test_transversal_structurally_singular():
    n = 4   # rows 0 and 1 both only in column 0
    rp = np.array([0, 1, 2, 4, 6], np.int32)
    ci = np.array([0, 0, 1, 2, 2, 3], np.int32)
    hs = psp.HostSymbolic()
    hs.set_option("transversal", 1)
    with pytest.raises(psp.PSPError) as e:
        hs.analyse(n, rp, ci)
    assert e.value.status == 10
