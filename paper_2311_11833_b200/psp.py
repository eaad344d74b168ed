"""Thin ctypes binding of libpsp.so (include/psp.h).  Argument marshalling only:
every numeric step runs in the library's CUDA kernels; there is no CPU fallback.
Functions keep the C names; `Solver` is a convenience wrapper over them that takes
torch tensors for device buffers (torch supplies memory and streams only)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PSP_LIB", os.path.join(_HERE, "libpsp.so"))

PSP_OK = 0
STATUS = {0: "PSP_OK", 1: "PSP_ERR_ARG", 2: "PSP_ERR_DIM", 3: "PSP_ERR_STATE",
          4: "PSP_ERR_ZERO_PIVOT", 5: "PSP_ERR_BATCH_INFEASIBLE", 6: "PSP_ERR_CUDA",
          7: "PSP_ERR_ALLOC", 8: "PSP_ERR_UNSUPPORTED", 9: "PSP_ERR_NCCL",
          10: "PSP_ERR_STRUCT_SINGULAR"}
PSP_ERR_ZERO_PIVOT = 4
PSP_ERR_BATCH_INFEASIBLE = 5
ORDER = {"natural": 0, "mindeg": 1, "user": 2, "mindeg_first": 3}

EXPORTS = ["psp_create", "psp_destroy", "psp_set_stream", "psp_status_string",
           "psp_last_error_detail", "psp_symbolic_analyse", "psp_get_symbolic_info",
           "psp_set_perturbations", "psp_factor_batch", "psp_solve_batch", "psp_factor_solve_batch",
           "psp_get_solutions", "psp_get_phase_times", "psp_get_lane_growth", "psp_estimate_rho",
           "psp_set_weights", "psp_recover", "psp_get_lane_status", "psp_solve_host", "psp_solve_host_async",
           "psp_synchronize", "psp_ladder_weights", "psp_set_option", "psp_get_factor", "psp_residual",
           "psp_rescale_failed_rows", "psp_get_perturbations", "psp_get_last_kernels",
           "psp_get_unique_id", "psp_comm_init", "psp_set_perturbations_shard", "psp_shard_weights",
           "psp_set_weights_dense", "psp_recover_reduce", "psp_get_dense_factor",
           "psp_set_perturbation_matrix", "psp_factor_batch_multi", "psp_solve_batch_multi",
           "psp_refine", "psp_get_transversal"]
KERNEL = {0: "none", 1: "coop", 2: "batch", 3: "batch_tmem", 4: "batch_spill", 5: "dense", 6: "coop_global", 7: "dataflow"}
PATH = {"sparse": 0, "dense": 1}
OPT = {"factor_groups": 1, "factor_warps": 2, "factor_lanes": 3, "factor_slab_warps": 4,
       "factor_pairs": 5, "factor_tmem": 6, "solve_tmem": 7, "phase_events": 8, "growth": 9, "coop": 10,
       "factor_spill": 11, "path": 12, "coop_global": 13,
       "transversal": 14, "dataflow": 15, "factor_hybrid": 16, "skip_zero_rows": 17}


class SymbolicInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("nnz_A", ctypes.c_int32), ("nnz_LU", ctypes.c_int32),
                ("nnz_L", ctypes.c_int32), ("n_struct_zero_diag", ctypes.c_int32),
                ("n_levels", ctypes.c_int32), ("factor_fma", ctypes.c_int64),
                ("factor_div", ctypes.c_int64), ("solve_fma", ctypes.c_int64),
                ("max_live", ctypes.c_int32), ("solve_live", ctypes.c_int32),
                ("births", ctypes.c_int32), ("factor_groups", ctypes.c_int32),
                ("factor_lanes_per_thread", ctypes.c_int32), ("factor_slab_warps", ctypes.c_int32),
                ("factor_warps_per_cta", ctypes.c_int32), ("factor_pend_smem", ctypes.c_int32),
                ("solve_live_smem", ctypes.c_int32), ("aug_ok", ctypes.c_int32),
                ("aug_max_live", ctypes.c_int32), ("aug_warps_per_cta", ctypes.c_int32),
                ("aug_pend_smem", ctypes.c_int32), ("spill_ok", ctypes.c_int32),
                ("spill_cap", ctypes.c_int32), ("spill_ops", ctypes.c_int32),
                ("spill_entries", ctypes.c_int32), ("aug_spill_ops", ctypes.c_int32),
                ("spill_warps_per_cta", ctypes.c_int32), ("struct_zero_l", ctypes.c_int32),
                ("skipped_rows", ctypes.c_int32), ("aug_skipped_rows", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class PSPError(RuntimeError):
    def __init__(self, status, detail=""):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status


_lib = None


def lib():
    """Load libpsp.so; fails loudly when the CUDA library is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        sig = {
            "psp_create": [ctypes.POINTER(P), I32, P],
            "psp_destroy": [P],
            "psp_set_stream": [P, P],
            "psp_synchronize": [P],
            "psp_symbolic_analyse": [P, I32, P, P, I32, P, I32],
            "psp_get_symbolic_info": [P, ctypes.POINTER(SymbolicInfo), P],
            "psp_set_perturbations": [P, I32, P, P],
            "psp_factor_batch": [P, P, D, P],
            "psp_solve_batch": [P, I32, P, I64],
            "psp_factor_solve_batch": [P, P, P, D, P],
            "psp_get_phase_times": [P, P],
            "psp_get_lane_growth": [P, P],
            "psp_estimate_rho": [P, I32, I32, D, P, P, P, P],
            "psp_residual": [P, P, I32, I32, P, P, P],
            "psp_rescale_failed_rows": [P, D, P],
            "psp_get_perturbations": [P, P],
            "psp_get_solutions": [P, P],
            "psp_set_weights": [P, I32, P, P, P],
            "psp_recover": [P, P],
            "psp_get_lane_status": [P, P],
            "psp_solve_host": [P, P, I32, P, D, P],
            "psp_solve_host_async": [P, P, I32, P, D, P],
            "psp_ladder_weights": [I32, P, P, P],
            "psp_set_option": [P, I32, I64],
            "psp_get_factor": [P, I32, P],
            "psp_get_last_kernels": [P, P],
            "psp_get_unique_id": [P],
            "psp_comm_init": [P, I32, I32, P],
            "psp_set_perturbations_shard": [P, I32, P, P, I32, I32],
            "psp_shard_weights": [I32, P, I32, I32, I32, P, P, P, P],
            "psp_set_weights_dense": [P, I32, P],
            "psp_recover_reduce": [P, P, I32],
            "psp_get_dense_factor": [P, I32, P],
            "psp_set_perturbation_matrix": [P, P],
            "psp_factor_batch_multi": [P, I32, P, D, P],
            "psp_solve_batch_multi": [P, I32, P, I64, I64],
            "psp_refine": [P, P, P, I32, P],
            "psp_get_transversal": [P, P],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = I32
        L.psp_status_string.argtypes = [I32]
        L.psp_status_string.restype = ctypes.c_char_p
        L.psp_last_error_detail.argtypes = [P]
        L.psp_last_error_detail.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _np_ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _t_ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def psp_ladder_weights(magnitudes):
    """C helper: (eps[2m], w[2m]) for one ladder (Remark 2, beta/2 per sign)."""
    s = np.ascontiguousarray(magnitudes, dtype=np.float64)
    m = len(s)
    eps = np.empty(2 * m)
    w = np.empty(2 * m)
    st = lib().psp_ladder_weights(m, _np_ptr(s), _np_ptr(eps), _np_ptr(w))
    if st:
        raise PSPError(st, "psp_ladder_weights")
    return eps, w


class Solver:
    """Owns one psp_handle on `device` / `stream` (a torch.cuda.Stream or None)."""

    def __init__(self, device=0, stream=None):
        import torch
        self.torch = torch
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = ctypes.c_void_p()
        self._check(lib().psp_create(ctypes.byref(h), device, ctypes.c_void_p(self.stream.cuda_stream)))
        self.h = h
        self.n = self.K = self.W = 0

    def _check(self, st):
        if st != PSP_OK:
            det = ""
            if getattr(self, "h", None) is not None and self.h:
                det = lib().psp_last_error_detail(self.h).decode()
            raise PSPError(st, det)
        return st

    def close(self):
        if getattr(self, "h", None) is not None and self.h and _lib is not None:
            _lib.psp_destroy(self.h)
        self.h = None

    __del__ = close

    # --- C-ABI wrappers ------------------------------------------------------
    def psp_set_option(self, name, value):
        if name == "path" and isinstance(value, str):
            value = PATH[value]
        self._check(lib().psp_set_option(self.h, OPT[name], int(value)))

    def psp_set_perturbation_matrix(self, D):
        """A general n x n perturbation matrix (host array, original ordering), or None to
        return to the diagonal d of psp_set_perturbations (include/psp.h)."""
        if D is None:
            self._check(lib().psp_set_perturbation_matrix(self.h, None))
            return
        Dm = np.ascontiguousarray(D, dtype=np.float64)
        if Dm.shape != (self.n, self.n):
            raise ValueError("D must be n x n")
        self._check(lib().psp_set_perturbation_matrix(self.h, _np_ptr(Dm)))

    def psp_factor_batch_multi(self, A_vals, pivot_tol=0.0, lane_status=None):
        """A_vals: device [n_jac, nnz_A]; lane k uses Jacobian k // (K // n_jac)."""
        if A_vals.dim() != 2 or A_vals.shape[1] != self.nnz_A:
            raise ValueError("A_vals must be [n_jac, nnz_A]")
        self._check_dev(A_vals, self.torch.float64, tuple(A_vals.shape))
        ls = None
        if lane_status is not None:
            self._check_dev(lane_status, self.torch.int32, (self.K,))
            ls = _t_ptr(lane_status)
        self._check(lib().psp_factor_batch_multi(self.h, int(A_vals.shape[0]), _t_ptr(A_vals), float(pivot_tol), ls))

    def psp_solve_batch_multi(self, B):
        """B: device [n_jac, R, n] (each Jacobian's right-hand sides, original ordering)."""
        if B.dim() != 3 or B.shape[2] != self.n:
            raise ValueError("B must be [n_jac, R, n]")
        self._check_dev(B, self.torch.float64, tuple(B.shape))
        R = int(B.shape[1])
        self._check(lib().psp_solve_batch_multi(self.h, R, _t_ptr(B), self.n, R * self.n))
        self.R = R

    def psp_refine(self, A_vals, b, iters, out=None):
        """Iterative-refinement baseline (include/psp.h): per lane, x^iters of the refinement
        with the lane's factor against the unperturbed A -> device [K, n] (original order)."""
        self._check_dev(A_vals, self.torch.float64, (self.nnz_A,))
        self._check_dev(b, self.torch.float64, (self.n,))
        out = out if out is not None else self.torch.empty((self.K, self.n), dtype=self.torch.float64,
                                                           device=f"cuda:{self.device}")
        self._check_dev(out, self.torch.float64, (self.K, self.n))
        self._check(lib().psp_refine(self.h, _t_ptr(A_vals), _t_ptr(b), int(iters), _t_ptr(out)))
        return out

    def psp_get_transversal(self):
        """The Hopcroft-Karp row matching q of the last analysis (PSP_OPT_TRANSVERSAL)."""
        q = np.empty(self.n, dtype=np.int32)
        self._check(lib().psp_get_transversal(self.h, _np_ptr(q)))
        return q

    def psp_get_dense_factor(self, k):
        """Lane k's dense factor (host numpy n x n, permuted order; L strict lower, U upper)."""
        out = np.empty((self.n, self.n), dtype=np.float64)
        self._check(lib().psp_get_dense_factor(self.h, int(k), _np_ptr(out)))
        return out

    def psp_symbolic_analyse(self, n, row_ptr, col_idx, ordering="mindeg", user_perm=None, first_node=-1):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        up = None if user_perm is None else np.ascontiguousarray(user_perm, dtype=np.int32)
        self._check(lib().psp_symbolic_analyse(self.h, int(n), _np_ptr(rp), _np_ptr(ci), ORDER[ordering],
                                               None if up is None else _np_ptr(up), int(first_node)))
        self.n = int(n)
        self.nnz_A = int(rp[-1])

    def psp_get_symbolic_info(self):
        info = SymbolicInfo()
        perm = np.empty(self.n, dtype=np.int32)
        self._check(lib().psp_get_symbolic_info(self.h, ctypes.byref(info), _np_ptr(perm)))
        return info.as_dict(), perm

    def psp_set_perturbations(self, eps, d):
        e = np.ascontiguousarray(eps, dtype=np.float64)
        dd = np.ascontiguousarray(d, dtype=np.float64)
        if dd.shape != (self.n,):
            raise ValueError("d must have n entries")
        self._check(lib().psp_set_perturbations(self.h, len(e), _np_ptr(e), _np_ptr(dd)))
        self.K = len(e)

    def psp_factor_batch(self, A_vals, pivot_tol=0.0, lane_status=None):
        self._check_dev(A_vals, self.torch.float64, (self.nnz_A,))
        ls = None
        if lane_status is not None:
            self._check_dev(lane_status, self.torch.int32, (self.K,))
            ls = _t_ptr(lane_status)
        self._check(lib().psp_factor_batch(self.h, _t_ptr(A_vals), float(pivot_tol), ls))

    def psp_solve_batch(self, B):
        """B: device float64 [R, n] (row r = RHS r; equals n x R column-major)."""
        self._check_dev(B, self.torch.float64, None)
        R, n = B.shape
        assert n == self.n and B.is_contiguous()
        self._check(lib().psp_solve_batch(self.h, R, _t_ptr(B), n))
        self.R = R

    def psp_factor_solve_batch(self, A_vals, b, pivot_tol=0.0, lane_status=None):
        """Factor + solve for one right-hand side b (device float64 [n] or [1, n]),
        forward substitution fused into the factorisation (psp.h)."""
        self._check_dev(A_vals, self.torch.float64, (self.nnz_A,))
        self._check_dev(b, self.torch.float64, None)
        assert b.numel() == self.n and b.is_contiguous()
        ls = None
        if lane_status is not None:
            self._check_dev(lane_status, self.torch.int32, (self.K,))
            ls = _t_ptr(lane_status)
        self._check(lib().psp_factor_solve_batch(self.h, _t_ptr(A_vals), _t_ptr(b), float(pivot_tol), ls))
        self.R = 1

    def psp_estimate_rho(self, w=0, max_iter=500, rtol=1e-6, v0=None):
        """rho(A^-1 D) by power iteration through recovered solution w (psp.h).
        Returns (rho, iterations, converged)."""
        v = np.ones(self.n) if v0 is None else np.ascontiguousarray(v0, dtype=np.float64)
        rho = ctypes.c_double()
        it = ctypes.c_int32()
        conv = ctypes.c_int32()
        self._check(lib().psp_estimate_rho(self.h, int(w), int(max_iter), float(rtol), _np_ptr(v),
                                           ctypes.byref(rho), ctypes.byref(it), ctypes.byref(conv)))
        self.R = 1
        return rho.value, it.value, bool(conv.value)

    def psp_residual(self, A_vals, B, x):
        """||A x[w][r] - B[r]||_2 for x device float64 [W, R, n] (original ordering, e.g.
        psp_recover's output), B device float64 [R, n]; returns numpy [W, R] (psp.h)."""
        self._check_dev(A_vals, self.torch.float64, (self.nnz_A,))
        self._check_dev(B, self.torch.float64, None)
        self._check_dev(x, self.torch.float64, None)
        R, n = B.shape
        assert n == self.n and B.is_contiguous() and x.is_contiguous()
        assert x.dim() == 3 and x.shape[1] == R and x.shape[2] == n
        W = x.shape[0]
        res = np.empty((W, R), dtype=np.float64)
        self._check(lib().psp_residual(self.h, _t_ptr(A_vals), W, R, _t_ptr(B), _t_ptr(x), _np_ptr(res)))
        return res

    def psp_rescale_failed_rows(self, scale):
        """Multiply the eps of every weight row holding a failed lane by `scale`;
        returns the number of rows rescaled (factor again afterwards; psp.h)."""
        n = ctypes.c_int32()
        self._check(lib().psp_rescale_failed_rows(self.h, float(scale), ctypes.byref(n)))
        return n.value

    def psp_get_perturbations(self):
        eps = np.empty(self.K, dtype=np.float64)
        self._check(lib().psp_get_perturbations(self.h, _np_ptr(eps)))
        return eps

    def psp_get_lane_growth(self):
        """g_k = max|U_k| / max|A_k| of the last factorisation (growth option on)."""
        g = np.empty(self.K, dtype=np.float64)
        self._check(lib().psp_get_lane_growth(self.h, _np_ptr(g)))
        return g

    def psp_get_phase_times(self):
        """(factor_ms, solve_ms) of the last factor / solve kernels (phase_events on)."""
        ms = (ctypes.c_float * 2)()
        self._check(lib().psp_get_phase_times(self.h, ms))
        return float(ms[0]), float(ms[1])

    def psp_comm_init(self, nranks, rank, uid: bytes):
        """Join the NCCL communicator with unique id `uid` (128 bytes, psp_get_unique_id)."""
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        self._check(lib().psp_comm_init(self.h, int(nranks), int(rank), buf))

    def psp_comm_init_from_group(self, group=None):
        """psp_comm_init over a torch.distributed process group: rank 0 draws the id,
        torch.distributed broadcasts it (plumbing), every rank joins."""
        import torch.distributed as dist
        obj = [psp_get_unique_id() if dist.get_rank(group) == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        self.psp_comm_init(dist.get_world_size(group), dist.get_rank(group), obj[0])

    def psp_set_perturbations_shard(self, eps_global, d, k_begin, k_count):
        e = np.ascontiguousarray(eps_global, dtype=np.float64)
        dd = np.ascontiguousarray(d, dtype=np.float64)
        if dd.shape != (self.n,):
            raise ValueError("d must have n entries")
        self._check(lib().psp_set_perturbations_shard(self.h, len(e), _np_ptr(e), _np_ptr(dd),
                                                      int(k_begin), int(k_count)))
        self.K = int(k_count)

    def psp_set_weights_dense(self, weights):
        """Dense GLOBAL weights [W, K_global]; this rank keeps its shard's columns."""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        self._check(lib().psp_set_weights_dense(self.h, w.shape[0], _np_ptr(w)))
        self.W = w.shape[0]

    def psp_recover_reduce(self, out=None, root=-1):
        """Partial sums on the device + the NCCL sum over the ranks (root = -1: every
        rank gets x; root >= 0: only `root`)."""
        out = out if out is not None else self.torch.empty((self.W, self.R, self.n), dtype=self.torch.float64,
                                                           device=f"cuda:{self.device}")
        self._check(lib().psp_recover_reduce(self.h, _t_ptr(out), int(root)))
        return out

    def psp_get_last_kernels(self):
        """(factor kernel, factor fused forward?, solve kernel, solve ran forward?) of the
        last numeric calls; kernel names from KERNEL (psp.h PSP_KERNEL_*)."""
        k = np.zeros(4, dtype=np.int32)
        self._check(lib().psp_get_last_kernels(self.h, _np_ptr(k)))
        return KERNEL[int(k[0])], bool(k[1]), KERNEL[int(k[2])], bool(k[3])

    def psp_get_solutions(self, out=None):
        out = out if out is not None else self.torch.empty((self.K, self.R, self.n), dtype=self.torch.float64,
                                                           device=f"cuda:{self.device}")
        self._check(lib().psp_get_solutions(self.h, _t_ptr(out)))
        return out

    def psp_get_factor(self, k, nnz_LU):
        """Lane k's factor values (host numpy, pivot-major layout of include/psp.h)."""
        out = np.empty(nnz_LU, dtype=np.float64)
        self._check(lib().psp_get_factor(self.h, int(k), _np_ptr(out)))
        return out

    def psp_set_weights(self, w_ptr, w_lane, w_val):
        p = np.ascontiguousarray(w_ptr, dtype=np.int32)
        la = np.ascontiguousarray(w_lane, dtype=np.int32)
        v = np.ascontiguousarray(w_val, dtype=np.float64)
        self._check(lib().psp_set_weights(self.h, len(p) - 1, _np_ptr(p), _np_ptr(la), _np_ptr(v)))
        self.W = len(p) - 1

    def psp_recover(self, out=None):
        out = out if out is not None else self.torch.empty((self.W, self.R, self.n), dtype=self.torch.float64,
                                                           device=f"cuda:{self.device}")
        self._check(lib().psp_recover(self.h, _t_ptr(out)))
        return out

    def psp_get_lane_status(self):
        st = np.empty(self.K, dtype=np.int32)
        rc = lib().psp_get_lane_status(self.h, _np_ptr(st))
        if rc not in (PSP_OK, PSP_ERR_ZERO_PIVOT, PSP_ERR_BATCH_INFEASIBLE):
            self._check(rc)
        return rc, st

    def psp_solve_host(self, A_vals_h, B_h, x_h, pivot_tol=0.0):
        """Host-buffer end-to-end call (torch CPU tensors, ideally pinned)."""
        R = B_h.shape[0]
        rc = lib().psp_solve_host(self.h, _t_ptr(A_vals_h), R, _t_ptr(B_h), float(pivot_tol), _t_ptr(x_h))
        if rc not in (PSP_OK, PSP_ERR_ZERO_PIVOT, PSP_ERR_BATCH_INFEASIBLE):
            self._check(rc)
        self.R = R
        return rc

    def psp_solve_host_async(self, A_vals_h, B_h, x_h, pivot_tol=0.0):
        """Pipelined host-buffer call (pinned torch CPU tensors); psp_synchronize to wait."""
        R = B_h.shape[0]
        self._check(lib().psp_solve_host_async(self.h, _t_ptr(A_vals_h), R, _t_ptr(B_h),
                                               float(pivot_tol), _t_ptr(x_h)))
        self.R = R

    def psp_synchronize(self):
        self._check(lib().psp_synchronize(self.h))

    def _check_dev(self, t, dtype, shape):
        if not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
            raise ValueError(f"expected a contiguous CUDA {dtype} tensor")
        if shape is not None and tuple(t.shape) != shape:
            raise ValueError(f"expected shape {shape}, got {tuple(t.shape)}")


def psp_get_unique_id() -> bytes:
    """C: a fresh NCCL unique id (128 bytes)."""
    buf = ctypes.create_string_buffer(128)
    st = lib().psp_get_unique_id(buf)
    if st:
        raise PSPError(st, "psp_get_unique_id")
    return buf.raw


def psp_shard_weights(weights, k_begin, k_count):
    """C helper: dense global weights [W, K_global] -> this shard's CSR over local lanes."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    W, Kg = w.shape
    ptr = np.zeros(W + 1, np.int32)
    lane = np.zeros(max(W * k_count, 1), np.int32)
    val = np.zeros(max(W * k_count, 1), np.float64)
    nnz = ctypes.c_int32()
    st = lib().psp_shard_weights(W, _np_ptr(w), Kg, int(k_begin), int(k_count), _np_ptr(ptr), _np_ptr(lane),
                                 _np_ptr(val), ctypes.byref(nnz))
    if st:
        raise PSPError(st, "psp_shard_weights")
    return ptr, lane[:nnz.value].copy(), val[:nnz.value].copy()


def ladder_weights_dense(ladders):
    """Dense GLOBAL weights [W, K] (psp_set_weights_dense) for ladders laid out
    consecutively in lane order, one recovered solution per ladder (C helper
    psp_ladder_weights: beta_j / 2 on each sign)."""
    K = 2 * sum(len(m) for m in ladders)
    out = np.zeros((len(ladders), K))
    k = 0
    for g, mags in enumerate(ladders):
        _, w = psp_ladder_weights(mags)
        out[g, k:k + len(w)] = w
        k += len(w)
    return out


def ladder_weights_csr(ladders, lane_offset=0, k_begin=0, k_end=None):
    """Weights CSR for ladders laid out consecutively in lane order (one recovered
    solution per ladder).  Only lanes in [k_begin, k_end) are kept, renumbered to
    local lanes (multi-GPU sharding: each rank recovers its own partial sums)."""
    ptr, lane, val = [0], [], []
    k = lane_offset
    for mags in ladders:
        _, w = psp_ladder_weights(mags)
        for j, c in enumerate(w):
            kk = k + j
            if k_end is None or (k_begin <= kk < k_end):
                lane.append(kk - k_begin)
                val.append(c)
        k += len(w)
        ptr.append(len(lane))
    return np.array(ptr, np.int32), np.array(lane, np.int32), np.array(val, np.float64)


def shard_range(K, rank, world):
    """Contiguous lane shard [k_begin, k_end) of `rank` among `world` ranks (SURVEY
    §8(e)): the K lanes split as evenly as possible, lower ranks first."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(int(K), world)
    k_begin = rank * base + min(rank, extra)
    return k_begin, k_begin + base + (1 if rank < extra else 0)


def recover_allreduce(solver, out, group=None):
    """Rows a5 + a6: psp_recover_reduce (partial sums on the device, NCCL all-reduce inside
    libpsp when the solver joined a communicator, psp_comm_init / psp_comm_init_from_group)."""
    return solver.psp_recover_reduce(out, root=-1)


class HostSymbolic:
    """Host-only handle (psp_create with device = -1): symbolic analysis only."""

    def __init__(self):
        h = ctypes.c_void_p()
        st = lib().psp_create(ctypes.byref(h), -1, None)
        if st:
            raise PSPError(st, "psp_create(host-only)")
        self.h = h

    def set_option(self, name, value):
        st = lib().psp_set_option(self.h, OPT[name], int(value))
        if st:
            raise PSPError(st, lib().psp_last_error_detail(self.h).decode())

    def get_transversal(self, n):
        q = np.empty(int(n), dtype=np.int32)
        st = lib().psp_get_transversal(self.h, _np_ptr(q))
        if st:
            raise PSPError(st, lib().psp_last_error_detail(self.h).decode())
        return q

    def analyse(self, n, row_ptr, col_idx, ordering="mindeg", user_perm=None, first_node=-1):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        up = None if user_perm is None else np.ascontiguousarray(user_perm, dtype=np.int32)
        st = lib().psp_symbolic_analyse(self.h, int(n), _np_ptr(rp), _np_ptr(ci), ORDER[ordering],
                                        None if up is None else _np_ptr(up), int(first_node))
        if st:
            raise PSPError(st, lib().psp_last_error_detail(self.h).decode())
        info = SymbolicInfo()
        perm = np.empty(int(n), dtype=np.int32)
        st = lib().psp_get_symbolic_info(self.h, ctypes.byref(info), _np_ptr(perm))
        if st:
            raise PSPError(st, "psp_get_symbolic_info")
        return info.as_dict(), perm

    def close(self):
        if self.h and _lib is not None:
            _lib.psp_destroy(self.h)
        self.h = None

    __del__ = close
