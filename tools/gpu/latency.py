"""Latency point (BASELINE configs[1]: the 300-bus system, K = 8, one RHS): device time of one
psp_factor_solve_batch step (all its launches, CUDA events on the handle's stream) for the
fused dataflow kernel vs the cooperative factor + solve, plus cfg0 (K = 4)."""
import os
import sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_11833_b200 import psp
from psp_inputs import config

for ci in (1, 0):
    w = config(ci)
    s = w.system()
    eps = w.eps()
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    for df in (1, 2):
        sv = psp.Solver(0)
        sv.psp_set_option("dataflow", df)
        sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
        sv.psp_set_perturbations(eps, s.d)
        st = torch.cuda.current_stream()
        for _ in range(10):
            sv.psp_factor_solve_batch(A, b, 0.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        N = 200
        for _ in range(N):
            sv.psp_factor_solve_batch(A, b, 0.0)
        e1.record(st)
        torch.cuda.synchronize()
        print(f"cfg{ci} K={len(eps)} {'dataflow' if df == 1 else 'coop factor + solve'}: "
              f"{e0.elapsed_time(e1) / N * 1e3:.1f} us per step  kernels {sv.psp_get_last_kernels()}", flush=True)
        sv.close()
