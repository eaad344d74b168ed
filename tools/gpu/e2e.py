"""Per-step slope of the pipelined host-buffer path (psp_solve_host_async)."""
import os
import sys
import time
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_11833_b200 import psp
import bench

w = bench.bench_workload(0)
s = w.system()
eps = w.eps()
solver = psp.Solver(0, torch.cuda.current_stream())
solver.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, ordering="mindeg")
solver.psp_set_perturbations(eps, s.d)
wp, wl, wv = psp.ladder_weights_csr(w.ladders)
solver.psp_set_weights(wp, wl, wv)
W = len(w.ladders)
A_h = torch.tensor(s.vals, dtype=torch.float64).pin_memory()
B_h = torch.tensor(s.b.T.copy(), dtype=torch.float64).pin_memory()
x_h = torch.empty((W, 1, s.n), dtype=torch.float64).pin_memory()
for _ in range(3):
    solver.psp_solve_host(A_h, B_h, x_h)
for mode in ("async", "sync", "async"):
    for N in (5, 20, 60):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(N):
            if mode == "async":
                solver.psp_solve_host_async(A_h, B_h, x_h)
            else:
                solver.psp_solve_host(A_h, B_h, x_h)
        solver.psp_synchronize()
        dt = time.perf_counter() - t0
        print(f"{mode} N={N}: {dt / N * 1e3:.3f} ms/step", flush=True)
# host-side enqueue cost alone
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    solver.psp_solve_host_async(A_h, B_h, x_h)
t1 = time.perf_counter()
solver.psp_synchronize()
print(f"enqueue {((t1 - t0) / 20) * 1e3:.3f} ms/call (host)")
