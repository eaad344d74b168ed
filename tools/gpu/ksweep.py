"""SURVEY §8(d) config 1*: the 300-bus K-sweep (fused factor + solve + combination per
step, default launch choices), device time per step, solves/s, algorithmic HBM GB/s."""
import os
import sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2311_11833_b200 import psp
import bench

for K in [int(k) for k in (sys.argv[1] if len(sys.argv) > 1 else "8,64,512,4096,16384,65536,131072").split(",")]:
    w = bench.bench_workload(0, max(1, K // 8))
    s = w.system()
    eps = w.eps()[:K]
    sv = psp.Solver(0, torch.cuda.current_stream())
    sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
    info, _ = sv.psp_get_symbolic_info()
    sv.psp_set_perturbations(eps, s.d)
    wp, wl, wv = psp.ladder_weights_csr(w.ladders)
    sv.psp_set_weights(wp, wl, wv)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    x = torch.empty((len(w.ladders), 1, s.n), dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(3):
        sv.psp_factor_solve_batch(A, b, 0.0)
        sv.psp_recover(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        sv.psp_factor_solve_batch(A, b, 0.0)
        sv.psp_recover(x)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nnzLU, nnzL, n = info["nnz_LU"], info["nnz_L"], s.n
    byts = K * (8.0 * nnzLU + 8.0 * n) + K * (8.0 * (nnzLU - nnzL) + 16.0 * n) + K * 8.0 * n
    print(f"K={K:7d} {ms:8.3f} ms/step  {K / (ms * 1e-3) / 1e6:8.3f} M solves/s  "
          f"{byts / (ms * 1e-3) / 1e9:7.0f} GB/s alg ({byts / (ms * 1e-3) / 6566.4e9:5.1%} of 6566)", flush=True)
    sv.close()
