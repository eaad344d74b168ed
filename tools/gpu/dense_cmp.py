"""Dense (DMMA) vs sparse path: factor / solve device times (library phase events) on
BASELINE configs (default cfg2: K = 256, R = 16; also cfg1 K = 8, cfg0), and the
achieved FP64 rate of the dense factor against its (2/3) N^3 per-lane flops."""
import os
import sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_11833_b200 import psp
from psp_inputs import config

for ci in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "2,1,0").split(",")]:
    w = config(ci)
    s = w.system()
    eps = w.eps()
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    B = torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda")
    out = {}
    for path in ("sparse", "dense"):
        sv = psp.Solver(0)
        sv.psp_set_option("phase_events", 1)
        sv.psp_set_option("path", path)
        sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
        sv.psp_set_perturbations(eps, s.d)
        for _ in range(3):
            sv.psp_factor_batch(A, 0.0)
            sv.psp_solve_batch(B)
        sv.psp_get_phase_times()
        for _ in range(10):
            sv.psp_factor_batch(A, 0.0)
            sv.psp_solve_batch(B)
        tf, ts = sv.psp_get_phase_times()
        out[path] = (tf, ts, sv.psp_get_last_kernels())
        sv.close()
    N = (s.n + 31) // 32 * 32
    K, R = len(eps), B.shape[0]
    fl = K * 2.0 / 3.0 * N ** 3
    sl = K * 2.0 * N * N * R
    tf, ts, kk = out["dense"]
    print(f"cfg{ci} n={s.n} N={N} K={K} R={R}: sparse factor {out['sparse'][0]:.3f} ms solve "
          f"{out['sparse'][1]:.3f} ms ({out['sparse'][2][0]}) | dense factor {tf:.3f} ms "
          f"({fl / tf / 1e9:.2f} TFLOP/s) solve {ts:.3f} ms ({sl / ts / 1e9:.2f} TFLOP/s) {kk}", flush=True)
