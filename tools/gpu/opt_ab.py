"""A/B of one library option on the bench workload (same process, alternating handles).

usage: python tools/gpu/opt_ab.py OPTION V0 V1 [--steps S] [--rounds R]
Prints the mean factor / solve launch times (library CUDA events) per value and whether
the solutions and statuses of the two settings are bitwise equal."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from bench import bench_workload
from paper_2311_11833_b200 import psp


def main():
    opt, v0, v1 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 20
    rounds = int(sys.argv[sys.argv.index("--rounds") + 1]) if "--rounds" in sys.argv else 3
    w = bench_workload(0)
    s = w.system()
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
    sol, X = {}, {}
    for v in (v0, v1):
        sv = psp.Solver(0)
        sv.psp_set_option("phase_events", 1)
        sv.psp_set_option(opt, v)
        sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
        sv.psp_set_perturbations(w.eps(), s.d)
        sol[v] = sv
    res = {v0: [], v1: []}
    for r in range(rounds):
        for v in ((v0, v1) if r % 2 == 0 else (v1, v0)):
            sv = sol[v]
            for _ in range(3):
                sv.psp_factor_solve_batch(A, b, 0.0)
            sv.psp_get_phase_times()
            for _ in range(steps):
                sv.psp_factor_solve_batch(A, b, 0.0)
            tf, ts = sv.psp_get_phase_times()
            res[v].append(tf)
            print(f"round {r} {opt}={v}: factor {tf:.4f} ms solve {ts:.4f} ms {sv.psp_get_last_kernels()}", flush=True)
    for v in (v0, v1):
        X[v] = sol[v].psp_get_solutions().cpu().numpy()
        f = sorted(res[v])
        print(f"{opt}={v}: factor median {f[len(f) // 2]:.4f} ms")
    st0, st1 = sol[v0].psp_get_lane_status()[1], sol[v1].psp_get_lane_status()[1]
    print("solutions bitwise equal:", bool(np.array_equal(X[v0], X[v1])), "statuses equal:", bool(np.array_equal(st0, st1)),
          "failed lanes:", int((st0 != 0).sum()))


if __name__ == "__main__":
    main()
