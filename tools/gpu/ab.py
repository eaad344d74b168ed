"""A/B device timing of the bench workload's factor (+ solve) across library builds.

usage: python tools/gpu/ab.py LIB1 LIB2 ... [--rounds R] [--steps S]
Each round runs every library in its own process (PSP_LIB=...) and reads the mean
factor / solve launch times (library CUDA events) over S steps of
psp_factor_solve_batch + psp_solve_batch on the bench workload (K = 65536); rounds
alternate the libraries so that clock / thermal drift hits all alike."""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from bench import bench_workload
from paper_2311_11833_b200 import psp
steps = int(sys.argv[1])
w = bench_workload(0)
s = w.system()
sv = psp.Solver(0)
sv.psp_set_option("phase_events", 1)
sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
sv.psp_set_perturbations(w.eps(), s.d)
A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
b = torch.tensor(s.b[:, 0].copy(), dtype=torch.float64, device="cuda")
for _ in range(3):
    sv.psp_factor_solve_batch(A, b, 0.0)
sv.psp_get_phase_times()
for _ in range(steps):
    sv.psp_factor_solve_batch(A, b, 0.0)
tf, ts = sv.psp_get_phase_times()
print(json.dumps({"factor": tf, "solve": ts, "kernels": list(sv.psp_get_last_kernels())}))
'''


def main():
    libs = [a for a in sys.argv[1:] if not a.startswith("--")]
    rounds = int(sys.argv[sys.argv.index("--rounds") + 1]) if "--rounds" in sys.argv else 3
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 20
    libs = [l for l in libs if not l.isdigit()]
    res = {l: [] for l in libs}
    for r in range(rounds):
        for l in (libs if r % 2 == 0 else libs[::-1]):
            env = dict(os.environ, PSP_LIB=os.path.abspath(l))   # (under ncu the child is profiled too)
            out = subprocess.run([sys.executable, "-c", CHILD, str(steps)], env=env, capture_output=True, text=True)
            try:
                d = json.loads(out.stdout.strip().splitlines()[-1])
            except Exception:
                print(l, "FAILED", out.stderr[-800:], flush=True)
                continue
            res[l].append(d)
            print(f"round {r} {l}: factor {d['factor']:.4f} ms solve {d['solve']:.4f} ms {d['kernels']}", flush=True)
    for l in libs:
        f = sorted(d["factor"] for d in res[l])
        if f:
            print(f"{l}: factor median {f[len(f) // 2]:.4f} min {f[0]:.4f} ms over {len(f)} runs")


if __name__ == "__main__":
    main()
