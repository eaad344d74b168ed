"""GPU diagnostic: codegen status and per-phase timings of each kernel variant.

usage: python tools/gpu/diag.py [--ladders G] [--grid 300|2000|10000] [--variants 2,0]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_11833_b200 import psp  # noqa: E402
from psp_inputs import build_system, integer_ladder  # noqa: E402

GRIDS = {300: (300, 411, 69), 2000: (2000, 2700, 400), 10000: (10000, 13500, 2000)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ladders", type=int, default=8192)
    ap.add_argument("--grid", type=int, default=300)
    ap.add_argument("--groups", default="0,1:1,2:2,2:1,4:2", help="G:J[:P[:T]] (T: 0 auto, 1 TMEM, 2 no TMEM)")
    ap.add_argument("--warps", type=int, default=0)
    ap.add_argument("--pairs", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--R", type=int, default=1)
    a = ap.parse_args()
    s = build_system(*GRIDS[a.grid], seed=0, R=a.R)
    rng = np.random.default_rng([0, 7, 0])
    base = 10.0 ** rng.uniform(np.log10(5e-4), np.log10(5e-3), a.ladders)
    ladders = [integer_ladder(e, 4) for e in base]
    eps = np.concatenate([psp.psp_ladder_weights(m)[0] for m in ladders])
    K = len(eps)
    A = torch.tensor(s.vals, dtype=torch.float64, device="cuda")
    B = torch.tensor(s.b.T.copy(), dtype=torch.float64, device="cuda")
    ref = None
    for gj in a.groups.split(","):
        v, J, P, T, S = (int(x) for x in (gj + ":0:0:0:0").split(":")[:5])
        sv = psp.Solver(0)
        sv.psp_set_option("factor_groups", v)
        sv.psp_set_option("factor_pairs", a.pairs)
        sv.psp_set_option("factor_lanes", J)
        sv.psp_set_option("factor_slab_warps", P)
        sv.psp_set_option("factor_warps", a.warps)
        sv.psp_set_option("factor_tmem", T)
        sv.psp_set_option("solve_tmem", S)
        t0 = time.perf_counter()
        sv.psp_symbolic_analyse(s.n, s.row_ptr, s.col_idx, "mindeg")
        t_an = time.perf_counter() - t0
        info, _ = sv.psp_get_symbolic_info()
        print(f"[{gj}] analyse {t_an:.2f}s G={info['factor_groups']} J={info['factor_lanes_per_thread']} P={info['factor_slab_warps']} warps/cta={info['factor_warps_per_cta']}"
              f" pend_smem={info['factor_pend_smem']} solve_live_smem={info['solve_live_smem']}"
              f" nnz_LU={info['nnz_LU']} fma={info['factor_fma']} max_live={info['max_live']}", flush=True)
        sv.psp_set_perturbations(eps, s.d)
        st = sv.stream
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        tf, ts = [], []
        for r in range(a.reps + 1):
            ev[0].record(st)
            sv.psp_factor_batch(A, 0.0)
            ev[1].record(st)
            sv.psp_solve_batch(B)
            ev[2].record(st)
            torch.cuda.synchronize()
            if r:
                tf.append(ev[0].elapsed_time(ev[1]))
                ts.append(ev[1].elapsed_time(ev[2]))
        X = sv.psp_get_solutions().cpu().numpy()
        rc, stat = sv.psp_get_lane_status()
        same = None if ref is None else bool(np.array_equal(ref, X))
        ref = X if ref is None else ref
        gb_f = 8.0 * info["nnz_LU"] * K / 1e9
        print(f"  K={K} factor {np.median(tf):.3f} ms ({gb_f / np.median(tf) * 1e3:.0f} GB/s alg)"
              f"  solve {np.median(ts):.3f} ms ({(gb_f + 8e-9 * s.n * a.R * K) / np.median(ts) * 1e3:.0f} GB/s alg)"
              f"  rc={rc} failed={(stat != 0).sum()} bitwise_vs_first={same}", flush=True)
        sv.close()


if __name__ == "__main__":
    main()
