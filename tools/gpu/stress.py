"""Randomized stress: many random patterns and batch sizes through every path, bitwise
against the oracle (tests/test_gpu_parity.py::test_random_patterns_all_paths, more seeds)."""
import os
import sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import test_gpu_parity as t

bad = 0
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    try:
        t.test_random_patterns_all_paths(int(os.environ.get("PSP_SEED0", "1000")) + seed,
                                         hubs=int(os.environ.get("PSP_HUBS", "3")),
                                         density=float(os.environ.get("PSP_DENS", "0.05")))
    except AssertionError as e:
        bad += 1
        print("seed", int(os.environ.get("PSP_SEED0", "1000")) + seed, "FAILED", str(e)[:200], flush=True)
print("failures", bad)
