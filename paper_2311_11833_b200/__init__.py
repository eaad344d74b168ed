"""B200-native batched perturbation-induced static pivoting (arXiv 2311.11833).

The numeric path lives in libpsp.so (csrc/: host symbolic analysis + sm_100a
kernels) behind the C ABI of include/psp.h; psp.py is its ctypes binding."""
from .psp import (HostSymbolic, PSPError, Solver, SymbolicInfo, ladder_weights_csr, lib,  # noqa: F401
                  psp_ladder_weights)
