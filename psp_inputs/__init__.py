"""Seeded synthetic inputs shared by the CUDA path and the oracle (no method arithmetic)."""
from .powerflow import (PowerFlowSystem, Workload, build_system, config, integer_ladder,
                        ladder_eps, perturbation_diagonal, power_injections)
