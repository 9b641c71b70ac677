"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no basis functions, no model,
no objective, no search). It only draws inputs: per-job counter vectors F,
partition tables, power-cap grids and coefficient tables, from a bit-stable
splitmix64 stream so that the CPU oracle and the CUDA path see the same bytes.
"""
from .generator import (  # noqa: F401
    SplitMix64,
    Problem,
    CLASS_RANGES,
    MIXES,
    partition_table,
    cap_grid,
    make_features,
    make_coefficients,
    make_problem,
    tie_stress_features,
    bench_config,
    BENCH_CONFIGS,
)
