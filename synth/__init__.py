"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path.

This package holds INPUTS only: the per-head pattern configuration types (the
output of the paper's offline search, Alg.4, consumed as input by the
hot path), the five BASELINE.json workload layouts, and deterministic Q/K/V /
modality-label generators.  It contains none of the method's arithmetic
(no estimation, no masks, no attention): both `oracle/` and the product package
import it, and neither imports the other.
"""
from .config import (  # noqa: F401
    KIND_NONE, KIND_FULL, KIND_ASHAPE, KIND_VSLASH, KIND_GRID,
    BND_NONE, BND_K, BND_Q, BND_2D, MAX_MOD,
    Pattern, HeadConfig, Problem,
    ashape, vslash, grid, full, none,
)
from .workloads import WORKLOADS, Workload, build_workload, layout_labels  # noqa: F401
from .gen import gen_qkv  # noqa: F401
