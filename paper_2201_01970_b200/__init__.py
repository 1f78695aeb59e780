"""B200-native CPR-GMRES SOLVE path — a drop-in for the reference package
cprkit's public API (src/__init__.py:15-54).

    from paper_2201_01970_b200 import build_cpr, gmres_solve, SolverConfig

Setup (aggregation, colouring, Galerkin, BILU(0)) runs in a host C++ library
and reproduces the reference's structures bit-exactly; the solve runs in
hand-written sm_100a kernels.  There is no CPU fallback for
the solve: device entry points raise if the CUDA library or device is missing.
"""

from .sparse import BlockCsrMatrix, CsrMatrix, axpy, dot, norm2, spmv, to_block
from .coloring import ColorPartition, strong_connections, vertices_grouping, verify_partition
from .amg import AmgParams, amg_cycle, build_hierarchy, hierarchy_summary, pairwise_aggregate
from .ilu import bilu0_factorize, bilu_apply, level_schedule
from .smoothers import PgsScmSmoother, SmootherSpec, gs_sweep, pgs_scm_sweep
from .cpr import (
    AscprCache,
    CprPreconditioner,
    GmresParams,
    GmresResult,
    SolverConfig,
    apply_cpr,
    ascpr_decide,
    ascpr_gmres_sequence,
    build_cpr,
    fingerprint_of,
    gmres_solve,
    pressure_matrix,
)
from .problems import ProblemSequence, generate_blackoil_like_sequence, load_sequence, save_sequence
from . import mmio

__version__ = "0.1.0"

__all__ = [
    "BlockCsrMatrix", "CsrMatrix", "axpy", "dot", "norm2", "spmv", "to_block",
    "ColorPartition", "strong_connections", "vertices_grouping", "verify_partition",
    "AmgParams", "amg_cycle", "build_hierarchy", "hierarchy_summary", "pairwise_aggregate",
    "bilu0_factorize", "bilu_apply", "level_schedule",
    "PgsScmSmoother", "SmootherSpec", "gs_sweep", "pgs_scm_sweep",
    "AscprCache", "CprPreconditioner", "GmresParams", "GmresResult", "SolverConfig",
    "apply_cpr", "ascpr_decide", "ascpr_gmres_sequence", "build_cpr", "fingerprint_of",
    "gmres_solve", "pressure_matrix",
    "ProblemSequence", "generate_blackoil_like_sequence", "save_sequence", "load_sequence", "mmio",
]
