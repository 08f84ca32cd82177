"""B200-native (sm_100a) Nekbone CG hot path, arXiv 2405.11065.

Public API (see include/nbk.h for the C ABI it wraps):
    cg_setup(MeshSpec, precision) -> Context with .ax_apply, .dssum, .glsc3,
    .cg_solve, .cg_solve_host, .load_arrays, .solution.
"""
from .configs import CONFIGS, Config  # noqa: F401
from .nbk import (AX_DSSUM, AX_LOCAL, AX_MASK, Context, Group, MeshSpec, NbkError,  # noqa: F401
                  cg_setup, load, nccl_unique_id, partition, version, workspace_bytes)

__all__ = ["CONFIGS", "Config", "Context", "Group", "MeshSpec", "NbkError", "cg_setup", "load",
           "nccl_unique_id", "partition", "version", "workspace_bytes", "AX_LOCAL", "AX_DSSUM",
           "AX_MASK"]
