"""paper_2109_05451_b200 — B200-native distributed H² matrix-vector product (arXiv 2109.05451).

    Y := alpha * A * X + beta * Y,   A = A_de + <U, S, V^T>

Hot path: hand-written sm_100a CUDA kernels behind the C ABI in include/h2.h (libh2b200.so);
this package is the thin ctypes binding (argument marshalling only).  See DESIGN.md.
"""
from ._binding import (H2Operator, H2Group, H2Error, load_library, nccl_unique_id, plan_census, LIB_PATH, EXPORTS, PHASES,
                       H2_OK, H2_ERR_ARG, H2_ERR_SHAPE, H2_ERR_STRUCT, H2_ERR_CUDA, H2_ERR_NCCL,
                       H2_ERR_OOM, H2_ERR_STATE)
from .operator import operator_from_h2data, group_from_h2data

__all__ = ["H2Operator", "H2Group", "group_from_h2data", "H2Error", "load_library", "nccl_unique_id", "plan_census", "operator_from_h2data",
           "LIB_PATH", "EXPORTS"]
