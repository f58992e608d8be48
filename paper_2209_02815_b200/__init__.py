"""gnw-b200: B200-native Woodbury-MINRES Gauss-Newton step solver (arXiv 2209.02815).

Hot path: the reference's Alg. 3 linear solve (proj/src/inversion.cpp:240-271) as
hand-written sm_100a FP64 CUDA kernels behind the C-ABI in include/gnw.h
(libgnw.so).  See DESIGN.md.
"""
from . import workload  # noqa: F401
from ._capi import AmgOptions, GnwDeviceError, LIB_PATH  # noqa: F401
from .solver import (Context, MinresReport, amg_setup, assemble_gn_rhs,  # noqa: F401
                     build_woodbury_preconditioner, geometric_factor, minres, nccl_unique_id,
                     partition_cells, partition_csr, partition_saddle, partitioned_from_torch_distributed,
                     run_ranks, shared_nccl_id)

__all__ = ["Context", "MinresReport", "AmgOptions", "GnwDeviceError", "amg_setup",
           "build_woodbury_preconditioner", "assemble_gn_rhs", "minres", "workload", "LIB_PATH",
           "nccl_unique_id", "partition_cells", "partition_saddle", "partition_csr", "partitioned_from_torch_distributed", "run_ranks", "shared_nccl_id"]
