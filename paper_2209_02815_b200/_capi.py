"""ctypes binding of the gnw C-ABI (include/gnw.h) exported by libgnw.so.

The library is built in-tree (``make -C paper_2209_02815_b200/csrc``) and loaded from
this directory.  There is no fallback: if libgnw.so is missing, importing the solver
raises; if no B200 is visible, ``gnw_create`` fails with GNW_DEVICE.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgnw.so")

GNW_OK, GNW_INVALID_ARGUMENT, GNW_NUMERICAL, GNW_DEVICE = 0, 1, 2, 3
GNW_HOST_POINTERS, GNW_DEVICE_POINTERS = 0, 1
GNW_COARSE_INVERSE, GNW_COARSE_CHOLESKY = 0, 1
GNW_LOOP_REFERENCE, GNW_LOOP_FUSED, GNW_LOOP_AUTO, GNW_LOOP_LEAN, GNW_LOOP_PERSISTENT = 0, 1, 2, 3, 4


class GnwDeviceError(RuntimeError):
    """CUDA failure or missing device (no reference analogue)."""


class AmgOptions(C.Structure):
    """AmgOptions (proj/include/ertinv/amg.hpp:11-23)."""

    _fields_ = [("coarse_threshold", C.c_uint64), ("strength", C.c_double),
                ("jacobi_damping", C.c_double), ("prolongation_damping", C.c_double),
                ("max_aggregate_size", C.c_uint64), ("max_levels", C.c_uint64)]

    def __init__(self, coarse_threshold=64, strength=0.08, jacobi_damping=2.0 / 3.0,
                 prolongation_damping=2.0 / 3.0, max_aggregate_size=3, max_levels=25):
        super().__init__(coarse_threshold, strength, jacobi_damping, prolongation_damping,
                         max_aggregate_size, max_levels)


class _Mesh(C.Structure):
    _fields_ = [("n_vertices", C.c_uint64), ("vertices", C.c_void_p),
                ("n_cells", C.c_uint64), ("cells", C.c_void_p)]


class Timings(C.Structure):
    _fields_ = [("t_H", C.c_double), ("t_C", C.c_double), ("t_chol", C.c_double)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("converged", C.c_int32),
                ("true_relative_residual", C.c_double), ("n_hist", C.c_uint64),
                ("relative_residuals", C.c_void_p), ("pnorm_relative_residuals", C.c_void_p),
                ("hist_cap", C.c_uint64)]


class Info(C.Structure):
    _fields_ = [("K", C.c_uint64), ("N", C.c_uint64), ("n_vertices", C.c_uint64),
                ("n_edges", C.c_uint64), ("n_boundary_edges", C.c_uint64), ("n_levels", C.c_uint64),
                ("coarse_n", C.c_uint64), ("m", C.c_uint64), ("beta", C.c_double),
                ("device_bytes", C.c_uint64), ("collapse_level", C.c_int64)]


class Stats(C.Structure):
    _fields_ = [("t_minres", C.c_double), ("t_rhs", C.c_double),
                ("kernel_launches", C.c_uint64), ("setup_kernel_launches", C.c_uint64),
                ("loop_restarts", C.c_uint64), ("fused_iterations", C.c_uint64),
                ("lean_iterations", C.c_uint64), ("persistent_iterations", C.c_uint64), ("comm_calls", C.c_uint64),
                ("comm_bytes", C.c_double)]


# every symbol include/gnw.h declares (checked by tests/test_capi_symbols.py)
EXPORTED = [
    "gnw_last_error", "gnw_version", "gnw_create", "gnw_destroy", "gnw_set_pointer_mode",
    "gnw_set_coarse_mode", "gnw_set_preconditioner", "gnw_set_loop_mode", "gnw_assemble", "gnw_assemble_amg_csr",
    "gnw_assemble_saddle_csr", "gnw_set_amg_hierarchy", "gnw_set_flux_scaling", "gnw_get_info",
    "gnw_set_jacobian", "gnw_prefetch_jacobian", "gnw_apply_operator", "gnw_precondition", "gnw_amg_apply",
    "gnw_get_woodbury", "gnw_assemble_rhs", "gnw_minres_solve", "gnw_gn_step_solve", "gnw_minres_history", "gnw_export_csr",
    "gnw_export_mesh", "gnw_dense_cholesky", "gnw_get_stats", "gnw_event_record",
    "gnw_event_elapsed", "gnw_profile_kernel", "gnw_set_electrodes", "gnw_response_jacobian",
    "gnw_geometric_factor", "gnw_nccl_unique_id", "gnw_create_partitioned", "gnw_create_local_group",
    "gnw_get_partition", "gnw_partition_cells", "gnw_partition_saddle", "gnw_partition_csr", "gnw_gauss_newton",
]


class ErtConfig(C.Structure):
    """ElectrodeConfig, survey.hpp:15-21 (b = -1: pole at infinity)."""

    _fields_ = [("a", C.c_int64), ("b", C.c_int64), ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_double)]


class ErtStats(C.Structure):
    _fields_ = [("t_assemble", C.c_double), ("t_amg", C.c_double), ("t_solve", C.c_double),
                ("t_jacobian", C.c_double), ("pcg_iterations", C.c_uint64),
                ("gmg_levels", C.c_uint64)]

class GnConfig(C.Structure):
    """GnConfig (inversion.hpp:66-75)."""

    _fields_ = [("beta", C.c_double), ("max_outer_steps", C.c_uint64), ("minres_tol", C.c_double),
                ("minres_maxit", C.c_uint64), ("algorithm", C.c_int32), ("misfit_reduction_tol", C.c_double),
                ("forward_tol", C.c_double)]


class GnStep(C.Structure):
    """GnStepReport (inversion.hpp:77-87) + t_forward."""

    _fields_ = [("misfit", C.c_double), ("minres_iters", C.c_uint64), ("converged", C.c_int32),
                ("euclid_relative_residual", C.c_double), ("pnorm_relative_residual", C.c_double),
                ("t_H", C.c_double), ("t_C", C.c_double), ("t_chol", C.c_double), ("t_norm", C.c_double),
                ("t_forward", C.c_double)]


KERNELS = {"row_gemv": 0, "saddle": 1, "combine_prec": 2, "finish_prec": 3, "vcycle": 4,
           "update": 5, "dgemm": 6, "iteration": 7, "body": 8, "saddle_fused": 9, "finish_fused": 10,
           "col_sweep": 11, "finish_lean": 12}

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libgnw.so not built at {LIB_PATH}: run `make -C {HERE}/csrc` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, u64, dbl, i32 = C.c_void_p, C.c_uint64, C.c_double, C.c_int
    L.gnw_last_error.restype = C.c_char_p
    L.gnw_version.restype = C.c_char_p
    L.gnw_create.argtypes = [i32, C.POINTER(C.c_int), C.POINTER(vp)]
    L.gnw_destroy.argtypes = [vp]
    L.gnw_destroy.restype = None
    L.gnw_set_pointer_mode.argtypes = [vp, i32]
    L.gnw_set_coarse_mode.argtypes = [vp, i32]
    L.gnw_set_preconditioner.argtypes = [vp, i32]
    L.gnw_set_loop_mode.argtypes = [vp, i32]
    L.gnw_assemble.argtypes = [vp, C.POINTER(_Mesh), C.POINTER(AmgOptions)]
    L.gnw_assemble_amg_csr.argtypes = [vp, u64, vp, vp, vp, C.POINTER(AmgOptions)]
    L.gnw_get_info.argtypes = [vp, C.POINTER(Info)]
    L.gnw_set_jacobian.argtypes = [vp, vp, u64, u64, dbl, C.POINTER(Timings)]
    L.gnw_prefetch_jacobian.argtypes = [vp, vp, u64, u64]
    L.gnw_apply_operator.argtypes = [vp, vp, vp]
    L.gnw_precondition.argtypes = [vp, vp, vp]
    L.gnw_amg_apply.argtypes = [vp, vp, vp]
    L.gnw_get_woodbury.argtypes = [vp, vp, vp]
    L.gnw_assemble_rhs.argtypes = [vp, vp, vp, vp, vp, vp]
    L.gnw_minres_solve.argtypes = [vp, vp, vp, vp, dbl, u64, C.POINTER(Report)]
    L.gnw_gn_step_solve.argtypes = [vp, vp, vp, vp, vp, vp, dbl, u64, C.POINTER(Report)]
    L.gnw_minres_history.argtypes = [vp, vp, vp, u64, C.POINTER(u64)]
    L.gnw_export_csr.argtypes = [vp, i32, u64, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), vp, vp, vp]
    L.gnw_export_mesh.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.gnw_dense_cholesky.argtypes = [vp, u64, vp, vp]
    L.gnw_get_stats.argtypes = [vp, C.POINTER(Stats)]
    L.gnw_event_record.argtypes = [vp, i32]
    L.gnw_event_elapsed.argtypes = [vp, i32, i32, C.POINTER(dbl)]
    L.gnw_profile_kernel.argtypes = [vp, i32, i32, C.POINTER(dbl), C.POINTER(dbl)]
    L.gnw_set_electrodes.argtypes = [vp, vp, u64]
    L.gnw_response_jacobian.argtypes = [vp, vp, C.POINTER(ErtConfig), u64, vp, vp, dbl, C.POINTER(ErtStats)]
    L.gnw_geometric_factor.argtypes = [vp, vp, vp, vp, i32, C.POINTER(dbl)]
    L.gnw_nccl_unique_id.argtypes = [vp]
    L.gnw_create_partitioned.argtypes = [i32, i32, i32, vp, C.POINTER(vp)]
    L.gnw_create_local_group.argtypes = [i32, i32, C.POINTER(vp)]
    L.gnw_partition_cells.argtypes = [u64, i32, vp]
    L.gnw_partition_saddle.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp]
    L.gnw_partition_csr.argtypes = [vp, i32, i32, i32, C.POINTER(u64), C.POINTER(u64), vp, vp, vp]
    L.gnw_gauss_newton.argtypes = [vp, vp, vp, C.POINTER(ErtConfig), u64, vp, C.POINTER(GnConfig), vp,
                                   C.POINTER(GnStep), u64, C.POINTER(u64), C.POINTER(dbl)]
    L.gnw_get_partition.argtypes = [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    for name in EXPORTED:
        fn = getattr(L, name)
        if name not in ("gnw_last_error", "gnw_version", "gnw_destroy"):
            fn.restype = C.c_int
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == GNW_OK:
        return
    msg = load().gnw_last_error().decode()
    if rc == GNW_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if rc == GNW_DEVICE:
        raise GnwDeviceError(msg)
    raise RuntimeError(msg)  # std::runtime_error


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)
