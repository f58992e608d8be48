"""Python face of the gnw C-ABI, mirroring the reference's interfaces.

The reference (proj/include/ertinv/inversion.hpp, minres.hpp, amg.hpp) exposes
``amg_setup``/``amg_apply``, ``build_woodbury_preconditioner``, ``SaddleOperator::apply``,
``WoodburyPreconditioner::apply``, ``assemble_gn_rhs`` and ``minres``.  ``Context`` binds
those to one B200 through libgnw.so; every heavy operation runs in the CUDA kernels of
``csrc/device``.  Errors keep the reference's semantics: ``std::invalid_argument`` ->
``ValueError``, ``std::runtime_error`` -> ``RuntimeError`` with the same message text.

Vectors may be numpy arrays (host pointers, copied in/out by the library) or, after
``use_device_pointers()``, torch CUDA float64 tensors (device pointers, no copies).
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np

from . import _capi as A
from .workload import Mesh


@dataclasses.dataclass
class MinresReport:
    """MinresReport, proj/include/ertinv/minres.hpp:13-22."""

    iterations: int
    relative_residuals: np.ndarray
    pnorm_relative_residuals: np.ndarray
    converged: bool
    true_relative_residual: float


def _dptr(x):
    """Raw pointer of a numpy array or a torch tensor."""
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


class Context:
    """One solver context on one GPU (``device=None``: host-only, setup/export only)."""

    def __init__(self, device: int | None = 0):
        self.L = A.load()
        h = C.c_void_p()
        if device is None:
            A.check(self.L.gnw_create(0, None, C.byref(h)))
        else:
            dev = (C.c_int * 1)(device)
            A.check(self.L.gnw_create(1, dev, C.byref(h)))
        self.h = h
        self.device = device
        self.device_pointers = False
        self._partitioned = False
        self.K = self.N = self.m = 0

    # ------------------------------------------------ partitioned (multi-GPU)
    @classmethod
    def _adopt(cls, handle, device):
        self = cls.__new__(cls)
        self.L = A.load()
        self.h = handle
        self.device = device
        self.device_pointers = False
        self._partitioned = True  # _adopt wraps the handles of partitioned / local-group contexts
        self.K = self.N = self.m = 0
        return self

    @classmethod
    def partitioned(cls, rank: int, world: int, nccl_id: bytes, device: int = 0) -> "Context":
        """One rank of a cell-partitioned P-GPU solve over NCCL (gnw_create_partitioned)."""
        L = A.load()
        buf = (C.c_ubyte * 128).from_buffer_copy(bytes(nccl_id))
        h = C.c_void_p()
        A.check(L.gnw_create_partitioned(device, rank, world, buf, C.byref(h)))
        return cls._adopt(h, device)

    @classmethod
    def local_group(cls, world: int, device: int = 0) -> list:
        """``world`` partitioned ranks in this process on one device; drive each from its own
        thread (``run_ranks``).  Same results as ``world`` GPUs over NCCL."""
        L = A.load()
        hs = (C.c_void_p * world)()
        A.check(L.gnw_create_local_group(device, world, hs))
        return [cls._adopt(C.c_void_p(hs[r]), device) for r in range(world)]

    def partition(self) -> dict:
        r, w = C.c_int(), C.c_int()
        lo, hi = C.c_int64(), C.c_int64()
        A.check(self.L.gnw_get_partition(self.h, C.byref(r), C.byref(w), C.byref(lo), C.byref(hi)))
        return {"rank": r.value, "world": w.value, "c_lo": lo.value, "c_hi": hi.value}

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            self.L.gnw_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----------------------------------------------------------- configuration
    def use_device_pointers(self, on: bool = True):
        A.check(self.L.gnw_set_pointer_mode(self.h, A.GNW_DEVICE_POINTERS if on else A.GNW_HOST_POINTERS))
        self.device_pointers = on

    def set_loop_mode(self, mode):
        """MINRES loop schedule (gnw.h): False / "reference" = SaddleOperator::apply's two sweeps
        over J; True / "fused" = one sweep (Woodbury identity); "auto" (the default) = fused
        for tol >= 1e-8, reference below."""
        modes = {False: A.GNW_LOOP_REFERENCE, True: A.GNW_LOOP_FUSED, "reference": A.GNW_LOOP_REFERENCE,
                 "fused": A.GNW_LOOP_FUSED, "auto": A.GNW_LOOP_AUTO, "lean": A.GNW_LOOP_LEAN,
                 "persistent": A.GNW_LOOP_PERSISTENT}
        A.check(self.L.gnw_set_loop_mode(self.h, modes[mode]))

    def loop_schedule(self) -> str:
        """The schedule the last solve's iterations ran: "reference", "fused", "lean" or "persistent"."""
        st = self.stats()
        if st["persistent_iterations"] > 0:
            return "persistent"
        if st["lean_iterations"] > 0:
            return "lean"
        return "fused" if st["fused_iterations"] > 0 else "reference"

    def set_coarse_mode(self, exact: bool):
        A.check(self.L.gnw_set_coarse_mode(self.h, A.GNW_COARSE_CHOLESKY if exact else A.GNW_COARSE_INVERSE))

    # ---------------------------------------------------------------- assembly
    def assemble(self, mesh: Mesh, opts: A.AmgOptions | None = None):
        """make_mixed_spaces + assemble_Q/D + amg_setup(assemble_lumped_schur(Q, D))."""
        v = A.f64(mesh.vertices).ravel()
        c = np.ascontiguousarray(mesh.cells, dtype=np.int64).ravel()
        m = A._Mesh(mesh.n_vertices, v.ctypes.data, mesh.n_cells, c.ctypes.data)
        A.check(self.L.gnw_assemble(self.h, C.byref(m), C.byref(opts) if opts is not None else None))
        info = self.info()
        self.K, self.N = info["K"], info["N"]
        self.m = 0
        return self

    def assemble_amg_csr(self, rowptr, cols, vals, opts: A.AmgOptions | None = None):
        """amg_setup(s_hat, opts) on a caller CSR matrix (amg.cpp:115-187)."""
        rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        vals = A.f64(vals)
        A.check(self.L.gnw_assemble_amg_csr(self.h, len(rowptr) - 1, rowptr.ctypes.data, cols.ctypes.data,
                                            vals.ctypes.data, C.byref(opts) if opts is not None else None))
        info = self.info()
        self.K, self.N = 0, info["N"]
        return self

    def info(self) -> dict:
        i = A.Info()
        A.check(self.L.gnw_get_info(self.h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in A.Info._fields_}

    def stats(self) -> dict:
        s = A.Stats()
        A.check(self.L.gnw_get_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in A.Stats._fields_}

    # ---------------------------------------------------------------- Jacobian
    def set_jacobian(self, J, beta: float, laplace_pc: bool = False) -> dict:
        """build_woodbury_preconditioner(q_diag_inv, amg, J, beta, &timings) (inversion.cpp:91-124).

        ``laplace_pc`` keeps J in the operator with the bare Laplace preconditioner
        (Alg. 4, inversion.cpp:251-256); ``J=None`` drops the low-rank term entirely."""
        A.check(self.L.gnw_set_preconditioner(self.h, 1 if laplace_pc else 0))
        t = A.Timings()
        if J is None:
            A.check(self.L.gnw_set_jacobian(self.h, None, 0, self.N, beta, C.byref(t)))
            self.m = 0
        else:
            if not self.device_pointers:
                J = A.f64(J)
            m, n = J.shape
            A.check(self.L.gnw_set_jacobian(self.h, _dptr(J), m, n, beta, C.byref(t)))
            self.m = m
        self.beta = beta
        return {"t_H": t.t_H, "t_C": t.t_C, "t_chol": t.t_chol}

    def prefetch_jacobian(self, J) -> None:
        """Start the host->device copy of the NEXT step's J beside the current solve
        (host-pointer mode; pinned J overlaps).  The next set_jacobian(J, ...) with the same
        array takes the staged copy.  J must not change in between."""
        if self.device_pointers:
            raise ValueError("gnw_prefetch_jacobian: host-pointer mode only")
        if not (isinstance(J, np.ndarray) and J.dtype == np.float64 and J.flags.c_contiguous):
            raise ValueError("gnw_prefetch_jacobian: J must be a C-contiguous float64 array (it is read later)")
        m, n = J.shape
        A.check(self.L.gnw_prefetch_jacobian(self.h, _dptr(J), m, n))

    # ----------------------------------------------------------------- applies
    def _out(self, n, like=None):
        if self.device_pointers:
            import torch
            return torch.empty(n, dtype=torch.float64, device=like.device if like is not None else "cuda")
        return np.zeros(n)

    def _in(self, x):
        return x if self.device_pointers else A.f64(x)

    def apply_operator(self, x):
        """SaddleOperator::apply (inversion.cpp:47-69)."""
        x = self._in(x)
        y = self._out(self.K + self.N, x)
        A.check(self.L.gnw_apply_operator(self.h, _dptr(x), _dptr(y)))
        return y

    def precondition(self, y):
        """WoodburyPreconditioner::apply (inversion.cpp:71-89)."""
        y = self._in(y)
        z = self._out(self.K + self.N, y)
        A.check(self.L.gnw_precondition(self.h, _dptr(y), _dptr(z)))
        return z

    def amg_apply(self, r):
        """amg_apply (amg.cpp:189-194): one V-cycle."""
        r = self._in(r)
        z = self._out(self.N, r)
        A.check(self.L.gnw_amg_apply(self.h, _dptr(r), _dptr(z)))
        return z

    def _check_out(self, out, n):
        if self.device_pointers or not (isinstance(out, np.ndarray) and out.dtype == np.float64
                                        and out.flags.c_contiguous and out.shape == (n,)):
            raise ValueError("out must be a C-contiguous float64 host array of the result's length")
        return out

    def assemble_rhs(self, m, m_ref, g, g_obs, out=None):
        """assemble_gn_rhs (inversion.cpp:126-146).  ``out``: optional host array (e.g. pinned)
        that receives the rhs."""
        m, m_ref, g, g_obs = (self._in(a) for a in (m, m_ref, g, g_obs))
        out = self._out(self.K + self.N, m) if out is None else self._check_out(out, self.K + self.N)
        A.check(self.L.gnw_assemble_rhs(self.h, _dptr(m), _dptr(m_ref), _dptr(g), _dptr(g_obs), _dptr(out)))
        return out

    def minres(self, b, x0=None, tol: float = 1e-8, maxit: int | None = None, hist_cap: int = 1 << 16,
               out=None):
        """minres(op.apply, pc.apply, b, x0, tol, maxit) (minres.cpp:20-155).  ``out``: optional
        host array (e.g. pinned) that receives x."""
        n = self.K + self.N
        b = self._in(b)
        if x0 is None and not self._partitioned:
            x0p = None  # NULL: the zero start, nothing transferred (gnw.h)
        elif x0 is None:
            x0 = self._out(n, b)
            if self.device_pointers:
                x0.zero_()
            x0p = _dptr(x0)
        else:
            x0 = self._in(x0)
            x0p = _dptr(x0)
        maxit = 2 * n if maxit is None else int(maxit)
        x = self._out(n, b) if out is None else self._check_out(out, n)
        he = np.zeros(hist_cap)
        hp = np.zeros(hist_cap)
        rep = A.Report(0, 0, 0.0, 0, he.ctypes.data, hp.ctypes.data, hist_cap)
        A.check(self.L.gnw_minres_solve(self.h, _dptr(b), x0p, _dptr(x), tol, maxit, C.byref(rep)))
        nh = min(int(rep.n_hist), hist_cap)
        return x, MinresReport(int(rep.iterations), he[:nh].copy(), hp[:nh].copy(), bool(rep.converged),
                               float(rep.true_relative_residual))

    def gn_step_solve(self, m, m_ref, g, g_obs, tol: float = 1e-8, maxit: int | None = None,
                      hist_cap: int = 1 << 16, out=None):
        """The reference's GN-step solve in one call (inversion.cpp:259-265): b = assemble_gn_rhs(...),
        x0 = 0, minres(op, pc, b, x0, tol, maxit).  The right-hand side never leaves the device."""
        n = self.K + self.N
        m, m_ref, g, g_obs = (self._in(v) for v in (m, m_ref, g, g_obs))
        maxit = 2 * n if maxit is None else int(maxit)
        x = self._out(n, m) if out is None else self._check_out(out, n)
        he = np.zeros(hist_cap)
        hp = np.zeros(hist_cap)
        rep = A.Report(0, 0, 0.0, 0, he.ctypes.data, hp.ctypes.data, hist_cap)
        A.check(self.L.gnw_gn_step_solve(self.h, _dptr(m), _dptr(m_ref), _dptr(g), _dptr(g_obs), _dptr(x), tol, maxit,
                                         C.byref(rep)))
        nh = min(int(rep.n_hist), hist_cap)
        return x, MinresReport(int(rep.iterations), he[:nh].copy(), hp[:nh].copy(), bool(rep.converged),
                               float(rep.true_relative_residual))

    def event_record(self, slot: int):
        A.check(self.L.gnw_event_record(self.h, slot))

    def event_elapsed(self, a: int, b: int) -> float:
        s = C.c_double()
        A.check(self.L.gnw_event_elapsed(self.h, a, b, C.byref(s)))
        return s.value

    def profile_kernel(self, name: str, reps: int = 10):
        """(seconds per launch, algorithmic bytes-or-flops per launch) of one hot kernel."""
        sec, alg = C.c_double(), C.c_double()
        A.check(self.L.gnw_profile_kernel(self.h, A.KERNELS[name], reps, C.byref(sec), C.byref(alg)))
        return sec.value, alg.value

    # ------------------------------------------------------------ ERT (C4/C5)
    def set_electrodes(self, nodes):
        """Mesh::electrode_nodes (mesh.hpp:32) of the assembled mesh."""
        nodes = np.ascontiguousarray(nodes, dtype=np.int64)
        A.check(self.L.gnw_set_electrodes(self.h, nodes.ctypes.data, len(nodes)))
        self.n_electrodes = len(nodes)

    def response_jacobian(self, model, cfgs, tol: float = 1e-14, J_out=None, g_out=None):
        """evaluate_response_and_jacobian (forward.cpp:100-172) -> (g, J, stats).

        ``cfgs``: dict of arrays a, b, m, n, k (b = -1: pole at infinity)."""
        nc = len(cfgs["k"])
        arr = (A.ErtConfig * nc)(*[A.ErtConfig(int(cfgs["a"][i]), int(cfgs["b"][i]), int(cfgs["m"][i]),
                                               int(cfgs["n"][i]), float(cfgs["k"][i])) for i in range(nc)])
        model = self._in(model)
        if self.device_pointers:
            import torch
            J = J_out if J_out is not None else torch.empty((nc, self.N), dtype=torch.float64, device="cuda")
            g = g_out if g_out is not None else torch.empty(nc, dtype=torch.float64, device="cuda")
        else:
            J = J_out if J_out is not None else np.zeros((nc, self.N))
            g = g_out if g_out is not None else np.zeros(nc)
        st = A.ErtStats()
        A.check(self.L.gnw_response_jacobian(self.h, _dptr(model), arr, nc, _dptr(J), _dptr(g), tol, C.byref(st)))
        return g, J, {f: getattr(st, f) for f, _ in A.ErtStats._fields_}

    def gauss_newton(self, m0, m_ref, cfgs, g_obs, beta: float = 0.1, max_outer_steps: int = 2,
                     minres_tol: float = 1e-7, minres_maxit: int = 0, algorithm: str = "woodbury",
                     misfit_reduction_tol: float = 0.0, forward_tol: float = 1e-14):
        """gauss_newton (inversion.cpp:187-292), kWoodburyMinres / kLaplaceMinres -> (m, report).

        ``cfgs`` as for ``response_jacobian``; the electrodes come from ``set_electrodes``."""
        nc = len(cfgs["k"])
        arr = (A.ErtConfig * nc)(*[A.ErtConfig(int(cfgs["a"][i]), int(cfgs["b"][i]), int(cfgs["m"][i]),
                                               int(cfgs["n"][i]), float(cfgs["k"][i])) for i in range(nc)])
        alg = {"woodbury": 0, "laplace": 1}[algorithm]
        cfg = A.GnConfig(beta, max_outer_steps, minres_tol, minres_maxit, alg, misfit_reduction_tol, forward_tol)
        m0, m_ref, g_obs = self._in(m0), self._in(m_ref), self._in(g_obs)
        m_out = self._out(self.N, like=m0 if self.device_pointers else None)
        cap = max(1, max_outer_steps)
        steps = (A.GnStep * cap)()
        n_steps, fin = C.c_uint64(), C.c_double()
        A.check(self.L.gnw_gauss_newton(self.h, _dptr(m0), _dptr(m_ref), arr, nc, _dptr(g_obs), C.byref(cfg),
                                        _dptr(m_out), steps, cap, C.byref(n_steps), C.byref(fin)))
        rep = {"steps": [{f: getattr(steps[k], f) for f, _ in A.GnStep._fields_} for k in range(n_steps.value)],
               "final_misfit": fin.value}
        return m_out, rep

    def woodbury_factors(self):
        """(H, L): H = S_hat^-1 J^T (N x m, h_hat layout) and the capacitance Cholesky factor."""
        H = np.zeros((self.N, self.m))
        Lf = np.zeros((self.m, self.m))
        A.check(self.L.gnw_get_woodbury(self.h, H.ctypes.data, Lf.ctypes.data))
        return H, Lf

    def dense_cholesky(self, Cm):
        Cm = A.f64(Cm)
        out = np.zeros_like(Cm)
        A.check(self.L.gnw_dense_cholesky(self.h, Cm.shape[0], Cm.ctypes.data, out.ctypes.data))
        return out

    # ---------------------------------------------------------------- exports
    def export_csr(self, which: int, level: int = 0):
        nr, nc, nnz = C.c_uint64(), C.c_uint64(), C.c_uint64()
        A.check(self.L.gnw_export_csr(self.h, which, level, C.byref(nr), C.byref(nc), C.byref(nnz), None, None, None))
        rp = np.zeros(nr.value + 1, np.int64)
        ci = np.zeros(nnz.value, np.int64)
        va = np.zeros(nnz.value, np.float64)
        A.check(self.L.gnw_export_csr(self.h, which, level, None, None, None, rp.ctypes.data, ci.ctypes.data,
                                      va.ctypes.data))
        return nr.value, nc.value, rp, ci, va

    def export_mesh(self):
        i = self.info()
        nc = self.N
        out = dict(cells=np.zeros(3 * nc, np.int64), edges=np.zeros(2 * i["n_edges"], np.int64),
                   cell_edges=np.zeros(3 * nc, np.int64), cell_edge_signs=np.zeros(3 * nc, np.int32),
                   boundary_edges=np.zeros(i["n_boundary_edges"], np.int64),
                   boundary_tags=np.zeros(i["n_boundary_edges"], np.int32))
        A.check(self.L.gnw_export_mesh(self.h, *(out[k].ctypes.data for k in (
            "cells", "edges", "cell_edges", "cell_edge_signs", "boundary_edges", "boundary_tags"))))
        return out


# ---------------------------------------------------------------------------
# Reference-shaped facade (inversion.hpp / minres.hpp names)
# ---------------------------------------------------------------------------
def geometric_factor(a, b, m, n, dim: int = 2) -> float:
    """geometric_factor (survey.cpp:22-46); b=None: electrode at infinity."""
    L = A.load()
    arr = lambda v: (C.c_double * 3)(*v)
    k = C.c_double()
    A.check(L.gnw_geometric_factor(arr(a), arr(b) if b is not None else None, arr(m), arr(n), dim, C.byref(k)))
    return k.value


def amg_setup(ctx: Context, rowptr, cols, vals, opts: A.AmgOptions | None = None) -> Context:
    return ctx.assemble_amg_csr(rowptr, cols, vals, opts)


def build_woodbury_preconditioner(ctx: Context, J, beta: float) -> dict:
    """Returns the WoodburyBuildTimings (t_H, t_C, t_chol); the factors live on the device."""
    return ctx.set_jacobian(J, beta)


def assemble_gn_rhs(ctx: Context, m, m_ref, g, g_obs):
    return ctx.assemble_rhs(m, m_ref, g, g_obs)


def minres(ctx: Context, b, x0=None, tol: float = 1e-8, maxit: int | None = None):
    return ctx.minres(b, x0, tol, maxit)


# ------------------------------------------------------------ partitioned helpers
def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for gnw_create_partitioned (create on one rank, broadcast)."""
    buf = (C.c_ubyte * 128)()
    A.check(A.load().gnw_nccl_unique_id(buf))
    return bytes(buf)


def partition_cells(n_cells: int, world: int) -> np.ndarray:
    """Cell boundaries of the partitioned solve (gnw_partition_cells): rank r owns [lo[r], lo[r+1])."""
    lo = np.zeros(world + 1, dtype=np.int64)
    A.check(A.load().gnw_partition_cells(n_cells, world, lo.ctypes.data))
    return lo


def partition_saddle(ctx: Context, world: int, rank: int) -> dict:
    """Rank `rank`'s part of the row partition of the saddle system (gnw_partition_saddle; host
    only): own edge / cell counts, local -> global map (own entries then ghosts), halo lists."""
    L = A.load()
    sz = np.zeros(4, dtype=np.uint64)
    A.check(L.gnw_partition_saddle(ctx.h, world, rank, sz.ctypes.data, None, None, None, None))
    ke, nc, ng, ns = (int(v) for v in sz)
    l2g = np.zeros(ke + nc + ng, np.int64)
    ro, so = np.zeros(world + 1, np.int64), np.zeros(world + 1, np.int64)
    si = np.zeros(max(ns, 1), np.int32)
    A.check(L.gnw_partition_saddle(ctx.h, world, rank, sz.ctypes.data, l2g.ctypes.data, ro.ctypes.data,
                                   so.ctypes.data, si.ctypes.data))
    return dict(own_edges=ke, own_cells=nc, ghosts=ng, local_to_global=l2g, recv_off=ro, send_off=so,
                send_idx=si[:ns])


def partition_csr(ctx: Context, world: int, rank: int, which: int):
    """(n_rows, rowptr, cols, vals) of that rank's local Q (0), D (1) or D^T (2)."""
    L = A.load()
    nr, nnz = C.c_uint64(), C.c_uint64()
    A.check(L.gnw_partition_csr(ctx.h, world, rank, which, C.byref(nr), C.byref(nnz), None, None, None))
    rp = np.zeros(nr.value + 1, np.int64)
    ci = np.zeros(max(nnz.value, 1), np.int32)
    va = np.zeros(max(nnz.value, 1), np.float64)
    A.check(L.gnw_partition_csr(ctx.h, world, rank, which, C.byref(nr), C.byref(nnz), rp.ctypes.data,
                                ci.ctypes.data, va.ctypes.data))
    return nr.value, rp, ci[:nnz.value], va[:nnz.value]


def shared_nccl_id() -> bytes:
    """Rank 0's NCCL unique id, broadcast over the initialised torch.distributed group (any
    backend, e.g. gloo for the bootstrap)."""
    import torch.distributed as dist

    obj = [nccl_unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def partitioned_from_torch_distributed(device: int) -> Context:
    """The calling rank's partitioned context (one rank per GPU, NCCL)."""
    import torch.distributed as dist

    nid = shared_nccl_id()
    return Context.partitioned(dist.get_rank(), dist.get_world_size(), nid, device)


def run_ranks(ctxs, fn):
    """Run ``fn(ctx, rank)`` for every in-process rank on its own thread (the collective calls
    of a local group must run concurrently); returns the per-rank results, re-raises the first
    failure."""
    import threading

    out, err = [None] * len(ctxs), [None] * len(ctxs)

    def body(r):
        try:
            out[r] = fn(ctxs[r], r)
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(len(ctxs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    primary = [e for e in err if e is not None and "another rank failed" not in str(e)]
    for e in primary + [e for e in err if e is not None]:
        raise e
    return out
