"""ctypes binding of the CPU oracles (orc_api.h).  TEST INFRASTRUCTURE ONLY.

``Oracle("restatement")`` loads oracle/build/liborc.so (plain-C restatement);
``Oracle("reference")`` loads oracle/_ref/libertinv_ref.so (the unmodified reference
sources compiled by oracle/Makefile).  Both expose the same API.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restatement": os.path.join(HERE, "build", "liborc.so"),
    "reference": os.path.join(HERE, "_ref", "libertinv_ref.so"),
}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u64 = C.c_uint64


class AmgOpts(C.Structure):
    """AmgOptions, proj/include/ertinv/amg.hpp:11-23 (exact_solve not exposed)."""

    _fields_ = [
        ("coarse_threshold", C.c_uint64),
        ("strength", C.c_double),
        ("jacobi_damping", C.c_double),
        ("prolongation_damping", C.c_double),
        ("max_aggregate_size", C.c_uint64),
        ("max_levels", C.c_uint64),
    ]

    @classmethod
    def make(cls, coarse_threshold=64, strength=0.08, jacobi_damping=2.0 / 3.0,
             prolongation_damping=2.0 / 3.0, max_aggregate_size=3, max_levels=25):
        return cls(coarse_threshold, strength, jacobi_damping, prolongation_damping,
                   max_aggregate_size, max_levels)


class MinresReport(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("converged", C.c_int32),
                ("true_relative_residual", C.c_double), ("n_hist", C.c_uint64)]


class OracleError(RuntimeError):
    pass


def build(kind: str) -> None:
    target = "restatement" if kind == "restatement" else "ref"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


class Oracle:
    def __init__(self, kind: str = "restatement"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        self.kind = kind
        L = C.CDLL(path)
        self.L = L
        L.orc_last_error.restype = C.c_char_p
        L.orc_flavor.restype = C.c_char_p
        L.orc_create_mixed.restype = C.c_void_p
        L.orc_create_mixed.argtypes = [_dp, _u64, _i64p, _u64, C.POINTER(AmgOpts)]
        L.orc_create_amg_csr.restype = C.c_void_p
        L.orc_create_amg_csr.argtypes = [_u64, _i64p, _i64p, _dp, C.POINTER(AmgOpts)]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_sizes.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(dtype=np.uint64)]
        L.orc_mesh.argtypes = [C.c_void_p] + [C.c_void_p] * 6
        L.orc_csr.argtypes = [C.c_void_p, C.c_int, _u64, C.POINTER(_u64), C.POINTER(_u64),
                              C.POINTER(_u64), C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_level_inv_diag.argtypes = [C.c_void_p, _u64, _dp]
        L.orc_coarse_cholesky.argtypes = [C.c_void_p, _dp]
        L.orc_q_diag_inv.argtypes = [C.c_void_p, _dp]
        L.orc_amg_apply.argtypes = [C.c_void_p, _dp, _dp]
        L.orc_set_jacobian.argtypes = [C.c_void_p, C.c_void_p, _u64, C.c_double, _dp]
        L.orc_set_pc_laplace.argtypes = [C.c_void_p, C.c_int]
        L.orc_get_H.argtypes = [C.c_void_p, _dp]
        L.orc_get_L.argtypes = [C.c_void_p, _dp]
        L.orc_apply_operator.argtypes = [C.c_void_p, _dp, _dp]
        L.orc_precondition.argtypes = [C.c_void_p, _dp, _dp]
        L.orc_assemble_rhs.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp]
        L.orc_minres.argtypes = [C.c_void_p, _dp, _dp, C.c_double, _u64, _dp,
                                 C.POINTER(MinresReport), _dp, _dp, _u64]
        L.orc_dense_cholesky.argtypes = [_u64, _dp, _dp]

    def err(self, rc: int):
        msg = self.L.orc_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise OracleError(msg)

    def check(self, rc: int):
        if rc:
            self.err(rc)

    def geometric_factor(self, a, b, m, n, dim=2) -> float:
        fn = self.L.orc_geometric_factor
        arr = lambda v: (C.c_double * 3)(*v)
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_double)]
        k = C.c_double()
        bb = arr(b) if b is not None else None
        self.check(fn(arr(a), bb, arr(m), arr(n), dim, C.byref(k)))
        return k.value

    def dense_cholesky(self, Cm: np.ndarray) -> np.ndarray:
        Cm = np.ascontiguousarray(Cm, dtype=np.float64)
        out = np.zeros_like(Cm)
        self.check(self.L.orc_dense_cholesky(Cm.shape[0], Cm, out))
        return out


class Problem:
    """A mixed RT0 x P0 problem (mesh -> Q, D, S_hat, AMG) held by one oracle."""

    def __init__(self, oracle: Oracle, handle):
        self.o = oracle
        self.h = handle
        s = np.zeros(8, dtype=np.uint64)
        oracle.L.orc_sizes(self.h, s)
        (self.K, self.N, self.n_vertices, self.n_cells, self.n_edges, self.n_levels,
         self.n_boundary, self.n_coarse) = (int(v) for v in s)
        self.m = 0

    @classmethod
    def mixed(cls, oracle: Oracle, mesh, opts: AmgOpts | None = None):
        v = np.ascontiguousarray(mesh.vertices, dtype=np.float64).ravel()
        c = np.ascontiguousarray(mesh.cells, dtype=np.int64).ravel()
        h = oracle.L.orc_create_mixed(v, mesh.n_vertices, c, mesh.n_cells,
                                      C.byref(opts) if opts is not None else None)
        if not h:
            msg = oracle.L.orc_last_error().decode()
            if "non-positive" in msg or "invalid" in msg or "range" in msg or "degenerate" in msg:
                raise ValueError(msg)
            raise OracleError(msg)
        return cls(oracle, h)

    @classmethod
    def amg_csr(cls, oracle: Oracle, rowptr, cols, vals, opts: AmgOpts | None = None):
        rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        h = oracle.L.orc_create_amg_csr(len(rowptr) - 1, rowptr,
                                        np.ascontiguousarray(cols, dtype=np.int64),
                                        np.ascontiguousarray(vals, dtype=np.float64),
                                        C.byref(opts) if opts is not None else None)
        if not h:
            raise ValueError(oracle.L.orc_last_error().decode())
        return cls(oracle, h)

    def __del__(self):
        if getattr(self, "h", None):
            self.o.L.orc_destroy(self.h)
            self.h = None

    # -- structure ---------------------------------------------------------
    def mesh_arrays(self):
        nc, ne, nb = self.n_cells, self.n_edges, self.n_boundary
        out = dict(cells=np.zeros(3 * nc, np.int64), edges=np.zeros(2 * ne, np.int64),
                   cell_edges=np.zeros(3 * nc, np.int64), cell_edge_signs=np.zeros(3 * nc, np.int32),
                   boundary_edges=np.zeros(nb, np.int64), boundary_tags=np.zeros(nb, np.int32))
        a = [out[k].ctypes.data for k in ("cells", "edges", "cell_edges", "cell_edge_signs",
                                          "boundary_edges", "boundary_tags")]
        self.o.check(self.o.L.orc_mesh(self.h, *a))
        return out

    def csr(self, which: int, level: int = 0):
        nr, ncol, nnz = _u64(), _u64(), _u64()
        self.o.check(self.o.L.orc_csr(self.h, which, level, C.byref(nr), C.byref(ncol),
                                      C.byref(nnz), None, None, None))
        rp = np.zeros(nr.value + 1, np.int64)
        ci = np.zeros(nnz.value, np.int64)
        va = np.zeros(nnz.value, np.float64)
        self.o.check(self.o.L.orc_csr(self.h, which, level, None, None, None, rp.ctypes.data,
                                      ci.ctypes.data, va.ctypes.data))
        return nr.value, ncol.value, rp, ci, va

    def inv_diag(self, level: int) -> np.ndarray:
        n = self.csr(3, level)[0]
        out = np.zeros(n)
        self.o.check(self.o.L.orc_level_inv_diag(self.h, level, out))
        return out

    def coarse_cholesky(self) -> np.ndarray:
        out = np.zeros(self.n_coarse * self.n_coarse)
        self.o.check(self.o.L.orc_coarse_cholesky(self.h, out))
        return out.reshape(self.n_coarse, self.n_coarse)

    def q_diag_inv(self) -> np.ndarray:
        out = np.zeros(self.K)
        self.o.check(self.o.L.orc_q_diag_inv(self.h, out))
        return out

    # -- numerics ------------------------------------------------------------
    def amg_apply(self, r: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros_like(r)
        self.o.check(self.o.L.orc_amg_apply(self.h, r, z))
        return z

    def set_jacobian(self, J: np.ndarray | None, beta: float, laplace_pc: bool = False):
        self.o.check(self.o.L.orc_set_pc_laplace(self.h, 1 if laplace_pc else 0))
        t = np.zeros(3)
        if J is None or J.size == 0:
            self.o.check(self.o.L.orc_set_jacobian(self.h, None, 0, beta, t))
            self.m = 0
        else:
            J = np.ascontiguousarray(J, dtype=np.float64)
            self.o.check(self.o.L.orc_set_jacobian(self.h, J.ctypes.data, J.shape[0], beta, t))
            self.m = J.shape[0]
        self.beta = beta
        return dict(t_H=t[0], t_C=t[1], t_chol=t[2])

    def response_jacobian(self, nodes, cfgs, model):
        """evaluate_response_and_jacobian (forward.cpp:100-172): (g, J)."""
        fn = self.o.L.orc_response_jacobian
        fn.argtypes = [C.c_void_p, _i64p, _u64, _i64p, _i64p, _i64p, _i64p, _dp, _u64, _dp, _dp, _dp]
        nodes = np.ascontiguousarray(nodes, dtype=np.int64)
        cols = [np.ascontiguousarray(cfgs[k], dtype=np.int64) for k in ("a", "b", "m", "n")]
        kk = np.ascontiguousarray(cfgs["k"], dtype=np.float64)
        nc = len(kk)
        J = np.zeros((nc, self.N))
        g = np.zeros(nc)
        self.o.check(fn(self.h, nodes, len(nodes), *cols, kk, nc, np.ascontiguousarray(model, dtype=np.float64),
                        J.ravel(), g))
        return g, J

    def gauss_newton(self, nodes, cfgs, g_obs, m_ref, m0, beta=0.1, max_outer_steps=2, minres_tol=1e-7,
                     minres_maxit=0, algorithm="woodbury", misfit_reduction_tol=0.0):
        """gauss_newton (inversion.cpp:187-292) for the iterative algorithms, composed from this
        oracle's own pieces in the reference's order: misfit = norm2(g - g_obs) (:225-226),
        preconditioner (:244-256), rhs (:259-260), MINRES from x0 = 0 (:261-265), m += x[K:]
        (:275-278), optional early exit (:280-283), final misfit (:286-291)."""
        K, N = self.K, self.N
        maxit = minres_maxit if minres_maxit > 0 else 2 * (K + N)
        m = np.array(m0, dtype=np.float64)
        g_obs = np.asarray(g_obs, dtype=np.float64)
        steps = []

        def misfit(gv):
            d = gv - g_obs
            s = 0.0
            for v in d:  # norm2: sequential dot (linalg.cpp:9-22)
                s += v * v
            return float(np.sqrt(s))

        for step in range(max_outer_steps):
            g, J = self.response_jacobian(nodes, cfgs, m)
            sr = dict(misfit=misfit(g))
            self.set_jacobian(J, beta, laplace_pc=(algorithm == "laplace"))
            b = self.assemble_rhs(m, m_ref, g, g_obs)
            x, rep = self.minres(b, np.zeros(K + N), tol=minres_tol, maxit=maxit)
            sr.update(minres_iters=rep["iterations"], converged=rep["converged"],
                      euclid_relative_residual=rep["true_relative_residual"],
                      pnorm_relative_residual=float(rep["pnorm_relative_residuals"][-1]))
            delta = x[K:]
            if not np.all(np.isfinite(delta)):
                raise RuntimeError("gauss_newton: non-finite model update")
            m = m + delta
            steps.append(sr)
            if misfit_reduction_tol > 0.0 and step > 0:
                if sr["misfit"] > (1.0 - misfit_reduction_tol) * steps[-2]["misfit"]:
                    break
        g, _ = self.response_jacobian(nodes, cfgs, m)
        return m, dict(steps=steps, final_misfit=misfit(g))

    def gauss_newton_reference(self, nodes, cfgs, g_obs, m_ref, m0, beta=0.1, max_outer_steps=2, minres_tol=1e-7,
                               minres_maxit=0, algorithm="woodbury", misfit_reduction_tol=0.0):
        """The unmodified reference gauss_newton (oracle/_ref only), same return shape."""
        fn = self.o.L.orc_gauss_newton
        fn.argtypes = [C.c_void_p, _i64p, _u64, _i64p, _i64p, _i64p, _i64p, _dp, _u64, _dp, _dp, _dp, C.c_double,
                       _u64, C.c_double, _u64, C.c_int, C.c_double, _dp, _dp, _u64, C.POINTER(_u64),
                       C.POINTER(C.c_double)]
        nodes = np.ascontiguousarray(nodes, dtype=np.int64)
        cols = [np.ascontiguousarray(cfgs[k], dtype=np.int64) for k in ("a", "b", "m", "n")]
        kk = np.ascontiguousarray(cfgs["k"], dtype=np.float64)
        f = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        m_out = np.zeros(self.N)
        cap = max(1, max_outer_steps)
        st = np.zeros(5 * cap)
        ns, fin = _u64(), C.c_double()
        self.o.check(fn(self.h, nodes, len(nodes), *cols, kk, len(kk), f(g_obs), f(m_ref), f(m0), beta,
                        max_outer_steps, minres_tol, minres_maxit, 1 if algorithm == "laplace" else 0,
                        misfit_reduction_tol, m_out, st, cap, C.byref(ns), C.byref(fin)))
        steps = [dict(misfit=st[5 * i], minres_iters=int(st[5 * i + 1]), converged=bool(st[5 * i + 2]),
                      euclid_relative_residual=st[5 * i + 3], pnorm_relative_residual=st[5 * i + 4])
                 for i in range(ns.value)]
        return m_out, dict(steps=steps, final_misfit=fin.value)

    def sample_gnstep(self, J: np.ndarray, beta: float, k_cols: int, k_rows: int, k_iters: int) -> dict:
        """Bounded CPU timing sample (reference library only); see orc_api.h."""
        fn = self.o.L.orc_sample_gnstep
        fn.argtypes = [C.c_void_p, C.c_void_p, _u64, C.c_double, _u64, _u64, _u64, _dp]
        J = np.ascontiguousarray(J, dtype=np.float64)
        out = np.zeros(5)
        self.o.check(fn(self.h, J.ctypes.data, J.shape[0], beta, k_cols, k_rows, k_iters, out))
        return dict(t_col=out[0], t_row=out[1], t_chol=out[2], t_iter=out[3], t_minres0=out[4])

    def H(self) -> np.ndarray:
        out = np.zeros(self.N * self.m)
        self.o.check(self.o.L.orc_get_H(self.h, out))
        return out.reshape(self.N, self.m)

    def L(self) -> np.ndarray:
        out = np.zeros(self.m * self.m)
        self.o.check(self.o.L.orc_get_L(self.h, out))
        return out.reshape(self.m, self.m)

    def apply_operator(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        self.o.check(self.o.L.orc_apply_operator(self.h, x, y))
        return y

    def precondition(self, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        z = np.zeros_like(y)
        self.o.check(self.o.L.orc_precondition(self.h, y, z))
        return z

    def assemble_rhs(self, m, m_ref, g, g_obs):
        out = np.zeros(self.K + self.N)
        f = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        self.o.check(self.o.L.orc_assemble_rhs(self.h, f(m), f(m_ref), f(g), f(g_obs), out))
        return out

    def minres(self, b, x0=None, tol=1e-8, maxit=None, hist_cap=100000):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.zeros_like(b) if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        maxit = 2 * b.size if maxit is None else maxit
        x = np.zeros_like(b)
        rep = MinresReport()
        he = np.zeros(hist_cap)
        hp = np.zeros(hist_cap)
        self.o.check(self.o.L.orc_minres(self.h, b, x0, tol, maxit, x, C.byref(rep), he, hp, hist_cap))
        nh = min(int(rep.n_hist), hist_cap)
        return x, dict(iterations=int(rep.iterations), converged=bool(rep.converged),
                       true_relative_residual=rep.true_relative_residual,
                       relative_residuals=he[:nh].copy(), pnorm_relative_residuals=hp[:nh].copy())
