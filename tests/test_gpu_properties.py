"""The reference's own property tests for this path, run through the
C-ABI on the GPU: MINRES (test_minres.cpp), the SA-AMG V-cycle (test_amg.cpp) and the
saddle operator / Woodbury preconditioner / rhs (test_inversion.cpp).  Each test cites the
reference test it restates; tolerances are the reference's."""
import numpy as np
import pytest

from paper_2209_02815_b200 import AmgOptions, Context, workload as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small():
    """unit_square(16), m = 8: K + N = 816 + 512."""
    inp = W.gnstep_inputs(16, 8, 0)
    c = Context(0)
    c.assemble(inp.mesh)
    return c, inp


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def test_saddle_operator_is_symmetric(small):
    """test_inversion.cpp:167-186: <A x, y> = <x, A y> within 1e-11 (with and without J)."""
    c, inp = small
    n = c.K + c.N
    x, y = W.gaussian(21, n), W.gaussian(22, n)
    for J in (None, inp.J):
        c.set_jacobian(J, 0.3)
        ax, ay = c.apply_operator(x), c.apply_operator(y)
        assert abs(ax @ y - x @ ay) <= 1e-11 * max(abs(ax @ y), 1.0)


def test_capacitance_is_identity_without_sensitivity(small):
    """test_inversion.cpp:188-206: J = 0 gives C = I, so chol(C) = I."""
    c, inp = small
    c.set_jacobian(np.zeros_like(inp.J), 0.5)
    H, L = c.woodbury_factors()
    assert np.all(H == 0.0)
    assert np.array_equal(L, np.eye(inp.J.shape[0]))


def test_woodbury_apply_zero_spd_and_beta_limit(small):
    """test_inversion.cpp:208-280: P^-1 0 = 0; <P^-1 y, y> > 0; as beta -> inf the Woodbury
    correction vanishes and P^-1 tends to the plain Laplace preconditioner."""
    c, inp = small
    n = c.K + c.N
    c.set_jacobian(inp.J, 0.1)
    assert np.all(c.precondition(np.zeros(n)) == 0.0)
    for s in range(3):
        y = W.gaussian(30 + s, n)
        assert c.precondition(y) @ y > 0.0
    y = W.gaussian(40, n)
    c.set_jacobian(inp.J, 1e12)
    zw = c.precondition(y)
    c.set_jacobian(inp.J, 1e12, laplace_pc=True)
    zl = c.precondition(y)
    assert rel(zw, zl) <= 1e-9


def test_rhs_zero_and_beta_halving(small):
    """test_inversion.cpp:44-95: m = m_ref and g = g_obs give b = 0; halving beta doubles the
    data block J^T (g - g_obs) / beta and leaves the model block alone."""
    c, inp = small
    m_ = inp.J.shape[0]
    c.set_jacobian(inp.J, 0.2)
    mdl, g = W.gaussian(50, c.N), W.gaussian(51, m_)
    assert np.all(c.assemble_rhs(mdl, mdl, g, g) == 0.0)
    b1 = c.assemble_rhs(mdl, np.zeros(c.N), g, np.zeros(m_))
    c.set_jacobian(inp.J, 0.1)
    b2 = c.assemble_rhs(mdl, np.zeros(c.N), g, np.zeros(m_))
    assert np.array_equal(b2[:c.K], b1[:c.K])
    assert np.array_equal(b2[c.K:], 2.0 * b1[c.K:])  # x / (beta / 2) == 2 (x / beta) exactly


def test_minres_preconditioned_residuals_do_not_increase(small):
    """test_minres.cpp:82-102: the recurred P-norm residual history is non-increasing (+1e-12);
    test_minres.cpp:104-135: on convergence the true residual is within 10 tol."""
    c, inp = small
    c.set_jacobian(inp.J, 0.05)
    b = c.assemble_rhs(inp.dm, np.zeros(c.N), inp.dg, np.zeros(inp.J.shape[0]))
    x, rep = c.minres(b, tol=1e-12)
    hp = np.asarray(rep.pnorm_relative_residuals)
    assert rep.converged and len(hp) == rep.iterations + 1
    assert np.all(np.diff(hp) <= 1e-12)
    assert np.all(np.isfinite(rep.relative_residuals))
    assert rep.true_relative_residual <= 10 * 1e-12


def test_minres_repeatable_and_linear(small):
    """test_amg.cpp:154-167 / test_minres.cpp style: the same solve twice gives the same bits;
    the solve is linear in b up to the tolerance."""
    c, inp = small
    c.set_jacobian(inp.J, 0.05)
    n = c.K + c.N
    b1, b2 = W.gaussian(60, n), W.gaussian(61, n)
    x1, r1 = c.minres(b1, tol=1e-12)
    x1b, r1b = c.minres(b1, tol=1e-12)
    assert r1.iterations == r1b.iterations and np.array_equal(x1, x1b)
    x2, _ = c.minres(b2, tol=1e-12)
    x3, _ = c.minres(2.0 * b1 - b2, tol=1e-12)
    assert rel(x3, 2.0 * x1 - x2) <= 1e-8


def test_vcycle_reduces_poisson_error():
    """test_amg.cpp:120-137: default AmgOptions on 2D Poisson 24^2; 30 steps of power iteration
    on the error propagator E = I - B A in the A-norm give rho <= 0.7."""
    n = 24
    idx = lambda i, j: j * n + i  # noqa: E731
    rows, cols, vals = [], [], []
    for j in range(n):
        for i in range(n):
            ent = [(idx(i, j), 4.0)]
            if i > 0: ent.append((idx(i - 1, j), -1.0))  # noqa: E701
            if i + 1 < n: ent.append((idx(i + 1, j), -1.0))  # noqa: E701
            if j > 0: ent.append((idx(i, j - 1), -1.0))  # noqa: E701
            if j + 1 < n: ent.append((idx(i, j + 1), -1.0))  # noqa: E701
            for cc, v in sorted(ent):
                rows.append(idx(i, j)); cols.append(cc); vals.append(v)  # noqa: E702
    rowptr = np.zeros(n * n + 1, np.int64)
    np.add.at(rowptr, np.array(rows) + 1, 1)
    rowptr = np.cumsum(rowptr)
    cols, vals = np.array(cols, np.int64), np.array(vals)
    A = np.zeros((n * n, n * n))
    A[np.array(rows), cols] = vals
    for exact in (True, False):
        c = Context(0)
        c.set_coarse_mode(exact)
        c.assemble_amg_csr(rowptr, cols, vals, AmgOptions())
        e = W.gaussian(70, n * n)
        rho = 0.0
        for _ in range(30):
            before = np.sqrt(e @ (A @ e))
            e = e - c.amg_apply(A @ e)
            after = np.sqrt(e @ (A @ e))
            rho = after / before
            if after > 0.0:
                e = e / after
        assert rho <= 0.7, rho
