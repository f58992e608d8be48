"""The default-mode V-cycle with one pass per level each way (vcycle_fused.cu: r_c = T^T r,
e = S r + T e_c with T = (I - Wd A) P, S = 2 Wd - Wd A Wd; host::fused_cycle_ops) is the same
linear operator as amg.cpp:90-111's four passes per level: against the reference oracle and
against the four-pass kernels (GNW_VC_FUSED=0), single right-hand side and the Woodbury setup's
multi-RHS cycle (H = S^-1 J^T)."""
import numpy as np
import pytest

import orc
from paper_2209_02815_b200 import AmgOptions, Context, workload as W

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def ctx(monkeypatch, mesh, fused, opts=None):
    monkeypatch.setenv("GNW_VC_FUSED", "1" if fused else "0")
    c = Context(0)
    c.assemble(mesh, opts)
    return c


@pytest.mark.parametrize("n,thr", [(16, 64), (64, 64), (256, 64), (512, 64)])
def test_fused_vcycle_matches_reference_and_four_pass(monkeypatch, oracle, n, thr):
    mesh = W.unit_square_mesh(n)
    a, b = ctx(monkeypatch, mesh, True, AmgOptions(coarse_threshold=thr)), ctx(monkeypatch, mesh, False,
                                                                                 AmgOptions(coarse_threshold=thr))
    p = orc.Problem.mixed(oracle, mesh, orc.AmgOpts.make(coarse_threshold=thr))
    for seed in range(2):
        r = W.gaussian(400 + seed, a.N)
        za, zb, zr = a.amg_apply(r), b.amg_apply(r), p.amg_apply(r)
        assert rel(za, zr) <= 1e-13 and rel(zb, zr) <= 1e-13 and rel(za, zb) <= 1e-13


def test_fused_batched_setup_matches_four_pass(monkeypatch, oracle):
    n, m = 128, 40  # m not a multiple of the batch: an odd tail batch
    inp = W.gnstep_inputs(n, m, 0)
    a, b = ctx(monkeypatch, inp.mesh, True), ctx(monkeypatch, inp.mesh, False)
    for c in (a, b):
        c.set_jacobian(inp.J, 1e-2)
    Ha, La = a.woodbury_factors()
    Hb, Lb = b.woodbury_factors()
    p = orc.Problem.mixed(oracle, inp.mesh)
    p.set_jacobian(inp.J, 1e-2)
    assert rel(Ha, p.H()) <= 1e-13 and rel(Ha, Hb) <= 1e-13
    assert rel(np.tril(La), np.tril(Lb)) <= 1e-12
    ba = a.assemble_rhs(inp.dm, np.zeros(a.N), inp.dg, np.zeros(m))
    xa, ra = a.minres(ba, tol=1e-10)
    xb, rb = b.minres(ba, tol=1e-10)
    assert abs(ra.iterations - rb.iterations) <= 1 and rel(xa, xb) <= 1e-8


def jittered_mesh(n, seed, amp=0.25):
    """unit_square_mesh(n) with its interior vertices moved by up to amp / n: no two level-operator
    entries share a value, so the coded lane-ELL tables are as large as the matrices."""
    mesh = W.unit_square_mesh(n)
    v = mesh.vertices.copy()
    rng = np.random.default_rng(seed)
    interior = (v[:, 0] > 0) & (v[:, 0] < 1) & (v[:, 1] > 0) & (v[:, 1] < 1)
    v[interior] += rng.uniform(-amp / n, amp / n, size=(int(interior.sum()), 2))
    return W.Mesh(np.ascontiguousarray(v), mesh.cells)


@pytest.mark.parametrize("make", ["unit", "jittered"])
def test_lane_ell_levels_bitwise_csr(monkeypatch, oracle, make):
    """The lane-ELL level kernels with coded 32-bit entries (k_vcl_*) against the CSR kernels they
    replace (GNW_VC_LELL=0, still the fallback for operators whose entries do not fit): the same
    sums in the same order, bit for bit -- on the structured mesh (a few distinct values per
    operator) and on a jittered one (every entry its own table slot), where the whole GN-step
    solve is also checked against the oracle."""
    n, m = 40, 12
    mesh = W.unit_square_mesh(n) if make == "unit" else jittered_mesh(n, 3)
    monkeypatch.setenv("GNW_VC_LELL", "1")
    a = Context(0)
    a.assemble(mesh)
    monkeypatch.setenv("GNW_VC_LELL", "0")
    b = Context(0)
    b.assemble(mesh)
    p = orc.Problem.mixed(oracle, mesh)
    for seed in range(3):
        r = W.gaussian(700 + seed, a.N)
        za, zb = a.amg_apply(r), b.amg_apply(r)
        assert np.array_equal(za, zb)
        assert rel(za, p.amg_apply(r)) <= 1e-12
    J = W.synthetic_jacobian(m, mesh.n_cells, 5)
    a.set_jacobian(J, 1e-2)
    p.set_jacobian(J, 1e-2)
    bvec = p.assemble_rhs(W.gaussian(1, a.N), np.zeros(a.N), W.gaussian(2, m), np.zeros(m))
    xr6, rr6 = p.minres(bvec, tol=1e-6)
    xr, rr = p.minres(bvec, tol=1e-10)
    for mode in ("lean", "persistent"):
        a.set_loop_mode(mode)
        x6, rep6 = a.minres(bvec, tol=1e-6)
        assert rep6.converged and abs(rep6.iterations - rr6["iterations"]) <= 1
        # near 1e-10 the recurred residual of the jittered problem plateaus (5.97e-11, 5.95e-11,
        # 3.6e-11 ...) and rounding decides where it crosses: the solutions are the bar there
        x, rep = a.minres(bvec, tol=1e-10)
        assert rep.converged and abs(rep.iterations - rr["iterations"]) <= 3
        assert rel(x, xr) <= 1e-8
