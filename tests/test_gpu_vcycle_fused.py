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
