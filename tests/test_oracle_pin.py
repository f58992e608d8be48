"""Pins the CPU oracle (TEST INFRASTRUCTURE) before it is trusted.

* the plain-C restatement (oracle/gnw_oracle.c) reproduces the golden vectors that the
  UNMODIFIED reference produced (tests/golden/make_golden.py) bit for bit;
* when the reference library is present (oracle/_ref), restatement and reference agree
  bit for bit on further seeded cases, AMG options and error paths;
* the reference's own known answers (single-triangle Q, 2x2 Cholesky).
"""
import os

import numpy as np
import pytest

import orc
from paper_2209_02815_b200 import workload as W

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def test_restatement_matches_golden_mesh_and_assembly(oracles):
    o = oracles["restatement"]
    p2 = orc.Problem.mixed(o, W.unit_square_mesh(2))
    for k, v in p2.mesh_arrays().items():
        assert np.array_equal(v, GOLD[f"n2_{k}"]), k
    # SURVEY 8(a) a1 golden n=2 dump: cell 0 = v(0,1,4) edges (0,1,2) signs (+,+,-)
    m = p2.mesh_arrays()
    assert list(m["cells"][:6]) == [0, 1, 4, 0, 4, 3]
    assert list(m["cell_edges"][:6]) == [0, 1, 2, 2, 3, 4]
    assert list(m["cell_edge_signs"][:6]) == [1, 1, -1, 1, -1, -1]
    p4 = orc.Problem.mixed(o, W.unit_square_mesh(4))
    for which, name in ((0, "Q"), (1, "D"), (2, "S")):
        nr, nc, rp, ci, va = p4.csr(which)
        assert [nr, nc] == list(GOLD[f"n4_{name}_shape"])
        assert np.array_equal(rp, GOLD[f"n4_{name}_rowptr"])
        assert np.array_equal(ci, GOLD[f"n4_{name}_cols"])
        assert np.array_equal(va, GOLD[f"n4_{name}_vals"]), name


def test_restatement_matches_golden_hierarchy_and_vcycle(oracles):
    o = oracles["restatement"]
    p8 = orc.Problem.mixed(o, W.unit_square_mesh(8), orc.AmgOpts.make(coarse_threshold=16))
    assert p8.n_levels == int(GOLD["n8_nlevels"][0])
    for l in range(p8.n_levels):
        for which, name in ((3, "A"), (4, "P")):
            nr, nc, rp, ci, va = p8.csr(which, l)
            assert np.array_equal(rp, GOLD[f"n8_L{l}_{name}_rowptr"])
            assert np.array_equal(ci, GOLD[f"n8_L{l}_{name}_cols"])
            assert np.array_equal(va, GOLD[f"n8_L{l}_{name}_vals"])
        assert np.array_equal(p8.inv_diag(l), GOLD[f"n8_L{l}_invdiag"])
    assert np.array_equal(p8.coarse_cholesky(), GOLD["n8_coarse_chol"])
    assert np.array_equal(p8.amg_apply(GOLD["n8_vcycle_in"]), GOLD["n8_vcycle_out"])


def test_restatement_matches_golden_woodbury_minres(oracles):
    o = oracles["restatement"]
    p8 = orc.Problem.mixed(o, W.unit_square_mesh(8), orc.AmgOpts.make(coarse_threshold=16))
    p8.set_jacobian(GOLD["n8_J"], float(GOLD["n8_beta"][0]))
    assert np.array_equal(p8.H(), GOLD["n8_H"])
    assert np.array_equal(p8.L(), GOLD["n8_L"])
    assert np.array_equal(p8.apply_operator(GOLD["n8_x"]), GOLD["n8_Ax"])
    assert np.array_equal(p8.precondition(GOLD["n8_x"]), GOLD["n8_Px"])
    b = p8.assemble_rhs(GOLD["n8_dm"], np.zeros(p8.N), GOLD["n8_dg"], np.zeros(4))
    assert np.array_equal(b, GOLD["n8_rhs"])
    x, rep = p8.minres(b, tol=1e-10)
    assert rep["iterations"] == int(GOLD["n8_iters"][0])
    assert np.array_equal(x, GOLD["n8_sol"])
    assert np.array_equal(rep["relative_residuals"], GOLD["n8_hist_e"])
    assert np.array_equal(rep["pnorm_relative_residuals"], GOLD["n8_hist_p"])


def test_known_answers(oracles):
    o = oracles["restatement"]
    assert np.array_equal(o.dense_cholesky(np.array([[4.0, 2.0], [2.0, 5.0]])), GOLD["chol22_L"])
    assert np.array_equal(GOLD["chol22_L"], np.array([[2.0, 0.0], [1.0, 2.0]]))
    tri = W.Mesh(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]), np.array([[0, 1, 2]], dtype=np.int64))
    p = orc.Problem.mixed(o, tri)
    assert p.K == 3 and p.N == 1
    nr, nc, rp, ci, va = p.csr(0)
    Qd = np.zeros((nr, nc))
    for i in range(nr):
        Qd[i, ci[rp[i]:rp[i + 1]]] = va[rp[i]:rp[i + 1]]
    assert np.array_equal(Qd, GOLD["tri_Q"])
    # test_fem_mixed.cpp:30-43 exact values (edge numbering of this triangle)
    expect = np.array([[1 / 3, 0.0, 1 / 6], [0.0, 1 / 6, 0.0], [1 / 6, 0.0, 1 / 3]])
    assert np.allclose(np.abs(Qd), expect, atol=1e-15)
    # K = 5 for n = 1 (test_fem_mixed.cpp:45-50); unit_square(5): K + N = 85 + 50
    assert orc.Problem.mixed(o, W.unit_square_mesh(1)).K == 5
    p5 = orc.Problem.mixed(o, W.unit_square_mesh(5))
    assert (p5.K, p5.N) == (85, 50)


@pytest.mark.parametrize("n,m,thr,strength", [(3, 2, 64, 0.08), (16, 6, 8, 0.08), (32, 8, 64, 0.0),
                                              (24, 5, 16, 0.1)])
def test_restatement_equals_reference(oracles, n, m, thr, strength):
    if "reference" not in oracles:
        pytest.skip("reference library not built (needs /root/reference)")
    opts = orc.AmgOpts.make(coarse_threshold=thr, strength=strength)
    mesh = W.unit_square_mesh(n)
    A = orc.Problem.mixed(oracles["reference"], mesh, opts)
    B = orc.Problem.mixed(oracles["restatement"], mesh, opts)
    assert A.n_levels == B.n_levels
    for l in range(A.n_levels):
        for which in (3, 4):
            for x, y in zip(A.csr(which, l), B.csr(which, l)):
                assert np.array_equal(np.asarray(x), np.asarray(y))
    inp = W.gnstep_inputs(n, m, 3)
    for alpha in (1e-3, 1.0):
        A.set_jacobian(inp.J, alpha)
        B.set_jacobian(inp.J, alpha)
        assert np.array_equal(A.H(), B.H()) and np.array_equal(A.L(), B.L())
        b = A.assemble_rhs(inp.dm, np.zeros(A.N), inp.dg, np.zeros(m))
        xa, ra = A.minres(b, tol=1e-9)
        xb, rb = B.minres(b, tol=1e-9)
        assert ra["iterations"] == rb["iterations"] and np.array_equal(xa, xb)
    # Laplace-only preconditioner (Alg. 4)
    A.set_jacobian(inp.J, 0.3, laplace_pc=True)
    B.set_jacobian(inp.J, 0.3, laplace_pc=True)
    b = A.assemble_rhs(inp.dm, np.zeros(A.N), inp.dg, np.zeros(m))
    xa, ra = A.minres(b, tol=1e-9)
    xb, rb = B.minres(b, tol=1e-9)
    assert ra["iterations"] == rb["iterations"] and np.array_equal(xa, xb)


def test_error_paths_match_reference(oracles):
    kinds = [k for k in ("restatement", "reference") if k in oracles]
    for k in kinds:
        o = oracles[k]
        # degenerate cell (mesh.cpp:104)
        bad = W.Mesh(np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]]), np.array([[0, 1, 2]], dtype=np.int64))
        with pytest.raises(ValueError, match="degenerate cell"):
            orc.Problem.mixed(o, bad)
        p = orc.Problem.mixed(o, W.unit_square_mesh(3))
        n = p.K + p.N
        with pytest.raises(ValueError, match="tol must be positive"):
            p.minres(np.ones(n), tol=0.0)
        with pytest.raises(ValueError, match="beta <= 0"):
            p.set_jacobian(np.ones((2, p.N)), 0.0)
        # non-symmetric AMG input (amg.cpp:119-120)
        with pytest.raises(ValueError, match="not symmetric"):
            orc.Problem.amg_csr(o, np.array([0, 2, 3]), np.array([0, 1, 1]), np.array([2.0, 1.0, 2.0]))
        # the survey's AMG caveat (filtered diagonal <= 0, amg.cpp:142-166 -> :81-88); strong
        # lumping at n = 24, strength 0.25 hits the same failure in both implementations
        with pytest.raises(ValueError, match="non-positive diagonal entry"):
            orc.Problem.mixed(o, W.unit_square_mesh(24), orc.AmgOpts.make(coarse_threshold=16, strength=0.25))
    # b = 0: converged with zero iterations and a zero solution (minres.cpp:32-39)
    p = orc.Problem.mixed(oracles["restatement"], W.unit_square_mesh(3))
    x, rep = p.minres(np.zeros(p.K + p.N), tol=1e-8)
    assert rep["converged"] and rep["iterations"] == 0 and np.all(x == 0)
