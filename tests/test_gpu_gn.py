"""gauss_newton on the device (inversion.cpp:187-292) against the
unmodified reference's gauss_newton (oracle/_ref) or, where that is not built, the pinned
restatement composition."""
import numpy as np
import pytest

import orc
from paper_2209_02815_b200 import Context, workload as W

pytestmark = pytest.mark.gpu


def gn_case(n=32, n_ele=8, first=2, step=4):
    mesh = W.unit_square_mesh(n)
    nodes = np.array([first + step * e for e in range(n_ele)], dtype=np.int64)
    sv = W.ert_survey(n_ele, mesh.vertices[nodes, 0])
    m_true = W.conductivity_model(mesh, 3)
    m0 = np.full(mesh.n_cells, float(np.mean(m_true)))
    return mesh, nodes, sv, m_true, m0


def oracle_gn(oracle, mesh, nodes, sv, g_obs, m0, **kw):
    p = orc.Problem.mixed(oracle, mesh)
    if oracle.kind == "reference":
        return p.gauss_newton_reference(nodes, sv, g_obs, m0, m0, **kw)
    return p.gauss_newton(nodes, sv, g_obs, m0, m0, **kw)


@pytest.mark.parametrize("algorithm,mode,tol", [("woodbury", "reference", 1e-10), ("woodbury", "auto", 1e-10),
                                                ("woodbury", "fused", 1e-8), ("woodbury", "lean", 1e-8),
                                                ("woodbury", "lean", 1e-10), ("woodbury", "fused", 1e-10),
                                                ("laplace", "auto", 1e-10)])
def test_gauss_newton_matches_reference(oracle, algorithm, mode, tol):
    mesh, nodes, sv, m_true, m0 = gn_case()
    p = orc.Problem.mixed(oracle, mesh)
    g_obs, _ = p.response_jacobian(nodes, sv, m_true)
    kw = dict(beta=0.1, max_outer_steps=3, minres_tol=tol, algorithm=algorithm)
    m_r, rep_r = oracle_gn(oracle, mesh, nodes, sv, g_obs, m0, **kw)
    c = Context(0)
    c.set_loop_mode(mode)  # Laplace-only preconditioning always runs the reference schedule
    c.assemble(mesh)
    c.set_electrodes(nodes)
    m_g, rep_g = c.gauss_newton(m0, m0, sv, g_obs, **kw)
    restarts = c.stats()["loop_restarts"]
    print("device", [s["minres_iters"] for s in rep_g["steps"]], "restarts", restarts,
          "reference", [s["minres_iters"] for s in rep_r["steps"]])
    assert len(rep_g["steps"]) == len(rep_r["steps"]) == 3
    for a, b in zip(rep_g["steps"], rep_r["steps"]):
        assert a["misfit"] == pytest.approx(b["misfit"], rel=1e-8)
        # J comes from each side's own forward solve (device PCG to 1e-14 vs the reference's
        # exact factorisation), so the solves do not see identical inputs: +-1 iteration for
        # Woodbury; the slowly converging Laplace-preconditioned solve gets 5 %
        slack = 1 if algorithm == "woodbury" else max(1, int(0.05 * b["minres_iters"]))
        if mode in ("fused", "lean") and tol < 1e-8:
            # below 1e-8 the identity-based schedules can stop a couple of iterations off the
            # literal one (measured: 74 vs 76 at step 2); that is why GNW_LOOP_AUTO keeps the
            # reference schedule there.  Solutions and misfits still match (asserted below).
            slack = 3
        assert abs(a["minres_iters"] - b["minres_iters"]) <= slack
        assert a["converged"] and b["converged"]
        assert a["euclid_relative_residual"] <= 10 * tol
    assert restarts == 0
    assert rep_g["final_misfit"] == pytest.approx(rep_r["final_misfit"], rel=1e-6)
    assert np.linalg.norm(m_g - m_r) <= 1e-6 * np.linalg.norm(m_r)
    if algorithm == "woodbury":
        assert all(s["t_H"] > 0 for s in rep_g["steps"])


def test_gauss_newton_early_exit_and_errors(oracle):
    mesh, nodes, sv, m_true, m0 = gn_case()
    p = orc.Problem.mixed(oracle, mesh)
    g_obs, _ = p.response_jacobian(nodes, sv, m_true)
    c = Context(0)
    c.assemble(mesh)
    with pytest.raises(ValueError, match="missing mesh or survey"):
        c.gauss_newton(m0, m0, sv, g_obs)
    c.set_electrodes(nodes)
    with pytest.raises(ValueError, match="beta must be positive"):
        c.gauss_newton(m0, m0, sv, g_obs, beta=0.0)
    # a huge reduction requirement stops after the second step (inversion.cpp:280-283)
    _, rep = c.gauss_newton(m0, m0, sv, g_obs, max_outer_steps=6, misfit_reduction_tol=0.999)
    assert len(rep["steps"]) == 2
