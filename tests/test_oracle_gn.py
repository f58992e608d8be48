"""gauss_newton (inversion.cpp:187-292): the oracle restatement (orc.Problem.gauss_newton,
composed from the pinned pieces) against the unmodified reference's own gauss_newton."""
import numpy as np
import pytest

import orc
from paper_2209_02815_b200 import workload as W


def gn_case(n=16, n_ele=6, first=2, step=2):
    mesh = W.unit_square_mesh(n)
    nodes = np.array([first + step * e for e in range(n_ele)], dtype=np.int64)
    sv = W.ert_survey(n_ele, mesh.vertices[nodes, 0])
    m_true = W.conductivity_model(mesh, 3)
    m0 = np.full(mesh.n_cells, float(np.mean(m_true)))
    return mesh, nodes, sv, m_true, m0


@pytest.mark.parametrize("algorithm", ["woodbury", "laplace"])
def test_gauss_newton_restatement_matches_reference(oracles, algorithm):
    if "reference" not in oracles:
        pytest.skip("reference library not built here")
    mesh, nodes, sv, m_true, m0 = gn_case()
    pr = orc.Problem.mixed(oracles["reference"], mesh)
    g_obs, _ = pr.response_jacobian(nodes, sv, m_true)
    kw = dict(beta=0.1, max_outer_steps=2, minres_tol=1e-10, algorithm=algorithm)
    m_ref_run, rep_ref = pr.gauss_newton_reference(nodes, sv, g_obs, m0, m0, **kw)
    ps = orc.Problem.mixed(oracles["restatement"], mesh)
    m_res, rep_res = ps.gauss_newton(nodes, sv, g_obs, m0, m0, **kw)
    assert len(rep_ref["steps"]) == len(rep_res["steps"]) == 2
    for a, b in zip(rep_ref["steps"], rep_res["steps"]):
        assert a["misfit"] == pytest.approx(b["misfit"], rel=1e-10)
        assert abs(a["minres_iters"] - b["minres_iters"]) <= 1
        assert a["converged"] and b["converged"]
    assert rep_ref["final_misfit"] == pytest.approx(rep_res["final_misfit"], rel=1e-8)
    assert np.linalg.norm(m_res - m_ref_run) <= 1e-8 * np.linalg.norm(m_ref_run)
    # the inversion makes progress on this well-posed toy problem
    assert rep_ref["final_misfit"] < rep_ref["steps"][0]["misfit"]
