"""ERT forward model on the GPU (row a15: forward.cpp:39-172, survey.cpp:22-46) against the
reference oracle, plus the reference's own property tests (test_forward.cpp)."""
import numpy as np
import pytest

import orc
from paper_2209_02815_b200 import AmgOptions, Context, geometric_factor, workload as W

pytestmark = pytest.mark.gpu


def small_case(n=32, n_ele=8, first=2, step=4, idx=3):
    mesh = W.unit_square_mesh(n)
    nodes = np.array([first + step * e for e in range(n_ele)], dtype=np.int64)
    sv = W.ert_survey(n_ele, mesh.vertices[nodes, 0])
    model = W.conductivity_model(mesh, idx)
    return mesh, nodes, sv, model


def gpu_ert(mesh, nodes):
    c = Context(0)
    c.assemble(mesh)
    c.set_electrodes(nodes)
    return c


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


@pytest.mark.parametrize("n,n_ele,first,step", [(32, 8, 2, 4), (64, 16, 2, 4)])
def test_response_jacobian_matches_reference(oracle, n, n_ele, first, step):
    mesh, nodes, sv, model = small_case(n, n_ele, first, step)
    c = gpu_ert(mesh, nodes)
    g, J, st = c.response_jacobian(model, sv, tol=1e-14)
    p = orc.Problem.mixed(oracle, mesh)
    gr, Jr = p.response_jacobian(nodes, sv, model)
    assert rel(g, gr) <= 1e-10
    assert rel(J, Jr) <= 1e-9
    assert st["pcg_iterations"] > 0
    # row-sum identity J 1 = -g (acceptance.cpp:188-192 form, 1e-10)
    assert np.max(np.abs(J.sum(axis=1) + g)) <= 1e-10 * np.max(np.abs(g))


def test_model_shift_scales_by_exp_minus_t():
    """test_forward.cpp:166-181"""
    mesh, nodes, sv, model = small_case()
    c = gpu_ert(mesh, nodes)
    g0, J0, _ = c.response_jacobian(model, sv)
    t = 0.42
    g1, J1, _ = c.response_jacobian(model + t, sv)
    assert np.allclose(g1, np.exp(-t) * g0, rtol=1e-9, atol=0)
    assert rel(J1, np.exp(-t) * J0) <= 1e-9


def test_jacobian_matches_finite_differences():
    """test_forward.cpp:141-164"""
    mesh, nodes, sv, model = small_case()
    c = gpu_ert(mesh, nodes)
    g, J, _ = c.response_jacobian(model, sv)
    rng = np.random.default_rng(23)
    step = 1e-5
    for cell in rng.integers(0, mesh.n_cells, 3):
        mp, mm = model.copy(), model.copy()
        mp[cell] += step
        mm[cell] -= step
        gp, _, _ = c.response_jacobian(mp, sv)
        gm, _, _ = c.response_jacobian(mm, sv)
        fd = (gp - gm) / (2 * step)
        scale = np.maximum(np.abs(J[:, cell]), 1e-3 * np.abs(g))
        assert np.all(np.abs(fd - J[:, cell]) <= 1e-5 * scale + 1e-12)


def test_errors_match_reference_text():
    mesh, nodes, sv, model = small_case()
    c = gpu_ert(mesh, nodes)
    with pytest.raises(ValueError, match="not a mesh node"):
        c.set_electrodes([mesh.n_vertices - 1])   # top-right corner, z = 1
    c.set_electrodes([0, 4, 8])                    # node 0 is a grounded corner
    sv3 = {"a": np.array([0]), "b": np.array([-1]), "m": np.array([1]), "n": np.array([2]), "k": np.array([1.0])}
    with pytest.raises(ValueError, match="grounded boundary"):
        c.response_jacobian(model, sv3)
    assert geometric_factor((0, 0, 0), None, (2, 0, 0), (4, 0, 0)) == pytest.approx(np.pi / np.log(2.0), rel=1e-14)


def test_c4_gn_step_against_restatement_reduced():
    """A C4-style GN step (ERT J, alpha=1e-2) at n=64 / 16 electrodes: GPU J and the
    oracle J each drive their own solver; iterations within +-1, solutions within 1e-6."""
    mesh, nodes, sv, model = small_case(64, 16, 2, 4)
    c = gpu_ert(mesh, nodes)
    g, J, _ = c.response_jacobian(model, sv)
    noise = W.gaussian(5, len(g))
    g_obs = g * (1 + 0.01 * noise)
    alpha = 1e-2
    c.set_jacobian(J, alpha)
    b = c.assemble_rhs(model, np.zeros(c.N), g, g_obs)
    x, rep = c.minres(b, tol=1e-10)
    oracle = orc.Oracle("restatement")
    p = orc.Problem.mixed(oracle, mesh)
    gr, Jr = p.response_jacobian(nodes, sv, model)
    p.set_jacobian(Jr, alpha)
    br = p.assemble_rhs(model, np.zeros(p.N), gr, gr * (1 + 0.01 * noise))
    xr, rr = p.minres(br, tol=1e-10)
    assert rep.converged and rr["converged"]
    assert abs(rep.iterations - rr["iterations"]) <= 1
    assert rel(x, xr) <= 1e-6


def test_geometric_mg_and_amg_preconditioners_agree(monkeypatch):
    """Structured unit-square meshes precondition the pole solves with the device geometric MG
    (ert_gmg.cu); GNW_ERT_PC=amg selects the host SA-AMG.  Both converge to the same g and J."""
    mesh, nodes, sv, model = small_case(64, 16, 2, 4)
    c = gpu_ert(mesh, nodes)
    g, J, st = c.response_jacobian(model, sv, tol=1e-13)
    assert st["gmg_levels"] == 3  # 64, 32, 16
    monkeypatch.setenv("GNW_ERT_PC", "amg")
    ga, Ja, sta = c.response_jacobian(model, sv, tol=1e-13)
    assert sta["gmg_levels"] == 0
    assert rel(g, ga) <= 1e-10 and rel(J, Ja) <= 1e-9
    assert st["pcg_iterations"] < sta["pcg_iterations"]


def test_unstructured_cell_order_falls_back_to_amg():
    """A mesh whose cells are not in make_unit_square_mesh order keeps the SA-AMG path and the
    same physics (g is invariant to the cell numbering; J's columns follow the cells)."""
    mesh, nodes, sv, model = small_case(32, 8, 2, 4)
    perm = np.random.default_rng(5).permutation(mesh.n_cells)
    pm = W.Mesh(mesh.vertices, np.ascontiguousarray(mesh.cells[perm]))
    c0, c1 = gpu_ert(mesh, nodes), gpu_ert(pm, nodes)
    g0, J0, st0 = c0.response_jacobian(model, sv, tol=1e-13)
    g1, J1, st1 = c1.response_jacobian(np.ascontiguousarray(model[perm]), sv, tol=1e-13)
    assert st0["gmg_levels"] == 2 and st1["gmg_levels"] == 0
    assert rel(g1, g0) <= 1e-10
    assert rel(J1, J0[:, perm]) <= 1e-9
