"""GPU path (libgnw.so) against the committed reference golden vectors and the reference's
own full C2 run (tests/golden/c2_reference.json) -- needs no reference library at run time."""
import json
import os

import numpy as np
import pytest

from paper_2209_02815_b200 import AmgOptions, Context, workload as W

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(__file__)
GOLD = np.load(os.path.join(HERE, "golden", "golden.npz"))


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


@pytest.fixture(scope="module")
def n8():
    def make(exact):
        c = Context(0)
        c.set_coarse_mode(exact)
        c.assemble(W.unit_square_mesh(8), AmgOptions(coarse_threshold=16))
        return c
    return make


def test_golden_vcycle_exact_bitwise(n8):
    c = n8(True)
    assert np.array_equal(c.amg_apply(GOLD["n8_vcycle_in"]), GOLD["n8_vcycle_out"])


def test_golden_woodbury_and_rhs(n8):
    c = n8(True)
    c.set_jacobian(GOLD["n8_J"], float(GOLD["n8_beta"][0]))
    H, L = c.woodbury_factors()
    assert np.array_equal(H, GOLD["n8_H"])           # batched V-cycles, bit-exact
    assert rel(np.tril(L), GOLD["n8_L"]) <= 1e-13     # tensor-core C, then reference-order Cholesky
    b = c.assemble_rhs(GOLD["n8_dm"], np.zeros(c.N), GOLD["n8_dg"], np.zeros(4))
    assert np.array_equal(b, GOLD["n8_rhs"])
    assert rel(c.apply_operator(GOLD["n8_x"]), GOLD["n8_Ax"]) <= 1e-14
    assert rel(c.precondition(GOLD["n8_x"]), GOLD["n8_Px"]) <= 1e-12


@pytest.mark.parametrize("exact", [True, False])
def test_golden_minres(n8, exact):
    c = n8(exact)
    c.set_jacobian(GOLD["n8_J"], float(GOLD["n8_beta"][0]))
    x, rep = c.minres(GOLD["n8_rhs"], tol=1e-10)
    assert abs(rep.iterations - int(GOLD["n8_iters"][0])) <= 1
    assert rel(x, GOLD["n8_sol"]) <= 1e-8
    k = min(len(rep.relative_residuals), len(GOLD["n8_hist_e"])) - 2
    assert np.allclose(rep.relative_residuals[:k], GOLD["n8_hist_e"][:k], rtol=1e-6, atol=1e-14)
    assert np.allclose(rep.pnorm_relative_residuals[:k], GOLD["n8_hist_p"][:k], rtol=1e-6, atol=1e-14)


def test_c2_iteration_counts_match_reference_run():
    """BASELINE C2 (512^2, m=256), full alpha sweep: iterations within +-1 of the reference's
    own solves on the same seeded bundle; true residual <= 10 tol."""
    rec = json.load(open(os.path.join(HERE, "golden", "c2_reference.json")))
    cfg = W.CONFIGS["C2"]
    inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
    c = Context(0)
    c.assemble(inp.mesh, AmgOptions(coarse_threshold=cfg.coarse_threshold))
    assert c.info()["n_levels"] == 10 and c.info()["coarse_n"] == 171
    for r in rec["runs"]:
        c.set_jacobian(inp.J, r["alpha"])
        b = c.assemble_rhs(inp.dm, np.zeros(c.N), inp.dg, np.zeros(cfg.m))
        x, rep = c.minres(b, tol=1e-8)
        assert rep.converged
        assert abs(rep.iterations - r["iterations"]) <= 1, (r["alpha"], rep.iterations, r["iterations"])
        assert rep.true_relative_residual <= 1e-7
        assert abs(np.linalg.norm(x) - r["x_norm"]) <= 1e-6 * r["x_norm"]
