"""The persistent small-level V-cycle tail (vcycle_persist.cu: levels below GNW_VC_PERSIST_ROWS
rows plus the dense level in one cooperative launch with grid barriers) computes exactly what
the kernel chain computes (amg.cpp:90-111 in the default-mode order): bit-identical V-cycles,
preconditioner applications and MINRES solves."""
import numpy as np
import pytest

from paper_2209_02815_b200 import AmgOptions, Context, workload as W

pytestmark = pytest.mark.gpu


def ctx_with(monkeypatch, mesh, rows, opts=None):
    monkeypatch.setenv("GNW_VC_PERSIST_ROWS", str(rows))
    c = Context(0)
    c.assemble(mesh, opts)
    return c


@pytest.mark.parametrize("n,thr,rows", [(16, 64, 65536), (64, 64, 65536), (512, 64, 65536), (512, 64, 200000),
                                        (256, 64, 1)])
def test_persistent_tail_bitwise(monkeypatch, n, thr, rows):
    mesh = W.unit_square_mesh(n)
    a = ctx_with(monkeypatch, mesh, rows, AmgOptions(coarse_threshold=thr))
    b = ctx_with(monkeypatch, mesh, 0, AmgOptions(coarse_threshold=thr))
    assert a.info()["persist_level"] >= 0 and b.info()["persist_level"] == -1
    for seed in range(3):
        r = W.gaussian(300 + seed, a.N)
        assert np.array_equal(a.amg_apply(r), b.amg_apply(r))


def test_persistent_tail_solve_bitwise(monkeypatch):
    n, m = 128, 16
    inp = W.gnstep_inputs(n, m, 0)
    out = []
    for rows in (65536, 0):
        c = ctx_with(monkeypatch, inp.mesh, rows)
        c.set_jacobian(inp.J, 1e-2)
        bb = c.assemble_rhs(inp.dm, np.zeros(c.N), inp.dg, np.zeros(m))
        z = c.precondition(bb)
        x, rep = c.minres(bb, tol=1e-10)
        out.append((z, x, rep.iterations))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1]) and out[0][2] == out[1][2]
