"""The product's host-side setup (libgnw.so, gnw_assemble on a host-only context) is
bit-identical to the reference: mesh connectivity, Q, D, S_hat and the whole SA-AMG
hierarchy ("bit-exact mesh and index structures")."""
import os

import numpy as np
import pytest

import orc
from paper_2209_02815_b200 import AmgOptions, Context, workload as W

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def host_ctx(mesh, opts=None):
    return Context(None).assemble(mesh, opts)


def test_golden_mesh_and_assembly():
    c = host_ctx(W.unit_square_mesh(2))
    for k, v in c.export_mesh().items():
        assert np.array_equal(v, GOLD[f"n2_{k}"]), k
    c = host_ctx(W.unit_square_mesh(4))
    for which, name in ((0, "Q"), (1, "D"), (2, "S")):
        nr, nc, rp, ci, va = c.export_csr(which)
        assert np.array_equal(rp, GOLD[f"n4_{name}_rowptr"])
        assert np.array_equal(ci, GOLD[f"n4_{name}_cols"])
        assert np.array_equal(va, GOLD[f"n4_{name}_vals"])


def test_golden_hierarchy():
    c = host_ctx(W.unit_square_mesh(8), AmgOptions(coarse_threshold=16))
    assert c.info()["n_levels"] == int(GOLD["n8_nlevels"][0])
    for l in range(c.info()["n_levels"]):
        for which, name in ((3, "A"), (4, "P")):
            nr, nc, rp, ci, va = c.export_csr(which, l)
            assert np.array_equal(rp, GOLD[f"n8_L{l}_{name}_rowptr"])
            assert np.array_equal(ci, GOLD[f"n8_L{l}_{name}_cols"])
            assert np.array_equal(va, GOLD[f"n8_L{l}_{name}_vals"])


@pytest.mark.parametrize("n,thr,strength", [(1, 64, 0.08), (5, 64, 0.08), (64, 64, 0.08), (48, 16, 0.0),
                                            (128, 64, 0.08), (256, 64, 0.08)])
def test_matches_oracle_bitwise(oracle, n, thr, strength):
    opts_o = orc.AmgOpts.make(coarse_threshold=thr, strength=strength)
    mesh = W.unit_square_mesh(n)
    ref = orc.Problem.mixed(oracle, mesh, opts_o)
    c = host_ctx(mesh, AmgOptions(coarse_threshold=thr, strength=strength))
    info = c.info()
    assert (info["K"], info["N"]) == (ref.K, ref.N) == W.mixed_sizes(n)
    ma, mb = ref.mesh_arrays(), c.export_mesh()
    for k in ma:
        assert np.array_equal(ma[k], mb[k]), k
    for which in (0, 1, 2):
        for x, y in zip(ref.csr(which), c.export_csr(which)):
            assert np.array_equal(np.asarray(x), np.asarray(y)), which
    assert info["n_levels"] == ref.n_levels and info["coarse_n"] == ref.n_coarse
    for l in range(ref.n_levels):
        for which in (3, 4):
            for x, y in zip(ref.csr(which, l), c.export_csr(which, l)):
                assert np.array_equal(np.asarray(x), np.asarray(y)), (which, l)


def test_structure_counts_match_survey():
    # K = 3n^2 + 2n, N = 2n^2, nnz(Q) = 5K - 8n, nnz(D) = 3N, nnz(S) = 4N - 4n
    for n in (16, 64):
        c = host_ctx(W.unit_square_mesh(n))
        K, N = W.mixed_sizes(n)
        assert c.export_csr(0)[4].size == 5 * K - 8 * n
        assert c.export_csr(1)[4].size == 3 * N
        assert c.export_csr(2)[4].size == 4 * N - 4 * n
        info = c.info()
        assert info["n_boundary_edges"] == 4 * n


def test_host_errors_match_reference_text():
    bad = W.Mesh(np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]]), np.array([[0, 1, 2]], dtype=np.int64))
    with pytest.raises(ValueError, match="finalize_mesh: degenerate cell"):
        host_ctx(bad)
    oob = W.Mesh(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]), np.array([[0, 1, 7]], dtype=np.int64))
    with pytest.raises(ValueError, match="vertex index out of range"):
        host_ctx(oob)
    with pytest.raises(ValueError, match="non-positive diagonal entry"):
        host_ctx(W.unit_square_mesh(24), AmgOptions(coarse_threshold=16, strength=0.25))
    c = Context(None)
    with pytest.raises(ValueError, match="not symmetric"):
        c.assemble_amg_csr(np.array([0, 2, 3]), np.array([0, 1, 1]), np.array([2.0, 1.0, 2.0]))


def test_host_only_context_refuses_device_work():
    from paper_2209_02815_b200 import GnwDeviceError
    c = host_ctx(W.unit_square_mesh(4))
    with pytest.raises(GnwDeviceError, match="no device"):
        c.apply_operator(np.zeros(c.K + c.N))
