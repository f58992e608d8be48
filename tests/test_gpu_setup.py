"""SA-AMG setup products on the device (spgemm.cu): the lumped Schur
complement, A_F T and the Galerkin products computed by the device sparse_matmul give a
hierarchy bit-identical to the host setup (itself pinned bit-exact to the reference in
test_host_setup.py) and to the reference oracle."""
import numpy as np
import pytest

import orc
from paper_2209_02815_b200 import AmgOptions, Context, workload as W

pytestmark = pytest.mark.gpu


def exported(c, n_levels):
    out = {("mat", w): c.export_csr(w) for w in (0, 1, 2)}
    for l in range(n_levels):
        for w in (3, 4):
            out[(w, l)] = c.export_csr(w, l)
    return out


@pytest.mark.parametrize("n,thr", [(32, 64), (64, 64), (256, 64)])
def test_device_setup_products_bitwise(monkeypatch, oracle, n, thr):
    mesh = W.unit_square_mesh(n)
    monkeypatch.setenv("GNW_DEVICE_SPGEMM", "1")
    monkeypatch.setenv("GNW_SPGEMM_MIN", "0")  # every product on the device, however small
    gpu = Context(0)
    gpu.assemble(mesh, AmgOptions(coarse_threshold=thr))
    host = Context(None)
    host.assemble(mesh, AmgOptions(coarse_threshold=thr))
    ig, ih = gpu.info(), host.info()
    assert (ig["n_levels"], ig["coarse_n"]) == (ih["n_levels"], ih["coarse_n"])
    eg, eh = exported(gpu, ig["n_levels"]), exported(host, ih["n_levels"])
    for k in eh:
        for x, y in zip(eg[k], eh[k]):
            assert np.array_equal(np.asarray(x), np.asarray(y)), k
    if n <= 64:  # and against the unmodified reference
        ref = orc.Problem.mixed(oracle, mesh, orc.AmgOpts.make(coarse_threshold=thr))
        for l in range(ref.n_levels):
            for w in (3, 4):
                for x, y in zip(ref.csr(w, l), eg[(w, l)]):
                    assert np.array_equal(np.asarray(x), np.asarray(y)), (w, l)


@pytest.mark.parametrize("n,thr,min_rows", [(32, 64, 0), (64, 64, 0), (256, 64, 0), (256, 64, None)])
def test_device_amg_setup_bitwise(monkeypatch, n, thr, min_rows):
    """The device-resident amg_setup (amg_setup_device.cu: filter, tentative prolongator, smoothing
    product, P merge, transposes, Galerkin product; default on device contexts) against the host
    setup: every level bit for bit, and the V-cycle built on the device-formed one-pass operators
    (S, T, T^T) bitwise the one built on the host-formed ones."""
    mesh = W.unit_square_mesh(n)
    monkeypatch.setenv("GNW_DEVICE_SETUP", "1")
    if min_rows is not None:  # every level on the device (by default levels <= 100000 rows finish on the host)
        monkeypatch.setenv("GNW_DEVICE_SETUP_MIN_ROWS", str(min_rows))
    gpu = Context(0)
    gpu.assemble(mesh, AmgOptions(coarse_threshold=thr))
    monkeypatch.setenv("GNW_DEVICE_SETUP", "0")
    ref = Context(0)
    ref.assemble(mesh, AmgOptions(coarse_threshold=thr))
    host = Context(None)
    host.assemble(mesh, AmgOptions(coarse_threshold=thr))
    ig, ih = gpu.info(), host.info()
    assert (ig["n_levels"], ig["coarse_n"]) == (ih["n_levels"], ih["coarse_n"])
    eg, eh = exported(gpu, ig["n_levels"]), exported(host, ih["n_levels"])
    for k in eh:
        for x, y in zip(eg[k], eh[k]):
            assert np.array_equal(np.asarray(x), np.asarray(y)), k
    rng = np.random.default_rng(n)
    r = rng.standard_normal(mesh.n_cells)
    assert np.array_equal(gpu.amg_apply(r), ref.amg_apply(r))


@pytest.mark.parametrize("name,min_rows", [("p1024", "0"), ("p2048", None)])
def test_device_amg_setup_baseline_mesh_hashes(monkeypatch, name, min_rows):
    """BASELINE C5 mesh (n = 1024, threshold 1024; every level forced onto the device) and C3 mesh
    (n = 2048, threshold 4096; the default split: levels above 100 000 rows on the device, the
    rest on the host): the device setup's hierarchy against the SHA-256 hashes of the unmodified
    reference's own amg_setup (tests/golden/ref_p1024.json, ref_p2048.json)."""
    import refdata

    if not refdata.available(name):
        pytest.skip(f"fixture ref_{name}.json not generated")
    ref = refdata.load(name)
    monkeypatch.setenv("GNW_DEVICE_SETUP", "1")
    if min_rows is not None:
        monkeypatch.setenv("GNW_DEVICE_SETUP_MIN_ROWS", min_rows)
    c = Context(0).assemble(W.unit_square_mesh(ref["n"]), AmgOptions(coarse_threshold=ref["coarse_threshold"]))
    info = c.info()
    assert info["n_levels"] == ref["n_levels"] and info["coarse_n"] == ref["coarse_n"]
    got = refdata.level_hashes_of(c.export_csr, info["n_levels"])
    for l, (g, r) in enumerate(zip(got, ref["levels"])):
        assert g == r, f"level {l}"


def test_setup_error_parity_nonpositive_filtered_diagonal(monkeypatch, oracle):
    """The reference's amg_setup throws std::invalid_argument("amg_setup: non-positive diagonal
    entry") on the 48 x 48 unit square with default options (lumping the weak couplings empties a
    filtered diagonal, amg.cpp:141-166 + 81-88).  The host setup and the device setup raise the
    same error, with the reference's text."""
    mesh = W.unit_square_mesh(48)
    with pytest.raises(Exception) as ref_err:
        orc.Problem.mixed(oracle, mesh)
    assert "non-positive diagonal entry" in str(ref_err.value)
    monkeypatch.setenv("GNW_DEVICE_SETUP", "1")  # small meshes default to the host setup
    monkeypatch.setenv("GNW_DEVICE_SETUP_MIN_ROWS", "0")
    for dev in (None, 0):
        with pytest.raises(ValueError) as err:
            Context(dev).assemble(mesh)
        assert str(err.value) == "amg_setup: non-positive diagonal entry"


@pytest.mark.parametrize("n", [2, 3, 5, 8, 12, 24, 40])
@pytest.mark.parametrize("thr", [4, 64])
def test_device_amg_setup_small_meshes(monkeypatch, n, thr):
    """Edge sizes through the forced device setup (a single level, tiny coarse levels, odd sizes):
    the hierarchy bit for bit the host's, and the V-cycles built on them equal bit for bit."""
    mesh = W.unit_square_mesh(n)
    opts = AmgOptions(coarse_threshold=thr)
    host = Context(None)
    host.assemble(mesh, opts)
    monkeypatch.setenv("GNW_DEVICE_SETUP", "1")
    monkeypatch.setenv("GNW_DEVICE_SETUP_MIN_ROWS", "0")
    dev = Context(0)
    dev.assemble(mesh, opts)
    monkeypatch.setenv("GNW_DEVICE_SETUP", "0")
    ref = Context(0)
    ref.assemble(mesh, opts)
    ih, ig = host.info(), dev.info()
    assert (ih["n_levels"], ih["coarse_n"]) == (ig["n_levels"], ig["coarse_n"])
    eg, eh = exported(dev, ig["n_levels"]), exported(host, ih["n_levels"])
    for k in eh:
        for x, y in zip(eg[k], eh[k]):
            assert np.array_equal(np.asarray(x), np.asarray(y)), k
    r = np.random.default_rng(n).standard_normal(mesh.n_cells)
    assert np.array_equal(dev.amg_apply(r), ref.amg_apply(r))
