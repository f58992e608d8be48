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
