"""Bit-exact setup structures on the BASELINE C3 and C5 meshes ("bit-exact mesh
and index structures"), against SHA-256 hashes of the unmodified reference's own hierarchy
(tests/golden/ref_p1024.json, ref_p2048.json; amg_setup, amg.cpp:115-187, with the per-config
AmgOptions of SURVEY 8(c): n = 1024 threshold 1024, n = 2048 threshold 4096).  CPU only: the
product's host setup (libgnw.so on a host-only context) is what the GPU path uploads."""
import pytest

import refdata
from paper_2209_02815_b200 import AmgOptions, Context, workload as W

pytestmark = pytest.mark.slow


@pytest.mark.parametrize("name", ["p1024", "p2048"])
def test_baseline_mesh_hierarchy_bitwise(name):
    if not refdata.available(name):
        pytest.skip(f"fixture ref_{name}.json not generated")
    ref = refdata.load(name)
    n, thr = ref["n"], ref["coarse_threshold"]
    c = Context(None).assemble(W.unit_square_mesh(n), AmgOptions(coarse_threshold=thr))
    info = c.info()
    assert (info["K"], info["N"]) == W.mixed_sizes(n)
    assert info["n_levels"] == ref["n_levels"] and info["coarse_n"] == ref["coarse_n"]
    got = refdata.level_hashes_of(c.export_csr, info["n_levels"])
    for l, (g, r) in enumerate(zip(got, ref["levels"])):
        assert g == r, f"level {l}"
